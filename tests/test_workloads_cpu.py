"""The numpy workload generators (oracle/workloads.py) produce exactly the
arrays of libveil's veil_scene_workload, so bench.py's reference arm can build
its input without mapping libveil.so."""
import numpy as np
import pytest

import workloads
from paper_2405_13364_b200 import veil


def same(a, b):
    return (a.vertices.tobytes() == b.vertices.tobytes() and a.quads.tobytes() == b.quads.tobytes()
            and a.materials.tobytes() == b.materials.tobytes() and a.flags == b.flags
            and np.array_equal(a.matrix, b.matrix) and (a.width, a.height) == (b.width, b.height)
            and a.eye is None and b.eye is None)


def test_mt19937_64_known_answer():
    # C++ [rand.predef]: the 10000th output of a default-constructed
    # std::mt19937_64 (seed 5489) is 9981545732273789042
    e = workloads.MT19937_64(5489)
    assert int(e.draws(10000)[-1]) == 9981545732273789042


@pytest.mark.parametrize("name,seed", [("stack64k", 2), ("stack64k", 7), ("tiny4m", 4)])
def test_workload_arrays_equal_libveil(name, seed):
    assert same(workloads.workload(name, seed), veil.Scene.workload(name, seed).arrays())


def test_grid_scene_matches_tiny4m_recipe():
    a = workloads.grid_scene(4, 2048, 2048, 3840, 2160)
    b = workloads.workload("tiny4m", 4)
    assert a.vertices.tobytes() == b.vertices.tobytes() and a.quads.tobytes() == b.quads.tobytes()
