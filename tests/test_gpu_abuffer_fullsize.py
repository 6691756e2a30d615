"""The GPU a-buffer (VEIL_RENDER_REFERENCE, k_abuffer: the reference's
oracle.cpp:28-117 exact per-pixel sort on the bin lists) validates images at
the benchmarked sizes, where the CPU oracle is too slow.

A pixel whose depth filter never emitted out of order (invalid mask 0) was
blended in exact key order, so the pipeline's pixel must equal the a-buffer's
there; the a-buffer's sample total equals the pipeline's fragment total
(acceptance.cpp:128-133). The a-buffer itself is pinned against the
restatement's a-buffer on small scenes (test_gpu_parity.py) and the
restatement's against the reference's (test_oracle.py)."""
import numpy as np
import pytest

from paper_2405_13364_b200 import veil
from paper_2405_13364_b200.abi import RENDER_REFERENCE, default_params

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,seed,df", [("stack64k", 2, 3), ("tiny4m", 4, 3), ("mixed16m", 5, 3),
                                          ("mixed16m", 5, 16)])
def test_pipeline_equals_gpu_abuffer_where_valid(name, seed, df):
    sc = veil.Scene.workload(name, seed)
    pipe = veil.render(sc, default_params(depth_filter_size=df))
    ref = veil.render(sc, default_params(flags=RENDER_REFERENCE))
    a, b, mask = pipe.pixels(), ref.pixels(), pipe.invalid_mask()
    valid = mask == 0
    assert np.array_equal(a[valid], b[valid]), (name, int((a != b).any(axis=-1)[valid].sum()))
    assert int(ref.stats().samples) == int(pipe.stats().fragments)
    if name != "mixed16m":  # the meshes and the stack have no disorder beyond DF 3
        assert int(mask.sum()) == 0 and np.array_equal(a, b)
