"""veil_render_scene_multi: a frame sharded over several devices from one
process (bins interleaved, every shard's shading kernels writing into the
first device's framebuffer). The box these tests run on has one GPU, so the
device lists repeat device 0: the shards then run one after another on it
(frames on one device are serialised) and write the same framebuffer, which
exercises the sharding, the peer-pointer writes and the stat merge; across
distinct devices the same writes go over NVLink. Output must be identical
for any device list (acceptance.cpp:423-453)."""
import numpy as np
import pytest

from common import boxes_arrays
from paper_2405_13364_b200 import veil
from paper_2405_13364_b200.abi import RENDER_ALPHA_THRESHOLD, VEIL_ERR_INVALID_ARG, default_params

pytestmark = pytest.mark.gpu

COUNTERS = ("samples", "fragments", "tri_half_blocks", "segments", "invalid_pixels", "bins_empty",
            "bins_low", "bins_high", "bins_propagated", "visible_quads", "input_quads")


def scenes():
    yield "stack64k", veil.Scene.workload("stack64k", 2), default_params()
    sc = veil.Scene.from_arrays(boxes_arrays(1920, 1080))
    yield "boxes1080", sc, default_params()
    yield "tiny4m", veil.Scene.workload("tiny4m", 4), default_params()
    yield "stack64k_df12_threshold", veil.Scene.workload("stack64k", 2), default_params(
        depth_filter_size=12, flags=RENDER_ALPHA_THRESHOLD)


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0], [0, 0, 0, 0, 0, 0, 0, 0]])
def test_multi_device_frame_identical_to_single(devices):
    for name, sc, p in scenes():
        one = veil.render(sc, p)
        many = veil.render_multi(sc, devices, p)
        assert np.array_equal(many.pixels(), one.pixels()), (name, devices)
        assert np.array_equal(many.invalid_mask(), one.invalid_mask()), (name, devices)
        a, b = many.stats(), one.stats()
        for k in COUNTERS:
            assert getattr(a, k) == getattr(b, k), (name, devices, k)
        ra, rb = many.report(), one.report()
        for k in ("samples", "fragments", "tri_half_blocks", "segments", "bins", "invalid_pixels"):
            assert ra[k] == rb[k], (name, k)


def test_multi_device_argument_errors():
    sc = veil.Scene.workload("stack64k", 2)
    with pytest.raises(veil.VeilError) as e:
        veil.render_multi(sc, [0, 99])
    assert e.value.status == VEIL_ERR_INVALID_ARG
    with pytest.raises(veil.VeilError):
        veil.render_multi(sc, [])
