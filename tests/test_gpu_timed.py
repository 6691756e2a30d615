"""veil_render_device_timed: the caller's CUDA events bracket exactly the
frame's device work (bench.py's timed region), and timing a frame does not
change it."""
import numpy as np
import pytest

from common import boxes_arrays
from paper_2405_13364_b200 import veil
from paper_2405_13364_b200.abi import default_params

pytestmark = pytest.mark.gpu


def test_timed_events_bracket_the_frame():
    import torch

    scene = veil.Scene.workload("stack64k", 2)
    params = default_params()
    ref = veil.render(scene, params)
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.ExternalStream(scene.stream())
    start.record(stream)  # torch creates its events at their first record
    end.record(stream)
    torch.cuda.synchronize()
    ms = []
    for _ in range(3):
        veil.render_device(scene, params, None, stats=False, events=(start.cuda_event, end.cuda_event))
        torch.cuda.synchronize()
        ms.append(start.elapsed_time(end))
    st = scene.last_stats()
    # the events hold the whole frame graph: at least the span of its stage
    # events, and not far beyond it (no host latency inside)
    assert min(ms) >= 0.95 * st.total_ms
    assert min(ms) <= st.total_ms + 0.5
    assert int(st.fragments) == int(ref.stats().fragments)
    # the same frame as veil_render_scene
    again = veil.render(scene, params)
    assert np.array_equal(again.pixels(), ref.pixels())
    assert np.array_equal(again.invalid_mask(), ref.invalid_mask())


def test_timed_events_are_optional():
    scene = veil.Scene.from_arrays(boxes_arrays(256, 256))
    veil.render_device(scene, default_params(), None, stats=False, events=(None, None))
    assert scene.last_stats().fragments > 0
