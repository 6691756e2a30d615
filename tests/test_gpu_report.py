"""veil_render_report_json value parity with the reference (report.cpp:21-68).

The reference's schema and values -- config echo, samples, tri_half_blocks,
s_per_thb, fragments, segments, setup_stats (visible_percent,
degenerate_quad_percent), bins, invalid_pixels (count, percent) -- must be
the same for the same scene and parameters, key order included. Only the
wall-clock timings_us differ, and libveil appends an additive "device"
object (CUDA-event stage times, kernel launches)."""
import json

import pytest

import bindings
from common import boxes_arrays
from paper_2405_13364_b200 import veil
from paper_2405_13364_b200.abi import (
    RENDER_ALPHA_THRESHOLD,
    RENDER_BACKFACE_CULLING,
    RENDER_FORCE_HIGH_PATH,
    RENDER_REFERENCE,
    RENDER_VISUALIZE_ERRORS,
    default_params,
)

pytestmark = pytest.mark.gpu


def strip(rep):
    rep = dict(rep)
    rep.pop("timings_us")
    rep.pop("device", None)
    return rep


def scenes():
    yield "boxes256", boxes_arrays(256, 256)
    for kind, size in (("random_soup", (160, 128)), ("dense_bin", (256, 256)),
                       ("intersecting_shells", (128, 96))):
        yield kind, bindings.RefScene.synthetic(kind, 9, *size).arrays()
    # degenerate quads (degenerate_quad_percent > 0) and frustum culls
    from common import fuzz_scene

    yield "fuzz3", fuzz_scene(3)[0]


@pytest.mark.parametrize("flags,df", [(0, 3), (RENDER_ALPHA_THRESHOLD, 3),
                                      (RENDER_BACKFACE_CULLING | RENDER_VISUALIZE_ERRORS, 1),
                                      (RENDER_FORCE_HIGH_PATH, 12), (RENDER_REFERENCE, 3)])
def test_report_json_equals_reference(flags, df):
    for name, arr in scenes():
        p = default_params(flags=flags, depth_filter_size=df, thread_count=4)
        _, _, ref = bindings.RefScene.from_arrays(arr).render(p)
        ours = veil.render(veil.Scene.from_arrays(arr), p).report()
        assert list(ours)[: len(ref)] == list(ref), name  # reference keys first, same order
        a, b = strip(ours), strip(ref)
        assert json.dumps(a) == json.dumps(b), (name, a, b)
