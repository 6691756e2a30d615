"""libveil (sm_100a) vs the reference: bit-exact parity through the C ABI.

Oracle: the committed reference fixtures (tests/golden, produced by the
unmodified reference via oracle/make_golden.py) and the C restatement
(oracle/liboracle.so) on the same seeded scenes. Bar: every setup record,
bin list, tri-half-block list, per-pixel blend-order hash, image byte, mask
byte and counter identical.
"""
import numpy as np
import pytest

import bindings
from common import PARITY_ARRAYS, boxes_arrays, clip_scene, compare, golden_names, load_golden
from paper_2405_13364_b200 import veil
from paper_2405_13364_b200.abi import (
    RENDER_ALPHA_THRESHOLD,
    RENDER_BACKFACE_CULLING,
    RENDER_FORCE_HIGH_PATH,
    RENDER_REFERENCE,
    RENDER_VISUALIZE_ERRORS,
    VEIL_ERR_CAPACITY,
    VEIL_ERR_INVALID_ARG,
    default_params,
)

pytestmark = pytest.mark.gpu


def gpu_dump(arrays, params):
    return veil.render_dump(veil.Scene.from_arrays(arrays), params)


@pytest.mark.parametrize("name", golden_names())
def test_golden_fixture(name):
    scene, params, expect = load_golden(name)
    bad = compare(gpu_dump(scene, params), expect)
    assert not bad, bad


FLAG_SETS = [0, RENDER_ALPHA_THRESHOLD, RENDER_FORCE_HIGH_PATH,
             RENDER_BACKFACE_CULLING | RENDER_VISUALIZE_ERRORS]


@pytest.mark.parametrize("kind,size", [("layered_quads", (128, 128)),
                                       ("intersecting_shells", (128, 96)),
                                       ("random_soup", (160, 128)),
                                       ("dense_bin", (256, 256))])
@pytest.mark.parametrize("flags", FLAG_SETS)
@pytest.mark.parametrize("df", [1, 3, 8])
def test_synthetic_vs_restatement(kind, size, flags, df):
    arr = veil.Scene.synthetic(kind, 11, *size).arrays()
    p = default_params(flags=flags, depth_filter_size=df)
    expect = bindings.oracle_render(arr, p)
    bad = compare(gpu_dump(arr, p), expect, PARITY_ARRAYS)
    assert not bad, bad


@pytest.mark.parametrize("frame", [0, 9, 21, 40])
@pytest.mark.parametrize("backface", [False, True])
def test_boxes_orbit_vs_restatement(frame, backface):
    """C3 camera path at 320x180: perspective, large quads."""
    arr = boxes_arrays(320, 180)
    R = np.hypot(5.5, 9.0)
    th = np.arctan2(5.5, 9.0) + 2 * np.pi * frame / 64
    eye = [R * np.sin(th), 4.5, R * np.cos(th)]
    m = veil.look_at(eye, [0, 0, 0], [0, 1, 0], 55.0, 0.5, 40.0, 320, 180)
    arr = arr.with_camera(m, eye)
    p = default_params(flags=RENDER_BACKFACE_CULLING if backface else 0)
    bad = compare(gpu_dump(arr, p), bindings.oracle_render(arr, p), PARITY_ARRAYS)
    assert not bad, bad


def test_camera_inside_scene_w_crossing():
    """Eye inside the boxes: edges cross w = 0 (Blinn AABB extension)."""
    arr = boxes_arrays(200, 150)
    eye = [0.2, 0.1, 0.3]
    m = veil.look_at(eye, [3, -1, -2], [0, 1, 0], 90.0, 0.05, 40.0, 200, 150)
    for e in (eye, None):
        a = arr.with_camera(m, e)
        p = default_params(flags=RENDER_BACKFACE_CULLING)
        bad = compare(gpu_dump(a, p), bindings.oracle_render(a, p), PARITY_ARRAYS)
        assert not bad, bad


def test_stack_workload_small_vs_restatement():
    """The C2 generator at a reduced viewport (every stage exercised)."""
    s = veil.Scene.workload("stack64k", 2, 320, 180)
    arr = s.arrays()
    keep = 3000
    arr.quads = arr.quads[:keep].copy()
    p = default_params()
    bad = compare(gpu_dump(arr, p), bindings.oracle_render(arr, p), PARITY_ARRAYS)
    assert not bad, bad


def test_tiny_grid_extended_vs_restatement():
    """C4-style jittered grid mesh with extended limits, reduced size."""
    s = veil.Scene.workload("tiny4m", 4, 3840, 2160)
    arr = s.arrays()
    # keep the first 64 grid rows (2048 quads per row), at a 2600x300 viewport
    arr.quads = arr.quads[: 2048 * 64].copy()
    arr.width, arr.height = 2600, 300
    p = default_params()
    exp = bindings.oracle_render(arr, p, extended=True)
    sc = veil.Scene.from_arrays(arr)
    got = veil.render_dump(sc, p)
    bad = compare(got, exp, PARITY_ARRAYS)
    assert not bad, bad


def test_reference_abuffer_mode_matches_restatement():
    arr = veil.Scene.synthetic("random_soup", 4, 128, 128).arrays()
    p = default_params(flags=RENDER_REFERENCE)
    exp = bindings.oracle_render(arr, p)
    got = gpu_dump(arr, p)
    for k in ("image", "emit_hash", "emit_count"):
        assert np.array_equal(got[k], exp[k]), k


def test_pipeline_equals_abuffer_when_disorder_within_df():
    """test_oracle.cpp:45-53 / acceptance criterion 1 analogue."""
    sc = veil.Scene.synthetic("layered_quads", 3, 160, 120)
    a = veil.render(sc, default_params()).pixels()
    b = veil.render(sc, default_params(flags=RENDER_REFERENCE)).pixels()
    assert np.array_equal(a, b)


def test_capacity_error_names_the_bin():
    """test_raster.cpp:279-295: 4100 stacked tiny triangles -> high limit."""
    b = clip_scene(32, 32)
    for i in range(4100):
        z = 0.1 + 0.0001 * (i % 1000)
        b.pixel_triangle((-2, -2), (10, -2), (-2, 6), z, (1, 1, 1, 0.2))
    sc = veil.Scene.from_arrays(b.build())
    with pytest.raises(veil.VeilError) as e:
        veil.render(sc)
    assert e.value.status == VEIL_ERR_CAPACITY
    assert "bin (0,0)" in e.value.message
    with pytest.raises(bindings.CheckerError) as e2:
        bindings.oracle_render(b.build())
    assert e2.value.message == e.value.message


def test_invalid_limits_rejected():
    sc = veil.Scene.synthetic("layered_quads", 6, 128, 128)
    with pytest.raises(veil.VeilError) as e:
        veil.render(sc, default_params(limit_low_tbr=1 << 20))
    assert e.value.status == VEIL_ERR_INVALID_ARG


def test_segment_arithmetic_300_layers():
    """test_raster.cpp:158-177: 300 full-coverage layers on 64x64."""
    b = clip_scene(64, 64)
    for i in range(300):
        b.pixel_triangle((-80, -80), (200, -10), (-10, 200), 0.1 + 0.6 * (i / 300.0),
                         (1, 1, 1, 0.01))
    r = veil.render(veil.Scene.from_arrays(b.build()))
    rep = r.report()
    assert rep["segments"] == 4 * 32 * 38
    assert rep["samples"] == 300 * 64 * 64
    assert rep["fragments"] == rep["samples"]
    assert rep["tri_half_blocks"] == 4 * 32 * 300
    assert rep["bins"]["low"] == 4 and rep["bins"]["propagated"] == 4


def test_alpha_threshold_opaque_front():
    """test_raster.cpp:197-214: exactly one blended sample per pixel."""
    b = clip_scene(64, 64)
    for i in range(6):
        b.pixel_triangle((-200, -200), (400, -20), (-20, 400), 0.2 + 0.1 * i,
                         (0.8, 0.6, 0.4, 1.0 if i == 0 else 0.5))
    sc = veil.Scene.from_arrays(b.build())
    base = veil.render(sc)
    fast = veil.render(sc, default_params(flags=RENDER_ALPHA_THRESHOLD))
    assert base.report()["samples"] == 6 * 64 * 64
    assert fast.report()["samples"] == 64 * 64
    assert np.array_equal(base.pixels(), fast.pixels())


def test_low_path_1023_vs_1025():
    """test_raster.cpp:216-239: 1023 triangle-equivalents stay low."""
    b = clip_scene(192, 64)
    for i in range(511):
        x0, y0 = 1 + (i % 5) * 6, 1 + ((i // 5) % 5) * 6
        b.pixel_rect(x0, y0, x0 + 5, y0 + 5, 0.1 + 0.001 * i, (1, 1, 1, 0.1))
    b.pixel_triangle((-5, 24), (200, 24), (-5, 30), 0.05)
    rep = veil.render(veil.Scene.from_arrays(b.build())).report()
    assert rep["bins"]["high"] == 0 and rep["bins"]["propagated"] == 0 and rep["bins"]["low"] == 6
    b.pixel_rect(5, 5, 11, 11, 0.5, (1, 1, 1, 0.1))
    assert veil.render(veil.Scene.from_arrays(b.build())).report()["bins"]["high"] == 1


def test_deterministic_across_runs():
    arr = veil.Scene.workload("stack64k", 2, 640, 360).arrays()
    arr.quads = arr.quads[:8000].copy()
    sc = veil.Scene.from_arrays(arr)
    a = veil.render_dump(sc)
    b = veil.render_dump(sc)
    assert not compare(a, b, PARITY_ARRAYS)


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_sharded_render_reassembles_full_frame(world):
    """Bin-interleaved shards (8(e)) combine to the single-GPU frame."""
    sc = veil.Scene.synthetic("random_soup", 8, 256, 192)
    full = veil.render(sc)
    img = np.zeros_like(full.pixels())
    mask = np.zeros_like(full.invalid_mask())
    total_samples = 0
    bx, by = (256 + 31) // 32, (192 + 31) // 32
    for r in range(world):
        part = veil.render(sc, shard=(r, world))
        px, m = part.pixels(), part.invalid_mask()
        for y in range(by):
            for x in range(bx):
                if (x + 3 * y) % world == r:
                    img[y * 32:(y + 1) * 32, x * 32:(x + 1) * 32] = px[y * 32:(y + 1) * 32, x * 32:(x + 1) * 32]
                    mask[y * 32:(y + 1) * 32, x * 32:(x + 1) * 32] = m[y * 32:(y + 1) * 32, x * 32:(x + 1) * 32]
        total_samples += part.report()["samples"]
    assert np.array_equal(img, full.pixels())
    assert np.array_equal(mask, full.invalid_mask())
    assert total_samples == full.report()["samples"]


def test_report_schema():
    rep = veil.render(veil.Scene.synthetic("layered_quads", 1, 64, 64)).report()
    for key in ("config", "timings_us", "samples", "tri_half_blocks", "s_per_thb", "fragments",
                "segments", "setup_stats", "bins", "invalid_pixels"):
        assert key in rep
    for key in ("setup", "binning", "low_raster", "hi_raster", "total"):
        assert key in rep["timings_us"]


def test_png_roundtrip(tmp_path):
    r = veil.render(veil.Scene.synthetic("intersecting_shells", 2, 96, 64))
    a, b = str(tmp_path / "a.png"), str(tmp_path / "b.png")
    r.write_png(a)
    r.write_png(b)
    d = veil.compare_png(a, b)
    assert d.differing_pixels == 0 and d.width == 96 and d.height == 64


def test_graph_replay_across_cameras_and_params():
    """Non-dump frames replay one cached CUDA graph per launch shape: the
    camera and colours change through the c_fc upload, depth-filter size and
    flags change the graph. Every frame must still equal the restatement."""
    arr = boxes_arrays(320, 180)
    sc = veil.Scene.from_arrays(arr)
    R = np.hypot(5.5, 9.0)
    cases = [(f, df, flags, bg) for f, (df, flags, bg) in enumerate(
        [(3, 0, (0, 0, 0, 1)), (3, 0, (0.2, 0.4, 0.1, 1)), (3, 0, (0, 0, 0, 1)),
         (1, 0, (0, 0, 0, 1)), (3, RENDER_ALPHA_THRESHOLD, (0, 0, 0, 1)),
         (3, RENDER_BACKFACE_CULLING, (0.5, 0.5, 0.5, 0.5)), (3, 0, (0, 0, 0, 1))])]
    for f, df, flags, bg in cases:
        th = np.arctan2(5.5, 9.0) + 2 * np.pi * f / 11
        eye = [R * np.sin(th), 4.5, R * np.cos(th)]
        m = veil.look_at(eye, [0, 0, 0], [0, 1, 0], 55.0, 0.5, 40.0, 320, 180)
        sc.set_camera(m, eye)
        p = default_params(flags=flags, depth_filter_size=df, background=bg)
        r = veil.render(sc, p)
        exp = bindings.oracle_render(arr.with_camera(m, eye), p, names=["image", "mask"])
        assert np.array_equal(r.pixels().reshape(-1), exp["image"].reshape(-1)), (f, df, flags)
        assert np.array_equal(r.invalid_mask().reshape(-1), exp["mask"].reshape(-1)), (f, df, flags)


@pytest.mark.parametrize("kind,size", [("random_soup", (160, 128)), ("dense_bin", (256, 256))])
def test_rasterizer_independent_of_bin_item_order(kind, size, monkeypatch):
    """Frames skip the canonical per-bin sort (only dumps need it): with the
    lists left in atomic-scatter order every THB list, per-pixel blend-order
    hash, image byte and counter must still equal the restatement, and each
    bin must hold the same items."""
    arr = veil.Scene.synthetic(kind, 5, *size).arrays()
    p = default_params()
    expect = bindings.oracle_render(arr, p)
    monkeypatch.setenv("VEIL_BIN_SORT", "0")
    got = gpu_dump(arr, p)
    names = [n for n in PARITY_ARRAYS if n != "bin_items"]
    bad = compare(got, expect, names)
    assert not bad, bad
    offs, qc, tc = expect["bin_offsets"], expect["bin_quad_counts"], expect["bin_tri_counts"]
    for b in range(len(offs)):
        o, n = int(offs[b]), int(qc[b]) + int(tc[b])
        assert np.array_equal(np.sort(got["bin_items"][o:o + n]), np.sort(expect["bin_items"][o:o + n])), b


@pytest.mark.parametrize("df", [2, 5, 16, 32])
@pytest.mark.parametrize("flags", [0, RENDER_ALPHA_THRESHOLD])
def test_depth_filter_capacities_vs_restatement(df, flags):
    """Depth-filter sizes beyond the default: exact-capacity register/slot
    filters (2, 5), the runtime-capacity ones (16, 32), with and without the
    alpha threshold, on a high-disorder scene."""
    arr = veil.Scene.synthetic("dense_bin", 4, 192, 160).arrays()
    p = default_params(flags=flags, depth_filter_size=df)
    bad = compare(gpu_dump(arr, p), bindings.oracle_render(arr, p), PARITY_ARRAYS)
    assert not bad, bad


def test_mixed_workload_window_vs_restatement():
    """The C5 generator (jittered grid + stacked translucent quads, extended
    limits) through a camera window of 512x480 grid cells at the original
    pixel density (960x540): the segment-routing shade path runs next to the
    wave walk in the same bins."""
    arr = veil.Scene.workload("mixed16m", 5, 7680, 4320).arrays()
    pos = arr.vertices["position"]
    q = arr.quads["v"].astype(np.int64)
    qx, qy = pos[q, 0], pos[q, 1]
    lo, hi = -1.0, -1.0 + 2.0 * 512 / 4096  # x window; y uses 480 of 3840 rows (same 1/8)
    keep = (qx.max(1) >= lo) & (qx.min(1) <= hi) & (qy.max(1) >= lo) & (qy.min(1) <= hi)
    arr.quads = arr.quads[keep].copy()
    assert 200_000 < len(arr.quads) < 400_000
    m = np.array([8, 0, 0, 7, 0, 8, 0, 7, 0, 0, 1, 0, 0, 0, 0, 1], dtype=np.float64)
    arr = arr.with_camera(m, None, 960, 540)
    p = default_params()
    exp = bindings.oracle_render(arr, p, extended=True)
    sc = veil.Scene.from_arrays(arr)
    sc.set_extended_limits(True)  # the C5 encodings (32-bit triangle keys, 16-bit bin boxes)
    got = veil.render_dump(sc, p)
    bad = compare(got, exp, PARITY_ARRAYS)
    assert not bad, bad


@pytest.mark.parametrize("kind,size", [("dense_bin", (256, 256)), ("intersecting_shells", (200, 150))])
def test_capacity_growth_retry(kind, size, monkeypatch):
    """Every grow-on-demand buffer (bin items, large-triangle pairs, THB pool)
    starts tiny, so the first frames overflow and re-run with grown
    capacities (also through the cached frame graph); dumps and plain frames
    must still equal the restatement."""
    monkeypatch.setenv("VEIL_INITIAL_CAPACITY", "64")
    arr = veil.Scene.synthetic(kind, 9, *size).arrays()
    p = default_params()
    exp = bindings.oracle_render(arr, p)
    sc = veil.Scene.from_arrays(arr)
    r = veil.render(sc, p)  # graph path first: grows inside render_frame's retry loop
    assert np.array_equal(r.pixels().reshape(-1), exp["image"].reshape(-1))
    bad = compare(veil.render_dump(veil.Scene.from_arrays(arr), p), exp, PARITY_ARRAYS)
    assert not bad, bad


@pytest.mark.parametrize("name", ["textured_scene", "textured_scene_df1_backface"])
def test_textured_scene_vs_reference_fixture(name):
    """Textured materials (map_Kd PNGs, mip chains, repeat wrap, perspective
    UV gradients) through libveil's OBJ/MTL/PNG ingest: culling, bins, THB
    lists, per-pixel blend order, mask and counters bit-exact against the
    reference's fixture; RGBA within 1/255 (the mip level comes from CUDA's
    log2f where the reference uses the C library's)."""
    from common import TEXTURED
    _, params, expect = load_golden(name)
    sc = veil.Scene.load(f"{TEXTURED}/scene.obj", None, f"{TEXTURED}/camera.cfg")
    got = veil.render_dump(sc, params)
    bad = compare(got, expect, [n for n in PARITY_ARRAYS if n != "image"])
    assert not bad, bad
    diff = np.abs(got["image"].astype(int) - expect["image"].astype(int))
    assert diff.max() <= 1, diff.max()
    assert (diff > 0).mean() < 1e-3


def _edge_case(b, params=None, extended=False):
    arr = b.build()
    p = params or default_params()
    exp = bindings.oracle_render(arr, p, extended=extended)
    sc = veil.Scene.from_arrays(arr)
    if extended:
        sc.set_extended_limits(True)
    got = veil.render_dump(sc, p)
    bad = compare(got, exp, PARITY_ARRAYS)
    assert not bad, bad
    r = veil.render(sc, p)  # the graph / zero-copy path as well
    assert np.array_equal(r.pixels().reshape(-1), exp["image"].reshape(-1))
    return got


def test_edge_all_culled():
    """Every quad culled (behind the camera, degenerate, outside, between samples)."""
    b = clip_scene(96, 64)
    b.pixel_rect(10, 10, 40, 40, -0.5)          # z < 0: outside the clip volume
    b.pixel_rect(200, 10, 240, 40, 0.5)         # right of the viewport
    b.pixel_rect(10.2, 10.2, 10.4, 10.4, 0.5)   # covers no pixel centre
    v = b.vertex(0.1, 0.1, 0.5)
    b.quad_ids([v, v, v, v])                    # degenerate
    got = _edge_case(b)
    assert int(got["counters"][1]) == 0


@pytest.mark.parametrize("df", [1, 3, 8])
def test_edge_flat_depth_planes(df):
    """Screen-parallel quads (depth plane a = b = 0, the plane every C2 quad
    has) at the clip-volume depth bounds and in between, over and under a
    sloped quad: libveil's flat-plane shortcuts (quantized depth staged per
    triangle for shading, no centroid divisions for the extraction keys)
    must give the same keys, order and image as per-sample evaluation."""
    b = clip_scene(96, 64)
    b.pixel_rect(-4, -4, 100, 70, 0.0, (0.9, 0.1, 0.1, 0.4))    # z = 0: quantizes to 0
    b.pixel_rect(8, 4, 90, 60, 1.0, (0.1, 0.9, 0.1, 0.4))       # z = w: quantizes to the max
    b.pixel_rect(20, 10, 70, 50, 1e-30, (0.1, 0.1, 0.9, 0.5))   # below one depth quantum
    b.pixel_rect(30, 0, 64, 64, 0.5, (0.7, 0.7, 0.2, 0.6))
    b.pixel_rect(33, 3, 61, 61, 0.5, (0.2, 0.7, 0.7, 0.6))      # same depth: tie-break by triangle
    ids = [b.vertex(-0.8, -0.8, 0.2, (1, 0.5, 0.2, 0.5)), b.vertex(0.8, -0.8, 0.6, (0.2, 1, 0.5, 0.5)),
           b.vertex(0.8, 0.8, 0.9, (0.5, 0.2, 1, 0.5)), b.vertex(-0.8, 0.8, 0.4, (1, 1, 1, 0.5))]
    b.quad_ids(ids)                                             # sloped depth plane
    _edge_case(b, default_params(depth_filter_size=df))


@pytest.mark.parametrize("w,h", [(1, 1), (33, 1), (1, 65), (31, 33)])
def test_edge_tiny_and_ragged_viewports(w, h):
    b = clip_scene(w, h)
    b.pixel_rect(-2, -2, w + 2, h + 2, 0.4, (0.9, 0.2, 0.1, 0.5))
    b.pixel_rect(0, 0, max(1, w // 2), max(1, h // 2), 0.3, (0.1, 0.8, 0.2, 0.7))
    _edge_case(b)


def test_edge_wide_extended_viewport():
    """A 16384-pixel-wide viewport (extended limits): 512 bin columns, the
    128-bit column masks of large-triangle binning widened."""
    b = clip_scene(16384, 48)
    b.pixel_rect(100, 4, 16300, 40, 0.5, (0.4, 0.4, 0.9, 0.6))
    b.pixel_rect(8000, 0, 8100, 48, 0.4, (0.9, 0.4, 0.1, 0.8))
    b.pixel_triangle((30, 2), (16000, 20), (40, 46), 0.45, (0.2, 0.9, 0.5, 0.5))
    _edge_case(b, extended=True)


@pytest.mark.parametrize("seed", range(48))
def test_fuzz_vs_restatement(seed):
    """Seeded random scenes, cameras, flags and depth-filter sizes (the same
    generator the restatement is checked with against the live reference in
    test_oracle.py); errors must match too."""
    from common import fuzz_scene
    arr, p = fuzz_scene(seed)
    try:
        expect = bindings.oracle_render(arr, p)
    except bindings.CheckerError as e:
        with pytest.raises(veil.VeilError) as g:
            gpu_dump(arr, p)
        assert (g.value.status, g.value.message) == (e.status, e.message)
        return
    bad = compare(gpu_dump(arr, p), expect, PARITY_ARRAYS)
    assert not bad, bad
