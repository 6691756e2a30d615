"""Depth-filter sizes above 8 on the device (ring filter), bit-exact.

The reference's DepthFilter has no capacity bound (depth_filter.hpp:31-60);
render_pipeline only requires DF >= 1 (renderer.cpp:70-72) and its CLI
allows 1..1024 (veil_cli.cpp:81-82). libveil runs DF <= 8 in register
filters and every larger DF in a per-pixel sorted ring (shared memory when it
fits beside the staged triangles, global scratch otherwise). Scenes:
intersecting_shells with 128 / 300 sheets (reference synthetic.cpp, via the
shim's generate_synthetic_scene with SyntheticParams), whose measured
disorder is 36 / 84, so filters of 33..84 emit out of order and larger ones
sort every pixel exactly.
"""
import os

import numpy as np
import pytest

import bindings
from common import PARITY_ARRAYS, compare
from paper_2405_13364_b200 import veil
from paper_2405_13364_b200.abi import (
    RENDER_ALPHA_THRESHOLD,
    RENDER_FORCE_HIGH_PATH,
    RENDER_REFERENCE,
    RENDER_VISUALIZE_ERRORS,
    default_params,
)

pytestmark = pytest.mark.gpu


def shells(sheets, size=(256, 256), seed=3):
    return bindings.RefScene.synthetic_params("intersecting_shells", seed, *size, sheets=sheets).arrays()


def gpu_dump(arrays, params):
    return veil.render_dump(veil.Scene.from_arrays(arrays), params)


@pytest.mark.parametrize("df", [9, 12, 16, 20, 21, 24, 32, 33, 64, 256, 1024])
@pytest.mark.parametrize("flags", [0, RENDER_ALPHA_THRESHOLD, RENDER_VISUALIZE_ERRORS | RENDER_FORCE_HIGH_PATH])
def test_large_depth_filter_vs_restatement(df, flags):
    arr = shells(128)
    p = default_params(flags=flags, depth_filter_size=df)
    bad = compare(gpu_dump(arr, p), bindings.oracle_render(arr, p), PARITY_ARRAYS)
    assert not bad, bad


@pytest.mark.parametrize("df", [40, 84, 85, 1024, 5000])
def test_large_depth_filter_300_sheets(df):
    """DF above the high-path THB limit (4096) behaves like an unbounded filter."""
    arr = shells(300, (192, 160))
    p = default_params(depth_filter_size=df)
    bad = compare(gpu_dump(arr, p), bindings.oracle_render(arr, p), PARITY_ARRAYS)
    assert not bad, bad


@pytest.mark.parametrize("df", [12, 16, 17])
def test_ring_in_global_memory_equals_shared(df, monkeypatch):
    """The global-scratch ring (VEIL_DFM_GLOBAL=1) is bit-identical."""
    arr = shells(128)
    p = default_params(depth_filter_size=df)
    monkeypatch.setenv("VEIL_DFM_GLOBAL", "1")
    got = gpu_dump(arr, p)
    bad = compare(got, bindings.oracle_render(arr, p), PARITY_ARRAYS)
    assert not bad, bad


def test_large_depth_filter_segment_kernel():
    """Tiny triangles (segment routing, k_shade mode 1) with a ring filter."""
    arr = bindings.RefScene.synthetic_params("random_soup", 5, 192, 160, triangles=20000).arrays()
    for df in (9, 40):
        p = default_params(depth_filter_size=df)
        bad = compare(gpu_dump(arr, p), bindings.oracle_render(arr, p), PARITY_ARRAYS)
        assert not bad, (df, bad)


def acceptance_cases():
    """acceptance.cpp:80-101 (criterion 1) plus deep intersecting shells."""
    cases = []
    for s in (1, 2):
        for layers in (4, 16, 48):
            cases.append(("layered_quads", s, dict(layers=layers)))
    for s in (1, 2):
        for tris in (1000, 3000, 10000):
            cases.append(("random_soup", s, dict(triangles=tris)))
    for s in range(1, 9):
        cases.append(("dense_bin", s, {}))
    for s, sheets in ((1, 64), (2, 128), (3, 300)):
        cases.append(("intersecting_shells", s, dict(sheets=sheets)))
    return cases


@pytest.mark.parametrize("kind,seed,kw", acceptance_cases())
def test_acceptance_oracle_exactness(kind, seed, kw):
    """Acceptance criterion 1 analogue (acceptance.cpp:80-160) at 512x512:
    DF = the reference pipeline's measured disorder; libveil's frame must
    equal the reference's a-buffer image byte for byte, with the a-buffer's
    fragment total, and libveil's own a-buffer mode must agree."""
    rs = bindings.RefScene.synthetic_params(kind, seed, 512, 512, **kw)
    arr = rs.arrays()
    disorder = max(0, rs.measure_disorder(default_params()))
    sc = veil.Scene.from_arrays(arr)
    assert veil.measure_disorder(sc, default_params()) == disorder  # libveil measures the same
    df = max(1, disorder)
    if disorder <= 3:
        df = 3  # the measuring render already repaired it (acceptance.cpp:118-124)
    img_ref, _, rep_ref = rs.render(default_params(flags=RENDER_REFERENCE))
    r = veil.render(sc, default_params(depth_filter_size=df))
    assert np.array_equal(r.pixels(), img_ref), (kind, seed, kw, df)
    assert int(r.stats().fragments) == int(rep_ref["samples"])
    assert int(r.stats().invalid_pixels) == 0
    g = veil.render(sc, default_params(flags=RENDER_REFERENCE))
    assert np.array_equal(g.pixels(), img_ref)


@pytest.mark.parametrize("kind,seed,kw", [
    ("intersecting_shells", 3, dict(sheets=128)), ("intersecting_shells", 3, dict(sheets=300)),
    ("intersecting_shells", 1, dict(sheets=64)), ("random_soup", 1, dict(triangles=10000)),
    ("random_soup", 2, dict(triangles=1000)), ("layered_quads", 1, dict(layers=48)),
    ("dense_bin", 4, {})])
@pytest.mark.parametrize("flags", [0, RENDER_FORCE_HIGH_PATH])
def test_measure_disorder_equals_reference(kind, seed, kw, flags):
    """veil_measure_disorder == the reference pipeline's max_disorder
    (RenderConfig::measure_disorder, raster.cpp:286-297, through the shim)."""
    rs = bindings.RefScene.synthetic_params(kind, seed, 256, 256, **kw)
    p = default_params(flags=flags)
    assert veil.measure_disorder(veil.Scene.from_arrays(rs.arrays()), p) == max(0, rs.measure_disorder(p))
