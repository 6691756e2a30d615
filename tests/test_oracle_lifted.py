"""The restatement's extended mode pinned against a limits-lifted reference.

`make -C oracle ref-lifted` builds the unmodified reference sources with
exactly three constants raised (kMaxViewportWidth/Height scene.hpp:90-91 ->
4096, kMaxBins setup.hpp:31 -> 16384). The C4 workload (tiny4m: jittered
grid mesh at 3840x2160, 120x68 bins) needs nothing else: its bin coordinates
fit the 7-bit AABB fields, its 120 bin columns the 128-column masks and its
triangle count 2^24. So on tiny4m-recipe scenes at 3840x2160 the lifted
reference and the restatement's extended mode must agree on every array.
Two encodings differ by design and are compared decoded:

* quad_aabb: 7-bit fields (pack_bin_aabb, packing.hpp:77-82) vs 16-bit ones;
* emit_hash: the extended sample key is (q << 32) | tri, the reference's
  (q << 24) | tri24 (raster.hpp:95-97); the restatement also hashes the
  reference-format key (emit_hash_std), which must equal the reference's.
"""
import numpy as np
import pytest

import bindings
import workloads
from common import PARITY_ARRAYS, compare
from paper_2405_13364_b200.abi import (
    RENDER_ALPHA_THRESHOLD,
    RENDER_FORCE_HIGH_PATH,
    RENDER_VISUALIZE_ERRORS,
    default_params,
)

needs_lifted = pytest.mark.skipif(not bindings.ref_available(lifted=True),
                                  reason="oracle/_ref/libveilref_lifted.so not built here")


def decode_std(a):
    a = a.astype(np.uint64)
    return np.stack([(a >> np.uint64(s)) & np.uint64(127) for s in (0, 7, 14, 21)], 1)


def decode_ext(a):
    a = a.astype(np.uint64)
    return np.stack([(a >> np.uint64(s)) & np.uint64(0xffff) for s in (0, 16, 32, 48)], 1)


def lifted_vs_restatement(arr, params):
    r = bindings.ref_dump_arrays(arr, params, lifted=True)
    assert np.array_equal(r["reenum_image"], r["image"])  # the shim's re-enumeration is the reference's
    o = bindings.oracle_render(arr, params, extended=True)
    assert np.array_equal(decode_std(r["quad_aabb"]), decode_ext(o["quad_aabb"]))
    assert np.array_equal(o["emit_hash_std"], r["emit_hash"])
    bad = compare(o, r, [k for k in PARITY_ARRAYS if k not in ("quad_aabb", "emit_hash")])
    assert not bad, bad
    return r


@needs_lifted
@pytest.mark.parametrize("seed,grid,flags,df", [
    (4, 512, 0, 3),
    (11, 1024, RENDER_VISUALIZE_ERRORS, 1),
    (12, 768, RENDER_ALPHA_THRESHOLD, 3),
    (13, 384, RENDER_FORCE_HIGH_PATH, 5),
])
def test_lifted_reference_vs_extended_restatement_4k(seed, grid, flags, df):
    arr = workloads.grid_scene(seed, grid, grid, 3840, 2160)
    r = lifted_vs_restatement(arr, default_params(flags=flags, depth_filter_size=df))
    assert int(r["counters"][1]) > 0  # fragments were generated


@needs_lifted
def test_lifted_reference_limits_are_the_only_change():
    """The lifted build still enforces the reference's other limits: the
    5120-bin message is gone only because kMaxBins moved, and a viewport over
    the lifted limit is refused with the reference's error."""
    arr = workloads.grid_scene(3, 64, 64, 4097, 64)
    with pytest.raises(bindings.CheckerError) as e:
        bindings.ref_dump_arrays(arr, default_params(), lifted=True)
    assert e.value.status == 3  # VEIL_ERR_INVALID_ARG (scene.cpp:41-42)
