"""The boundary from C: tests/c/capi_render.c is compiled with gcc against
include/veil.h and linked against libveil.so (no Python, no torch on the
path), like an application of the reference's C library. On CPU it must
compile and link; on a GPU it renders and its pixels must equal the
restatement's image of the same synthetic scene."""
import json
import os
import subprocess

import numpy as np
import pytest

import bindings
from paper_2405_13364_b200 import veil
from paper_2405_13364_b200.abi import default_params

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.dirname(veil.LIB_PATH)


def _build(tmp_path):
    exe = tmp_path / "capi_render"
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-O2",
                    "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "c", "capi_render.c"),
                    "-L", LIBDIR, "-l:libveil.so", f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)],
                   check=True)
    return exe


def test_c_embedder_compiles_and_links(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run(["ldd", str(exe)], capture_output=True, text=True).stdout
    assert "libveil.so" in out


@pytest.mark.gpu
@pytest.mark.parametrize("kind,seed,w,h,df", [("layered_quads", 7, 256, 192, 3),
                                              ("random_soup", 3, 200, 150, 8)])
def test_c_embedder_renders_reference_image(tmp_path, kind, seed, w, h, df):
    exe = _build(tmp_path)
    png, raw = tmp_path / "f.png", tmp_path / "f.raw"
    p = subprocess.run([str(exe), kind, str(seed), str(w), str(h), str(df), str(png), str(raw)],
                       capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr
    report = json.loads(p.stdout)
    data = np.fromfile(raw, dtype=np.uint8)
    rgba, mask = data[: w * h * 4], data[w * h * 4:]
    arr = veil.Scene.synthetic(kind, seed, w, h).arrays()
    exp = bindings.oracle_render(arr, default_params(depth_filter_size=df), names=["image", "mask", "counters"])
    assert np.array_equal(rgba, exp["image"].reshape(-1))
    assert np.array_equal(mask, exp["mask"].reshape(-1))
    assert report["fragments"] == int(exp["counters"][1])
    assert veil.compare_png(str(png), str(png)).differing_pixels == 0
