"""The drop-in boundary on CPU: libveil.so loads, exports every symbol the
headers declare, the headers are C-clean (reference tests/capi_compiles.c),
parameter defaults and error statuses match the reference C API
(reference c_api.cpp:85-249), and host-side scene ingest produces exactly the
reference's scenes. No kernel runs here."""
import ctypes as C
import os
import subprocess
import zlib
import struct

import numpy as np
import pytest

import bindings
from common import REF_SCENES
from paper_2405_13364_b200 import veil
from paper_2405_13364_b200.abi import (
    VEIL_ERR_INVALID_ARG,
    VEIL_ERR_IO,
    VEIL_ERR_PARSE,
    RenderParams,
)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
needs_ref = pytest.mark.skipif(not bindings.ref_available(), reason="oracle/_ref not built here")

REFERENCE_SYMBOLS = [  # reference veil.h:43-124
    "veil_status_string", "veil_last_error", "veil_scene_load", "veil_scene_synthetic",
    "veil_scene_group_quads", "veil_scene_set_viewport", "veil_scene_set_camera",
    "veil_scene_destroy", "veil_render_params_init", "veil_render_scene", "veil_render_width",
    "veil_render_height", "veil_render_pixels", "veil_render_invalid_mask",
    "veil_render_report_json", "veil_render_write_png", "veil_render_destroy", "veil_compare_png",
]


def _exported():
    out = subprocess.run(["nm", "-D", "--defined-only", veil.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if " T " in line}


def test_library_exports_every_declared_symbol():
    exported = _exported()
    declared = veil.exported_symbols()
    assert set(REFERENCE_SYMBOLS) <= set(declared)
    missing = [s for s in declared if s not in exported]
    assert not missing, missing


@pytest.mark.parametrize("header", ["veil.h", "veil_cuda.h"])
def test_headers_are_c_clean(tmp_path, header):
    src = tmp_path / "t.c"
    src.write_text(f'#include "{header}"\nint main(void) {{ veil_render_params p; '
                   'veil_render_params_init(&p); return p.depth_filter_size == 3 ? 0 : 1; }\n')
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-fsyntax-only",
                    "-I", os.path.join(ROOT, "include"), str(src)], check=True)


def test_params_layout_and_defaults():
    p = RenderParams()
    veil.lib().veil_render_params_init(C.byref(p))
    assert C.sizeof(p) == 64
    assert (p.flags, p.depth_filter_size, p.thread_count) == (0, 3, 0)
    assert list(p.background) == [0, 0, 0, 1]
    assert np.allclose(list(p.light_dir), [0.3, -0.5, 0.8]) and abs(p.ambient - 0.2) < 1e-7
    assert (p.limit_low_tbr, p.limit_low_tri_blocks, p.limit_low_frags,
            p.limit_high_tbr, p.limit_high_thb) == (0, 0, 0, 0, 0)


def test_status_strings():
    L = veil.lib()
    expect = {0: "ok", 1: "I/O error", 2: "parse error", 3: "invalid argument",
              4: "capacity exceeded", 5: "internal error", 9: "unknown status"}
    for k, v in expect.items():
        assert L.veil_status_string(k).decode() == v


def test_null_arguments_are_invalid():
    L = veil.lib()
    h = C.c_void_p()
    assert L.veil_scene_load(None, None, None, C.byref(h)) == VEIL_ERR_INVALID_ARG
    assert L.veil_render_scene(None, None, C.byref(h)) == VEIL_ERR_INVALID_ARG
    assert L.veil_scene_set_viewport(None, 10, 10) == VEIL_ERR_INVALID_ARG
    assert L.veil_scene_group_quads(None, None) == VEIL_ERR_INVALID_ARG
    L.veil_scene_destroy(None)
    L.veil_render_destroy(None)
    assert L.veil_render_width(None) == 0 and L.veil_render_report_json(None) == b""


def test_unknown_synthetic_kind():
    with pytest.raises(veil.VeilError) as e:
        veil.Scene.synthetic("teapot", 1)
    assert e.value.status == VEIL_ERR_INVALID_ARG


def test_viewport_limits():
    s = veil.Scene.synthetic("layered_quads", 1, 64, 64)
    with pytest.raises(veil.VeilError) as e:
        s.set_viewport(3840, 2160)
    assert e.value.status == VEIL_ERR_INVALID_ARG
    assert e.value.message == "viewport exceeds the 2560x2048 limit"
    with pytest.raises(veil.VeilError):
        s.set_viewport(0, 10)
    s.set_viewport_ext(3840, 2160)  # veil_cuda.h extended limits
    assert (s.arrays().width, s.arrays().height) == (3840, 2160)


def test_obj_errors(tmp_path):
    bad = tmp_path / "bad.obj"
    bad.write_text("v 0 0 0\nv 1 0 0\nv 0 1 0\nv 1 1 0\nv 2 2 0\nf 1 2 3 4 5\n")
    with pytest.raises(veil.VeilError) as e:
        veil.Scene.load(str(bad))
    assert e.value.status == VEIL_ERR_PARSE and "arity 5" in e.value.message
    oob = tmp_path / "oob.obj"
    oob.write_text("v 0 0 0\nf 1 2 99\n")
    with pytest.raises(veil.VeilError) as e:
        veil.Scene.load(str(oob))
    assert e.value.status == VEIL_ERR_PARSE and "out of range" in e.value.message
    with pytest.raises(veil.VeilError) as e:
        veil.Scene.load(str(tmp_path / "missing.obj"))
    assert e.value.status == VEIL_ERR_IO
    cam = tmp_path / "c.cfg"
    cam.write_text("zoom = 3\n")
    good = tmp_path / "tri.obj"
    good.write_text("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n")
    with pytest.raises(veil.VeilError) as e:
        veil.Scene.load(str(good), None, str(cam))
    assert e.value.status == VEIL_ERR_PARSE and "unknown camera key" in e.value.message
    a = veil.Scene.load(str(good)).arrays()
    assert len(a.quads) == 1 and list(a.quads[0]["v"]) == [0, 1, 2, 2]  # degenerate quad


def _write_png(path, rgba):
    h, w, _ = rgba.shape
    raw = b"".join(b"\x00" + rgba[y].tobytes() for y in range(h))
    def chunk(t, d):
        return struct.pack(">I", len(d)) + t + d + struct.pack(">I", zlib.crc32(t + d) & 0xFFFFFFFF)
    data = (b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, 8, 6, 0, 0, 0))
            + chunk(b"IDAT", zlib.compress(raw)) + chunk(b"IEND", b""))
    open(path, "wb").write(data)


def test_compare_png(tmp_path):
    rng = np.random.default_rng(0)
    a = rng.integers(0, 255, (17, 23, 4), dtype=np.uint8)
    b = a.copy()
    b[3, 4, 1] = (int(b[3, 4, 1]) + 7) % 256
    b[10, 2, 0] = (int(b[10, 2, 0]) + 1) % 256
    _write_png(tmp_path / "a.png", a)
    _write_png(tmp_path / "b.png", b)
    d = veil.compare_png(str(tmp_path / "a.png"), str(tmp_path / "b.png"))
    assert (d.differing_pixels, d.width, d.height) == (2, 23, 17)
    assert d.max_channel_delta == max(abs(int(b[3, 4, 1]) - int(a[3, 4, 1])),
                                      abs(int(b[10, 2, 0]) - int(a[10, 2, 0])))


def test_workloads_deterministic_and_sized():
    a = veil.Scene.workload("stack64k", 2).arrays()
    b = veil.Scene.workload("stack64k", 2).arrays()
    assert np.array_equal(a.vertices, b.vertices) and len(a.quads) == 65536
    t = veil.Scene.workload("tiny4m", 4).arrays()
    assert len(t.quads) == 2048 * 2048 and len(t.vertices) == 2049 * 2049
    assert (t.width, t.height) == (3840, 2160)


@needs_ref
def test_boxes_ingest_matches_reference():
    mine = veil.Scene.load(f"{REF_SCENES}/boxes.obj", None, f"{REF_SCENES}/boxes_camera.cfg")
    ref = bindings.RefScene.load(f"{REF_SCENES}/boxes.obj", None, f"{REF_SCENES}/boxes_camera.cfg")
    for w, h in ((512, 512), (256, 256), (1920, 1080)):
        mine.set_viewport(w, h)
        ref.set_viewport(w, h)
        a, b = mine.arrays(), ref.arrays()
        assert np.array_equal(a.vertices, b.vertices) and np.array_equal(a.quads, b.quads)
        assert np.array_equal(a.materials, b.materials) and a.flags == b.flags
        assert np.array_equal(a.matrix, b.matrix) and np.array_equal(a.eye, b.eye)


@needs_ref
@pytest.mark.parametrize("kind", ["layered_quads", "intersecting_shells", "random_soup", "dense_bin"])
@pytest.mark.parametrize("seed", [0, 3, 77])
def test_synthetic_ingest_matches_reference(kind, seed):
    a = veil.Scene.synthetic(kind, seed, 200, 150).arrays()
    b = bindings.RefScene.synthetic(kind, seed, 200, 150).arrays()
    assert np.array_equal(a.vertices, b.vertices) and np.array_equal(a.quads, b.quads)
    assert np.array_equal(a.materials, b.materials) and a.flags == b.flags


@needs_ref
def test_look_at_matches_reference(tmp_path):
    cfg = tmp_path / "cam.cfg"
    cfg.write_text("width = 640\nheight = 360\nlook_from = 3 2 7\nlook_at = 0.5 0 0\n"
                   "up = 0 1 0\nfov_deg = 41\nnear = 0.25\nfar = 90\n")
    obj = tmp_path / "tri.obj"
    obj.write_text("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n")
    ref = bindings.RefScene.load(str(obj), None, str(cfg)).arrays()
    m = veil.look_at([3, 2, 7], [0.5, 0, 0], [0, 1, 0], 41.0, 0.25, 90.0, 640, 360)
    assert np.array_equal(m, ref.matrix)
    mine = veil.Scene.load(str(obj), None, str(cfg)).arrays()
    assert np.array_equal(mine.matrix, ref.matrix) and np.array_equal(mine.eye, ref.eye)


@needs_ref
def test_group_quads_matches_reference(tmp_path):
    rng = np.random.default_rng(5)
    n = 12
    lines = [f"v {x} {y} {rng.uniform(-0.1, 0.1):.4f}" for y in range(n) for x in range(n)]
    for y in range(n - 1):
        for x in range(n - 1):
            a, b, c, d = y * n + x + 1, y * n + x + 2, (y + 1) * n + x + 2, (y + 1) * n + x + 1
            if rng.random() < 0.5:
                lines += [f"f {a} {b} {c}", f"f {a} {c} {d}"]
            else:
                lines += [f"f {a} {b} {d}", f"f {b} {c} {d}"]
    obj = tmp_path / "tris.obj"
    obj.write_text("\n".join(lines) + "\n")
    mine = veil.Scene.load(str(obj))
    ref = bindings.RefScene.load(str(obj))
    assert abs(mine.group_quads() - ref.group_quads()) < 1e-12
    assert np.array_equal(mine.arrays().quads, ref.arrays().quads)
    with pytest.raises(veil.VeilError):
        mine.group_quads()  # already paired: invalid argument (grouping.cpp:159-162)


def test_render_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(veil.VeilError) as e:
        veil.render(veil.Scene.synthetic("layered_quads", 1, 32, 32))
    assert "no CUDA device" in e.value.message


@needs_ref
def test_textured_obj_ingest_matches_reference():
    from common import TEXTURED
    mine = veil.Scene.load(f"{TEXTURED}/scene.obj", None, f"{TEXTURED}/camera.cfg").arrays()
    ref = bindings.RefScene.load(f"{TEXTURED}/scene.obj", None, f"{TEXTURED}/camera.cfg").arrays()
    assert np.array_equal(mine.vertices, ref.vertices) and np.array_equal(mine.quads, ref.quads)
    assert np.array_equal(mine.materials, ref.materials) and mine.flags == ref.flags
    assert np.array_equal(mine.matrix, ref.matrix)
