"""OBJ / MTL / camera ingest equals the reference loader (scene.cpp:195-454):
same vertices (numbered by first use of each position/uv/normal corner),
quads, materials, flags and camera, and the same status and message on
malformed input. CPU only: both loaders run on the host."""
import numpy as np
import pytest

import bindings
from paper_2405_13364_b200 import veil

needs_ref = pytest.mark.skipif(not bindings.ref_available(), reason="oracle/_ref not built here")

MTL = """# materials
newmtl red
Kd 1 0.2 0.1
d 0.5
newmtl glass
Kd 0.3 0.3 0.9
d 0.25
bogus line here
"""

OBJS = {
    "plain": "v 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nf 1 2 3 4\nf 1 3 4\n",
    "colours_crlf": "v 0 0 0 1 0 0\r\nv 1 0 0 0 1 0\r\nv 1 1 0 0 0 1\r\n# c\r\nf 1 2 3\r\n",
    "negative_refs": "v 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nvt 0 0\nvt 1 1\nvn 0 0 2\nf -4/-2/-1 -3/-1/-1 -2/-2/-1 -1/-1/-1\n",
    "slashes": ("v 0 0 0\nv 1 0 0\nv 1 1 0\nvt 0.5 0.25\nvn 0 0 0\nvn 1 1 0\n"
                "f 1//1 2//2 3//1\nf 1/1 2/1 3/1\nf 1/1/2 2/1/2 3/1/2\nf 1 2 3\n"),
    "materials": ("mtllib m.mtl\nv 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nusemtl glass\nf 1 2 3 4\n"
                  "usemtl nope\nf 1 2 3\nusemtl red\nf 2 3 4\n"),
    "partial_colour": "v 0 0 0 0.5\nv 1 0 0 0.5 0.5\nv 1 1 0 1 1 1\nf 1 2 3\n",
    "exponents": "v 1e-1 2.5E+0 -3.\nv .5 1 0\nv 0 1e1 0\nf 1 2 3\n",
    "blank_and_tabs": "\n\t v\t0 0 0\nv 1 0 0   \n\nv 0 1 0\nf\t1 2\t3\n",
    # errors
    "bad_vertex": "v 0 0\nf 1 1 1\n",
    "bad_normal": "vn 1 x 0\n",
    "bad_texcoord": "vt 0\n",
    "out_of_range": "v 0 0 0\nv 1 0 0\nv 1 1 0\nf 1 2 9\n",
    "zero_index": "v 0 0 0\nv 1 0 0\nv 1 1 0\nf 0 1 2\n",
    "malformed_corner": "v 0 0 0\nv 1 0 0\nv 1 1 0\nvn 0 0 1\nf //1 2 3\n",
    "arity5": "v 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nv 2 2 0\nf 1 2 3 4 5\n",
    "arity2": "v 0 0 0\nv 1 0 0\nf 1 2\n",
    "bad_uv_ref": "v 0 0 0\nv 1 0 0\nv 1 1 0\nf 1/3 2 3\n",
}


def load_both(tmp_path, name, text, mtl_text=MTL, cam_text=None):
    (tmp_path / "m.mtl").write_text(mtl_text)
    obj = tmp_path / f"{name}.obj"
    obj.write_bytes(text.encode())
    cam = None
    if cam_text is not None:
        cam = tmp_path / "c.cfg"
        cam.write_text(cam_text)
        cam = str(cam)
    mine = ref = None
    try:
        mine = veil.Scene.load(str(obj), None, cam).arrays()
    except veil.VeilError as e:
        mine = (e.status, e.message.replace(str(tmp_path), ""))
    try:
        ref = bindings.RefScene.load(str(obj), None, cam).arrays()
    except bindings.CheckerError as e:
        ref = (e.status, e.message.replace(str(tmp_path), ""))
    return mine, ref


def same_arrays(a, b):
    return (a.vertices.tobytes() == b.vertices.tobytes() and a.quads.tobytes() == b.quads.tobytes()
            and a.materials.tobytes() == b.materials.tobytes() and a.flags == b.flags
            and np.array_equal(a.matrix, b.matrix) and (a.width, a.height) == (b.width, b.height)
            and ((a.eye is None and b.eye is None) or np.array_equal(a.eye, b.eye)))


@needs_ref
@pytest.mark.parametrize("name", sorted(OBJS))
def test_obj_ingest_equals_reference(tmp_path, name):
    mine, ref = load_both(tmp_path, name, OBJS[name])
    if isinstance(ref, tuple) or isinstance(mine, tuple):
        assert mine == ref
    else:
        assert same_arrays(mine, ref)


@needs_ref
@pytest.mark.parametrize("cam", [
    "width = 320\nheight = 200\nlook_from = 1 2 3\nlook_at = 0 0 0\nup = 0 1 0\nfov_deg = 45\nnear=0.2\nfar = 50\n",
    "view_projection = 1 0 0 0 0 1 0 0 0 0 1 0 0 0 0 1\nwidth=64\nheight=32\neye = 0 0 -4\n",
    "# c\nwidth = 100\nlook_from = 0 0 9\neye = 1 1 1\n",
    "width = 100\nfoo = 1\n",
    "width = 100\nlook_from = 1 2\n",
    "width = 9000\n",
])
def test_camera_config_equals_reference(tmp_path, cam):
    mine, ref = load_both(tmp_path, "tri", OBJS["plain"], cam_text=cam)
    if isinstance(ref, tuple) or isinstance(mine, tuple):
        assert mine == ref
    else:
        assert same_arrays(mine, ref)


@needs_ref
def test_mtl_dissolve_range_error(tmp_path):
    mine, ref = load_both(tmp_path, "m", OBJS["materials"], mtl_text="newmtl a\nd 1.5\n")
    assert isinstance(mine, tuple) and mine == ref
