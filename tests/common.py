"""Shared test helpers: golden fixtures, scene builders, dump comparison."""
import glob
import json
import os

import numpy as np

from paper_2405_13364_b200.abi import (
    MATERIAL_DTYPE,
    MATERIAL_VERTEX_COLORS,
    MATERIAL_VERTEX_NORMALS,
    QUAD_DTYPE,
    SCENE_HAS_COLORS,
    SCENE_HAS_NORMALS,
    VERTEX_DTYPE,
    SceneArrays,
    default_params,
)

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")
REF_SCENES = "/root/reference/proj/scenes"

# Every array both the reference dump and the restatement/libveil produce.
PARITY_ARRAYS = [
    "quad_source", "quad_aabb", "quad_class", "quad_attr", "tri_valid", "tri_yrange", "tri_fn",
    "tri_meta", "setup_stats", "bin_dims", "bin_quad_counts", "bin_tri_counts", "bin_offsets",
    "bin_categories", "bin_items", "bin_path", "thb_offsets", "thb", "thb_prefix", "emit_hash",
    "emit_count", "image", "mask", "counters",
]


def golden_names():
    """Array-scene fixtures (the textured OBJ fixtures load their scene from
    tests/golden/textured and have their own tests)."""
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if not os.path.basename(p).startswith("textured"))


TEXTURED = os.path.join(GOLDEN, "textured")


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    eye = z["scene_eye"]
    scene = SceneArrays(z["scene_vertices"], z["scene_quads"], z["scene_materials"],
                        int(z["scene_flags"][0]), z["scene_matrix"], int(z["scene_size"][0]),
                        int(z["scene_size"][1]), eye if len(eye) else None)
    p = json.loads(bytes(z["params"]).decode())
    params = default_params(**p)
    expect = {k: z[k] for k in PARITY_ARRAYS if k in z}
    return scene, params, expect


def compare(got, expect, names=None, label=""):
    """Returns the list of arrays that differ (empty = bit-exact)."""
    bad = []
    for k in names or expect:
        if k not in expect:
            continue
        if k not in got:
            bad.append(f"{k}: missing")
            continue
        a, b = np.asarray(got[k]), np.asarray(expect[k])
        if k == "quad_aabb":
            a, b = a.astype(np.uint64), b.astype(np.uint64)
        if a.shape != b.shape:
            bad.append(f"{k}: shape {a.shape} != {b.shape}")
        elif not np.array_equal(a, b):
            idx = np.flatnonzero(a.reshape(-1) != b.reshape(-1))
            bad.append(f"{k}: {len(idx)} differ, first at {idx[0]}: {a.reshape(-1)[idx[0]]} vs {b.reshape(-1)[idx[0]]}")
    return bad


def clip_scene(width, height, flags=SCENE_HAS_COLORS | SCENE_HAS_NORMALS):
    """ClipSceneBuilder of the reference tests (test_util.hpp:51-90)."""

    class B:
        def __init__(self):
            self.v = []
            self.q = []
            self.w, self.h = width, height

        def vertex(self, x, y, z, color=(1, 1, 1, 1)):
            self.v.append(((x, y, z), (0, 0, -1), tuple(color), (0, 0)))
            return len(self.v) - 1

        def ndc(self, px, py):
            return 2.0 * px / self.w - 1.0, 1.0 - 2.0 * py / self.h

        def pixel_rect(self, px0, py0, px1, py1, z, color=(1, 1, 1, 1)):
            c = [self.ndc(px0, py0), self.ndc(px1, py0), self.ndc(px1, py1), self.ndc(px0, py1)]
            ids = [self.vertex(x, y, z, color) for x, y in c]
            self.q.append((ids, 0))

        def pixel_triangle(self, p0, p1, p2, z, color=(1, 1, 1, 1)):
            ids = [self.vertex(*self.ndc(*p), z, color) for p in (p0, p1, p2)]
            self.q.append((ids + [ids[2]], 0))

        def quad_ids(self, ids):
            self.q.append((list(ids), 0))

        def build(self):
            v = np.zeros(len(self.v), dtype=VERTEX_DTYPE)
            for i, (p, n, c, uv) in enumerate(self.v):
                v[i] = (p, n, c, uv)
            q = np.zeros(len(self.q), dtype=QUAD_DTYPE)
            for i, (ids, m) in enumerate(self.q):
                q[i] = (ids, m)
            m = np.zeros(1, dtype=MATERIAL_DTYPE)
            m[0] = ((1, 1, 1, 1), 1.0, -1, MATERIAL_VERTEX_COLORS | MATERIAL_VERTEX_NORMALS)
            return SceneArrays(v, q, m, flags, np.eye(4).reshape(16), self.w, self.h)

    return B()


def boxes_arrays(width=256, height=256):
    """The bundled boxes scene (reference proj/scenes/boxes.obj + camera), as
    captured from the reference loader into the C1 golden fixture."""
    scene, _, _ = load_golden("c1_boxes_256")
    scene.width, scene.height = width, height
    return scene


def fuzz_scene(seed):
    """Seeded random scene + render parameters for the fuzz parity tests:
    random quads and triangles (some degenerate, some reaching behind the
    eye), random per-vertex colours/normals (zero normals included), several
    materials with mixed flags, a random perspective camera (sometimes inside
    the geometry) and viewport, random render flags and depth-filter size."""
    from paper_2405_13364_b200 import veil
    from paper_2405_13364_b200.abi import (
        RENDER_ALPHA_THRESHOLD, RENDER_BACKFACE_CULLING, RENDER_FORCE_HIGH_PATH,
        RENDER_VISUALIZE_ERRORS)
    rng = np.random.default_rng(1000 + seed)
    w, h = int(rng.integers(8, 300)), int(rng.integers(8, 200))
    nq = int(rng.integers(1, 600))
    spread = float(rng.choice([0.5, 2.0, 6.0]))
    centres = rng.uniform(-2, 2, (nq, 3))
    size = rng.choice([0.02, 0.2, 1.0, 3.0], nq)[:, None, None]
    v = np.zeros(4 * nq, dtype=VERTEX_DTYPE)
    pos = centres[:, None, :] + size * rng.normal(0, 1, (nq, 4, 3)) * spread / 2
    v["position"] = pos.reshape(-1, 3)
    nrm = rng.normal(0, 1, (4 * nq, 3))
    nrm[rng.random(4 * nq) < 0.05] = 0.0
    v["normal"] = nrm
    col = rng.uniform(0, 1, (4 * nq, 4))
    col[:, 3] = rng.choice([0.05, 0.3, 0.6, 0.95, 1.0], 4 * nq)
    v["color"] = col
    q = np.zeros(nq, dtype=QUAD_DTYPE)
    ids = np.arange(4 * nq, dtype=np.uint32).reshape(nq, 4)
    tri = rng.random(nq) < 0.3
    ids[tri, 3] = ids[tri, 2]  # triangles
    dup = rng.random(nq) < 0.05
    ids[dup, 1] = ids[dup, 0]  # degenerate
    q["v"] = ids
    nm = int(rng.integers(1, 4))
    q["material"] = rng.integers(0, nm, nq)
    m = np.zeros(nm, dtype=MATERIAL_DTYPE)
    for i in range(nm):
        m[i] = (tuple(rng.uniform(0.2, 1, 4)), float(rng.choice([0.1, 0.5, 1.0])), -1,
                int(rng.integers(0, 4)))
    eye = rng.uniform(-1, 1, 3) * (1.0 if rng.random() < 0.25 else 8.0)
    at = rng.uniform(-1, 1, 3)
    fov = float(rng.choice([30.0, 60.0, 100.0]))
    near = float(rng.choice([0.01, 0.1, 1.0]))
    mat = veil.look_at(list(eye), list(at), [0, 1, 0], fov, near, 50.0, w, h)
    arr = SceneArrays(v, q, m, SCENE_HAS_COLORS | SCENE_HAS_NORMALS, mat, w, h,
                      list(eye) if rng.random() < 0.5 else None)
    flags = 0
    for f in (RENDER_ALPHA_THRESHOLD, RENDER_FORCE_HIGH_PATH, RENDER_BACKFACE_CULLING,
              RENDER_VISUALIZE_ERRORS):
        if rng.random() < 0.3:
            flags |= f
    params = default_params(flags=flags, depth_filter_size=int(rng.choice([1, 2, 3, 5, 8, 16])))
    return arr, params


def read_png_rgba(path):
    """Decodes an 8-bit RGBA, non-interlaced PNG (what veil_render_write_png
    writes) with zlib: IHDR, IDAT chunks, per-row filters 0-4."""
    import struct
    import zlib

    data = open(path, "rb").read()
    assert data[:8] == b"\x89PNG\r\n\x1a\n"
    pos, idat, w, h = 8, b"", 0, 0
    while pos < len(data):
        n, kind = struct.unpack(">I4s", data[pos:pos + 8])
        body = data[pos + 8:pos + 8 + n]
        if kind == b"IHDR":
            w, h, depth, ctype, _, _, interlace = struct.unpack(">IIBBBBB", body)
            assert depth == 8 and ctype == 6 and interlace == 0
        elif kind == b"IDAT":
            idat += body
        pos += 12 + n
    raw = np.frombuffer(zlib.decompress(idat), dtype=np.uint8).reshape(h, 1 + 4 * w)
    out = np.zeros((h, 4 * w), dtype=np.int32)
    for y in range(h):
        f, line = raw[y, 0], raw[y, 1:].astype(np.int32)
        prev = out[y - 1] if y else np.zeros(4 * w, dtype=np.int32)
        if f == 0:
            out[y] = line
        elif f == 2:
            out[y] = (line + prev) & 255
        else:
            row = np.zeros(4 * w, dtype=np.int32)
            for i in range(4 * w):
                a = row[i - 4] if i >= 4 else 0
                b = prev[i]
                c = prev[i - 4] if i >= 4 else 0
                if f == 1:
                    p = a
                elif f == 3:
                    p = (a + b) // 2
                else:
                    pa, pb, pc = abs(b - c), abs(a - c), abs(a + b - 2 * c)
                    p = a if (pa <= pb and pa <= pc) else (b if pb <= pc else c)
                row[i] = (line[i] + p) & 255
            out[y] = row
    return out.astype(np.uint8).reshape(h, w, 4)
