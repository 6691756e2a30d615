"""Generates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Test infrastructure: run here (where /root/reference exists) after
`make -C oracle ref`. Each fixture stores the scene arrays, the render
params and the reference's outputs (setup records, bin lists, tri-half-block
lists, per-pixel blend-order hashes, image, mask, counters), so tests on the
GPU box can check both the C restatement and libveil without the reference.

    python oracle/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from bindings import RefScene  # noqa: E402
from paper_2405_13364_b200.abi import (  # noqa: E402
    RENDER_ALPHA_THRESHOLD,
    RENDER_BACKFACE_CULLING,
    RENDER_FORCE_HIGH_PATH,
    RENDER_VISUALIZE_ERRORS,
    default_params,
)

SCENES = "/root/reference/proj/scenes"
OUT = os.path.join(ROOT, "tests", "golden")

KEEP = ["quad_source", "quad_aabb", "quad_class", "quad_attr", "tri_valid", "tri_yrange",
        "tri_fn", "tri_meta", "setup_stats", "bin_dims", "bin_quad_counts", "bin_tri_counts",
        "bin_offsets", "bin_categories", "bin_items", "bin_path", "thb_offsets", "thb",
        "thb_prefix", "emit_hash", "emit_count", "image", "mask", "counters"]


def params_dict(p):
    return {
        "flags": p.flags, "depth_filter_size": p.depth_filter_size,
        "background": list(p.background), "light_dir": list(p.light_dir), "ambient": p.ambient,
        "limit_low_tbr": p.limit_low_tbr, "limit_low_tri_blocks": p.limit_low_tri_blocks,
        "limit_low_frags": p.limit_low_frags, "limit_high_tbr": p.limit_high_tbr,
        "limit_high_thb": p.limit_high_thb,
    }


def save(name, rs, params, note):
    arr = rs.arrays()
    d = rs.dump(params)
    out = {k: d[k] for k in KEEP if k in d}
    assert np.array_equal(d["reenum_image"], d["image"]), name
    out.update(
        scene_vertices=arr.vertices, scene_quads=arr.quads, scene_materials=arr.materials,
        scene_flags=np.array([arr.flags]), scene_matrix=arr.matrix,
        scene_size=np.array([arr.width, arr.height]),
        scene_eye=arr.eye if arr.eye is not None else np.zeros(0),
        params=np.frombuffer(json.dumps(params_dict(params)).encode(), dtype=np.uint8),
        note=np.frombuffer(note.encode(), dtype=np.uint8),
    )
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **out)
    print(f"{name}: {os.path.getsize(path)} bytes, counters {d['counters'].tolist()}")


def main():
    os.makedirs(OUT, exist_ok=True)
    boxes = RefScene.load(f"{SCENES}/boxes.obj", None, f"{SCENES}/boxes_camera.cfg")
    boxes.set_viewport(256, 256)
    save("c1_boxes_256", boxes, default_params(), "BASELINE.json configs[0]: boxes at 256x256")
    save("c1_boxes_256_backface", boxes,
         default_params(flags=RENDER_BACKFACE_CULLING | RENDER_ALPHA_THRESHOLD),
         "boxes 256x256 with backface culling and alpha threshold")
    s = RefScene.synthetic("layered_quads", 6, 128, 128)
    save("layered_s6_tight", s, default_params(limit_low_tri_blocks=4),
         "test_raster.cpp:258-277 analogue: tight low limits propagate every bin")
    s = RefScene.synthetic("intersecting_shells", 5, 128, 128)
    save("shells_s5_df1_vis", s,
         default_params(depth_filter_size=1, flags=RENDER_VISUALIZE_ERRORS),
         "test_raster.cpp:297-315 analogue: DF=1 invalid pixels + magenta overlay")
    s = RefScene.synthetic("random_soup", 17, 128, 128)
    save("soup_s17_forcehigh", s, default_params(flags=RENDER_FORCE_HIGH_PATH),
         "test_raster.cpp:241-256 analogue: forced high path")
    s = RefScene.synthetic("dense_bin", 3, 256, 256)
    save("dense_s3", s, default_params(), "dense bin: one high-category bin")
    s = RefScene.synthetic("layered_quads", 2, 96, 80)
    save("layered_s2_threshold", s, default_params(flags=RENDER_ALPHA_THRESHOLD, depth_filter_size=2),
         "alpha threshold with ragged viewport 96x80")
    # textured materials (map_Kd, mip-mapped, repeat wrap, perspective UV
    # gradients): the scene is the OBJ/MTL/PNG set in tests/golden/textured
    tex = os.path.join(OUT, "textured")
    s = RefScene.load(os.path.join(tex, "scene.obj"), None, os.path.join(tex, "camera.cfg"))
    save("textured_scene", s, default_params(), "tests/golden/textured: 3 materials, 2 mip-mapped textures")
    save("textured_scene_df1_backface", s,
         default_params(depth_filter_size=1, flags=RENDER_BACKFACE_CULLING | RENDER_VISUALIZE_ERRORS),
         "textured scene with DF=1, backface culling, error overlay")


if __name__ == "__main__":
    main()
