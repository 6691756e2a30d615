"""ctypes mirrors of the C structures in include/veil.h and include/veil_cuda.h.

Pure data definitions (no library is loaded here) so that the product
binding (``paper_2405_13364_b200.veil``) and the test-side oracle bindings
(``oracle/bindings.py``) describe the C ABI once.
"""
import ctypes as C

import numpy as np

VEIL_OK = 0
VEIL_ERR_IO = 1
VEIL_ERR_PARSE = 2
VEIL_ERR_INVALID_ARG = 3
VEIL_ERR_CAPACITY = 4
VEIL_ERR_INTERNAL = 5

# veil.h:72-78 (reference) / include/veil.h
RENDER_REFERENCE = 1 << 0
RENDER_ALPHA_THRESHOLD = 1 << 1
RENDER_VISUALIZE_ERRORS = 1 << 2
RENDER_FORCE_HIGH_PATH = 1 << 3
RENDER_BACKFACE_CULLING = 1 << 4

MATERIAL_VERTEX_COLORS = 1
MATERIAL_VERTEX_NORMALS = 2
MATERIAL_UVS = 4
SCENE_HAS_NORMALS = 1
SCENE_HAS_COLORS = 2
SCENE_HAS_UVS = 4


class RenderParams(C.Structure):
    """veil_render_params (64 bytes, reference veil.h:80-95)."""

    _fields_ = [
        ("flags", C.c_uint32),
        ("depth_filter_size", C.c_int),
        ("thread_count", C.c_int),
        ("background", C.c_float * 4),
        ("light_dir", C.c_float * 3),
        ("ambient", C.c_float),
        ("limit_low_tbr", C.c_uint32),
        ("limit_low_tri_blocks", C.c_uint32),
        ("limit_low_frags", C.c_uint32),
        ("limit_high_tbr", C.c_uint32),
        ("limit_high_thb", C.c_uint32),
    ]


assert C.sizeof(RenderParams) == 64


def default_params(**overrides):
    """veil_render_params_init (reference c_api.cpp:167-176) + overrides."""
    p = RenderParams()
    p.depth_filter_size = 3
    p.background[3] = 1.0
    p.light_dir[0], p.light_dir[1], p.light_dir[2] = 0.3, -0.5, 0.8
    p.ambient = 0.2
    for k, v in overrides.items():
        if k in ("background", "light_dir"):
            for i, x in enumerate(v):
                getattr(p, k)[i] = x
        else:
            setattr(p, k, v)
    return p


class SceneDesc(C.Structure):
    """veil_scene_desc (include/veil_cuda.h)."""

    _fields_ = [
        ("vertices", C.c_void_p),
        ("vertex_count", C.c_uint64),
        ("quads", C.c_void_p),
        ("quad_count", C.c_uint64),
        ("materials", C.c_void_p),
        ("material_count", C.c_uint32),
        ("flags", C.c_uint32),
        ("view_projection", C.c_double * 16),
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("has_eye", C.c_int32),
        ("reserved", C.c_int32),
        ("eye", C.c_double * 3),
    ]


class ImageDiff(C.Structure):
    _fields_ = [
        ("differing_pixels", C.c_uint64),
        ("max_channel_delta", C.c_int),
        ("width", C.c_int),
        ("height", C.c_int),
    ]


class IpcFramebuffer(C.Structure):
    """veil_ipc_framebuffer (include/veil_cuda.h): CUDA IPC handles of a
    device framebuffer (RGBA8 and invalid mask) plus its size."""

    _fields_ = [("rgba", C.c_uint8 * 64), ("mask", C.c_uint8 * 64),
                ("width", C.c_int32), ("height", C.c_int32)]


class Shard(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world_size", C.c_int32)]


class FrameStats(C.Structure):
    _fields_ = (
        [(n, C.c_double) for n in ("setup_ms", "binning_ms", "low_raster_ms", "hi_raster_ms", "total_ms")]
        + [
            (n, C.c_uint64)
            for n in (
                "samples", "fragments", "tri_half_blocks", "segments",
                "input_quads", "visible_quads",
                "culled_degenerate", "culled_backfacing", "culled_frustum", "culled_between_samples",
                "bins_empty", "bins_low", "bins_high", "bins_propagated",
                "invalid_pixels", "bin_pairs", "small_quads", "large_tris", "kernel_launches",
            )
        ]
        + [("shade_ms", C.c_double)]
    )


VERTEX_DTYPE = np.dtype(
    [("position", "<f4", 3), ("normal", "<f4", 3), ("color", "<f4", 4), ("uv", "<f4", 2)]
)
QUAD_DTYPE = np.dtype([("v", "<u4", 4), ("material", "<u4")])
MATERIAL_DTYPE = np.dtype(
    [("base_color", "<f4", 4), ("opacity", "<f4"), ("texture", "<i4"), ("flags", "<u4")]
)
assert VERTEX_DTYPE.itemsize == 48 and QUAD_DTYPE.itemsize == 20 and MATERIAL_DTYPE.itemsize == 28

# element dtypes of the parity dump arrays (veil_cuda.h, veil_render_dump_array)
DUMP_DTYPES = {
    "quad_source": np.uint32, "quad_aabb": np.uint64, "quad_class": np.uint8,
    "quad_attr": np.uint32, "tri_valid": np.uint8, "tri_yrange": np.int32,
    "tri_fn": np.float64, "tri_meta": np.uint32, "setup_stats": np.uint64,
    "bin_dims": np.int32, "bin_quad_counts": np.uint32, "bin_tri_counts": np.uint32,
    "bin_offsets": np.uint32, "bin_categories": np.uint8, "bin_items": np.uint32,
    "bin_path": np.uint8, "thb_offsets": np.uint64, "thb": np.uint64, "thb_tri": np.uint32,
    "thb_prefix": np.uint32, "emit_hash": np.uint64, "emit_hash_std": np.uint64, "emit_count": np.uint32,
    "image": np.uint8, "mask": np.uint8, "counters": np.uint64,
    "tbr_offsets": np.uint64, "tbr": np.uint64, "reenum_image": np.uint8, "reenum_mask": np.uint8,
}

COUNTER_NAMES = (
    "samples", "fragments", "tri_half_blocks", "segments",
    "bins_empty", "bins_low", "bins_high", "bins_propagated", "invalid_pixels",
)


class SceneArrays:
    """Host arrays of one scene (the veil_scene_desc payload) kept alive for ctypes."""

    def __init__(self, vertices, quads, materials, flags, matrix, width, height, eye=None):
        self.vertices = np.ascontiguousarray(vertices, dtype=VERTEX_DTYPE)
        self.quads = np.ascontiguousarray(quads, dtype=QUAD_DTYPE)
        self.materials = np.ascontiguousarray(materials, dtype=MATERIAL_DTYPE)
        self.flags = int(flags)
        self.matrix = np.asarray(matrix, dtype=np.float64).reshape(16).copy()
        self.width, self.height = int(width), int(height)
        self.eye = None if eye is None else np.asarray(eye, dtype=np.float64).reshape(3).copy()

    def desc(self):
        d = SceneDesc()
        d.vertices = self.vertices.ctypes.data
        d.vertex_count = len(self.vertices)
        d.quads = self.quads.ctypes.data
        d.quad_count = len(self.quads)
        d.materials = self.materials.ctypes.data
        d.material_count = len(self.materials)
        d.flags = self.flags
        for i in range(16):
            d.view_projection[i] = float(self.matrix[i])
        d.width, d.height = self.width, self.height
        if self.eye is not None:
            d.has_eye = 1
            for i in range(3):
                d.eye[i] = float(self.eye[i])
        return d

    @classmethod
    def from_desc(cls, d):
        """Copies a veil_scene_desc view into owned numpy arrays."""
        def view(ptr, n, dtype):
            if n == 0:
                return np.zeros(0, dtype=dtype)
            buf = (C.c_uint8 * (n * dtype.itemsize)).from_address(ptr)
            return np.frombuffer(buf, dtype=dtype).copy()

        return cls(
            view(d.vertices, d.vertex_count, VERTEX_DTYPE),
            view(d.quads, d.quad_count, QUAD_DTYPE),
            view(d.materials, d.material_count, MATERIAL_DTYPE),
            d.flags,
            np.array(list(d.view_projection)),
            d.width,
            d.height,
            np.array(list(d.eye)) if d.has_eye else None,
        )

    def with_camera(self, matrix, eye=None, width=None, height=None):
        s = SceneArrays(self.vertices, self.quads, self.materials, self.flags, matrix,
                        width or self.width, height or self.height, eye)
        return s
