"""Python binding of libveil.so (the B200 renderer) through its C ABI.

Mirrors the reference's C interface (reference veil.h:43-124) one call per
function, with the same status semantics: a non-OK status raises VeilError
carrying the status code and veil_last_error(). There is no Python or CPU
rendering path here: if libveil.so is missing or no CUDA device is present,
rendering fails loudly.
"""
import ctypes as C
import json
import os

import numpy as np

from .abi import (
    DUMP_DTYPES,
    FrameStats,
    ImageDiff,
    IpcFramebuffer,
    RenderParams,
    SceneArrays,
    SceneDesc,
    Shard,
    default_params,
)

HERE = os.path.dirname(os.path.abspath(__file__))
# VEIL_LIB selects another build of the library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("VEIL_LIB") or os.path.join(HERE, "libveil.so")

STATUS_NAMES = {0: "VEIL_OK", 1: "VEIL_ERR_IO", 2: "VEIL_ERR_PARSE", 3: "VEIL_ERR_INVALID_ARG",
                4: "VEIL_ERR_CAPACITY", 5: "VEIL_ERR_INTERNAL"}


class VeilError(RuntimeError):
    def __init__(self, status, message):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status
        self.message = message


_lib = None

_P = C.c_void_p
_PP = C.POINTER(C.c_void_p)


def lib():
    """Loads libveil.so (build it with __graft_entry__.build() / make)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FileNotFoundError(
            f"{LIB_PATH} is missing: the CUDA extension must be built "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no fallback")
    L = C.CDLL(LIB_PATH)
    sig = {
        "veil_status_string": ([C.c_int], C.c_char_p),
        "veil_last_error": ([], C.c_char_p),
        "veil_scene_load": ([C.c_char_p, C.c_char_p, C.c_char_p, _PP], C.c_int),
        "veil_scene_synthetic": ([C.c_char_p, C.c_uint64, C.c_int, C.c_int, _PP], C.c_int),
        "veil_scene_group_quads": ([_P, C.POINTER(C.c_double)], C.c_int),
        "veil_scene_set_viewport": ([_P, C.c_int, C.c_int], C.c_int),
        "veil_scene_set_camera": ([_P, C.POINTER(C.c_double), C.POINTER(C.c_double)], C.c_int),
        "veil_scene_destroy": ([_P], None),
        "veil_render_params_init": ([C.POINTER(RenderParams)], None),
        "veil_render_scene": ([_P, C.POINTER(RenderParams), _PP], C.c_int),
        "veil_render_width": ([_P], C.c_int),
        "veil_render_height": ([_P], C.c_int),
        "veil_render_pixels": ([_P], C.POINTER(C.c_uint8)),
        "veil_render_invalid_mask": ([_P], C.POINTER(C.c_uint8)),
        "veil_render_report_json": ([_P], C.c_char_p),
        "veil_render_write_png": ([_P, C.c_char_p], C.c_int),
        "veil_render_destroy": ([_P], None),
        "veil_compare_png": ([C.c_char_p, C.c_char_p, C.POINTER(ImageDiff)], C.c_int),
        # veil_cuda.h
        "veil_scene_create": ([C.POINTER(SceneDesc), _PP], C.c_int),
        "veil_scene_describe": ([_P, C.POINTER(SceneDesc)], C.c_int),
        "veil_scene_workload": ([C.c_char_p, C.c_uint64, C.c_int, C.c_int, _PP], C.c_int),
        "veil_camera_look_at": ([C.POINTER(C.c_double)] * 3 + [C.c_double] * 3
                                + [C.c_int, C.c_int, C.POINTER(C.c_double)], C.c_int),
        "veil_scene_set_extended_limits": ([_P, C.c_int], C.c_int),
        "veil_scene_set_viewport_ext": ([_P, C.c_int, C.c_int], C.c_int),
        "veil_cuda_set_device": ([C.c_int], C.c_int),
        "veil_render_scene_shard": ([_P, C.POINTER(RenderParams), C.POINTER(Shard), _PP], C.c_int),
        "veil_render_scene_multi": ([_P, C.POINTER(RenderParams), C.POINTER(C.c_int), C.c_int, _PP], C.c_int),
        "veil_measure_disorder": ([_P, C.POINTER(RenderParams), C.POINTER(C.c_int)], C.c_int),
        "veil_shard_tile_count": ([C.c_int, C.c_int, C.POINTER(Shard)], C.c_uint64),
        "veil_shard_pack_tiles": ([_P, C.POINTER(Shard), _P, C.c_uint64], C.c_int),
        "veil_shard_unpack_tiles": ([_P, C.POINTER(Shard), _P, C.c_uint64], C.c_int),
        "veil_shard_pack_tiles_device": ([_P, C.POINTER(Shard), _P, C.c_uint64], C.c_int),
        "veil_shard_unpack_tiles_device": ([_P, C.POINTER(Shard), _P, C.c_uint64], C.c_int),
        "veil_render_device": ([_P, C.POINTER(RenderParams), C.POINTER(Shard)], C.c_int),
        "veil_render_device_timed": ([_P, C.POINTER(RenderParams), C.POINTER(Shard), _P, _P], C.c_int),
        "veil_device_framebuffer": ([_P, _PP, _PP], C.c_int),
        "veil_export_framebuffer": ([_P, C.POINTER(IpcFramebuffer)], C.c_int),
        "veil_import_peer_framebuffer": ([_P, C.POINTER(IpcFramebuffer)], C.c_int),
        "veil_scene_stream": ([_P], C.c_void_p),
        "veil_render_stats": ([_P, C.POINTER(FrameStats)], C.c_int),
        "veil_scene_last_stats": ([_P, C.POINTER(FrameStats)], C.c_int),
        "veil_render_scene_dump": ([_P, C.POINTER(RenderParams), _PP], C.c_int),
        "veil_render_dump_array": ([_P, C.c_char_p, C.POINTER(C.c_uint64)], C.c_void_p),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def _check(status):
    if status != 0:
        raise VeilError(status, lib().veil_last_error().decode())


def exported_symbols():
    """Names declared in include/veil.h and include/veil_cuda.h."""
    import re

    names = []
    inc = os.path.join(os.path.dirname(HERE), "include")
    for h in ("veil.h", "veil_cuda.h"):
        src = open(os.path.join(inc, h)).read()
        names += re.findall(r"^\s*(?:const\s+)?[\w\s\*]*?\b(veil_\w+)\s*\(", src, re.M)
    return sorted(set(names))


class Scene:
    """A veil_scene handle."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle)

    def __del__(self):
        self.close()

    def close(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.veil_scene_destroy(self.h)
        self.h = None

    @classmethod
    def load(cls, mesh, mtl=None, cam=None):
        h = C.c_void_p()
        _check(lib().veil_scene_load(mesh.encode(), mtl.encode() if mtl else None,
                                     cam.encode() if cam else None, C.byref(h)))
        return cls(h.value)

    @classmethod
    def synthetic(cls, kind, seed=1, width=0, height=0):
        h = C.c_void_p()
        _check(lib().veil_scene_synthetic(kind.encode(), seed, width, height, C.byref(h)))
        return cls(h.value)

    @classmethod
    def workload(cls, name, seed, width=0, height=0):
        h = C.c_void_p()
        _check(lib().veil_scene_workload(name.encode(), seed, width, height, C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_arrays(cls, arrays: SceneArrays):
        d = arrays.desc()
        h = C.c_void_p()
        _check(lib().veil_scene_create(C.byref(d), C.byref(h)))
        return cls(h.value)

    def arrays(self) -> SceneArrays:
        d = SceneDesc()
        _check(lib().veil_scene_describe(self.h, C.byref(d)))
        return SceneArrays.from_desc(d)

    def set_viewport(self, w, h):
        _check(lib().veil_scene_set_viewport(self.h, w, h))

    def set_viewport_ext(self, w, h):
        _check(lib().veil_scene_set_viewport_ext(self.h, w, h))

    def set_extended_limits(self, on=True):
        _check(lib().veil_scene_set_extended_limits(self.h, int(bool(on))))

    def set_camera(self, matrix, eye=None):
        m = (C.c_double * 16)(*[float(x) for x in np.asarray(matrix).reshape(16)])
        e = None if eye is None else (C.c_double * 3)(*[float(x) for x in eye])
        _check(lib().veil_scene_set_camera(self.h, m, e))

    def group_quads(self):
        d = C.c_double(0)
        _check(lib().veil_scene_group_quads(self.h, C.byref(d)))
        return d.value

    def stream(self):
        return lib().veil_scene_stream(self.h)

    def last_stats(self):
        s = FrameStats()
        _check(lib().veil_scene_last_stats(self.h, C.byref(s)))
        return s

    def device_framebuffer(self):
        a, b = C.c_void_p(), C.c_void_p()
        _check(lib().veil_device_framebuffer(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value


def look_at(frm, at, up, fov_deg, near, far, width, height):
    """make_look_at_camera (reference scene.cpp:128-158) -> row-major 4x4."""
    out = (C.c_double * 16)()
    arr = lambda v: (C.c_double * 3)(*[float(x) for x in v])
    _check(lib().veil_camera_look_at(arr(frm), arr(at), arr(up), fov_deg, near, far,
                                     width, height, out))
    return np.array(list(out))


class Render:
    """A veil_render handle: framebuffer, invalid mask, report."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.veil_render_destroy(self.h)
        self.h = None

    @property
    def width(self):
        return lib().veil_render_width(self.h)

    @property
    def height(self):
        return lib().veil_render_height(self.h)

    def pixels(self, copy=True):
        """RGBA8 (H, W, 4). copy=False returns a view valid while this handle lives."""
        w, h = self.width, self.height
        p = lib().veil_render_pixels(self.h)
        a = np.ctypeslib.as_array(p, shape=(h * w * 4,)).reshape(h, w, 4)
        return a.copy() if copy else a

    def invalid_mask(self, copy=True):
        w, h = self.width, self.height
        p = lib().veil_render_invalid_mask(self.h)
        a = np.ctypeslib.as_array(p, shape=(h * w,)).reshape(h, w)
        return a.copy() if copy else a

    def report(self):
        return json.loads(lib().veil_render_report_json(self.h).decode())

    def stats(self):
        s = FrameStats()
        _check(lib().veil_render_stats(self.h, C.byref(s)))
        return s

    def write_png(self, path):
        _check(lib().veil_render_write_png(self.h, path.encode()))

    def dumps(self, names=None):
        out = {}
        for name, dt in DUMP_DTYPES.items():
            if names is not None and name not in names:
                continue
            n = C.c_uint64(0)
            ptr = lib().veil_render_dump_array(self.h, name.encode(), C.byref(n))
            if not ptr:
                continue
            dt = np.dtype(dt)
            if n.value == 0:
                out[name] = np.zeros(0, dtype=dt)
                continue
            buf = (C.c_uint8 * (n.value * dt.itemsize)).from_address(ptr)
            out[name] = np.frombuffer(buf, dtype=dt).copy()
        return out


def render(scene: Scene, params=None, shard=None) -> Render:
    params = params or default_params()
    r = C.c_void_p()
    if shard is None:
        _check(lib().veil_render_scene(scene.h, C.byref(params), C.byref(r)))
    else:
        sh = Shard(*shard)
        _check(lib().veil_render_scene_shard(scene.h, C.byref(params), C.byref(sh), C.byref(r)))
    return Render(r.value)


def render_multi(scene: Scene, devices, params=None) -> Render:
    """veil_render_scene_multi: one frame over several devices in this process
    (bins interleaved over len(devices) shards, peer-memory gather)."""
    params = params or default_params()
    devs = (C.c_int * len(devices))(*[int(x) for x in devices])
    r = C.c_void_p()
    _check(lib().veil_render_scene_multi(scene.h, C.byref(params), devs, len(devices), C.byref(r)))
    return Render(r.value)


def measure_disorder(scene: Scene, params=None) -> int:
    """veil_measure_disorder: the pipeline's maximum per-pixel sort disorder."""
    params = params or default_params()
    out = C.c_int(0)
    _check(lib().veil_measure_disorder(scene.h, C.byref(params), C.byref(out)))
    return out.value


def render_dump(scene: Scene, params=None, names=None):
    """Renders with parity capture; returns {name: ndarray} (veil_cuda.h)."""
    params = params or default_params()
    r = C.c_void_p()
    _check(lib().veil_render_scene_dump(scene.h, C.byref(params), C.byref(r)))
    return Render(r.value).dumps(names)


def render_device(scene: Scene, params=None, shard=None, stats=True, events=None):
    """One frame into device memory only (bench path); returns FrameStats
    (or None with stats=False, so a caller can close its timed region first
    and read scene.last_stats() afterwards). events = (start, end) raw
    cudaEvent_t handles (int or None) the library records on the scene's
    stream right before and after the frame's device work."""
    params = params or default_params()
    sh = None if shard is None else C.byref(Shard(*shard))
    if events is None:
        _check(lib().veil_render_device(scene.h, C.byref(params), sh))
    else:
        _check(lib().veil_render_device_timed(scene.h, C.byref(params), sh, events[0], events[1]))
    return scene.last_stats() if stats else None


def export_framebuffer(scene: Scene) -> bytes:
    """The scene's device framebuffer as CUDA IPC handles (root rank)."""
    fb = IpcFramebuffer()
    _check(lib().veil_export_framebuffer(scene.h, C.byref(fb)))
    return bytes(fb)


def import_peer_framebuffer(scene: Scene, blob):
    """Write this rank's sharded frames into the root's framebuffer too
    (blob from export_framebuffer on the root; None detaches)."""
    if blob is None:
        _check(lib().veil_import_peer_framebuffer(scene.h, None))
        return
    fb = IpcFramebuffer.from_buffer_copy(blob)
    _check(lib().veil_import_peer_framebuffer(scene.h, C.byref(fb)))


def pack_tiles_device(scene: Scene, rank, world, dev_ptr, nbytes):
    sh = Shard(rank, world)
    _check(lib().veil_shard_pack_tiles_device(scene.h, C.byref(sh), C.c_void_p(dev_ptr), nbytes))


def unpack_tiles_device(scene: Scene, rank, world, dev_ptr, nbytes):
    sh = Shard(rank, world)
    _check(lib().veil_shard_unpack_tiles_device(scene.h, C.byref(sh), C.c_void_p(dev_ptr), nbytes))


def compare_png(a, b):
    d = ImageDiff()
    _check(lib().veil_compare_png(a.encode(), b.encode(), C.byref(d)))
    return d


def set_device(dev):
    _check(lib().veil_cuda_set_device(int(dev)))


def shard_tile_count(bins_x, bins_y, rank, world):
    sh = Shard(rank, world)
    return int(lib().veil_shard_tile_count(bins_x, bins_y, C.byref(sh)))
