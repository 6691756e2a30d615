"""ctypes bindings of the parity checkers. TEST INFRASTRUCTURE ONLY.

* ``liboracle.so``  -- the C restatement (oracle/veil_oracle.c)
* ``_ref/libveilref.so`` -- the unmodified reference + ref_shim.cpp

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module.
"""
import ctypes as C
import json
import os

import numpy as np

from paper_2405_13364_b200.abi import (
    DUMP_DTYPES,
    ImageDiff,
    RenderParams,
    SceneArrays,
    SceneDesc,
    default_params,
)

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libveilref.so")
# limits-lifted build (viewport 4096x4096, 16384 bins; `make -C oracle ref-lifted`)
REF_LIFTED_SO = os.path.join(HERE, "_ref", "libveilref_lifted.so")


class CheckerError(RuntimeError):
    def __init__(self, status, message):
        super().__init__(f"status {status}: {message}")
        self.status = status
        self.message = message


_oracle = None
_refs = {}


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            raise FileNotFoundError(f"{ORACLE_SO} missing: run `make -C oracle`")
        lib = C.CDLL(ORACLE_SO)
        lib.vo_render.argtypes = [C.POINTER(SceneDesc), C.POINTER(RenderParams), C.c_int,
                                  C.POINTER(C.c_void_p)]
        lib.vo_render.restype = C.c_int
        lib.vo_array.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_uint64)]
        lib.vo_array.restype = C.c_void_p
        lib.vo_message.argtypes = [C.c_void_p]
        lib.vo_message.restype = C.c_char_p
        lib.vo_free.argtypes = [C.c_void_p]
        _oracle = lib
    return _oracle


def ref_available(lifted=False):
    return os.path.exists(REF_LIFTED_SO if lifted else REF_SO)


def ref_lib(lifted=False):
    if lifted not in _refs:
        lib = C.CDLL(REF_LIFTED_SO if lifted else REF_SO)
        lib.vref_scene_create.argtypes = [C.POINTER(SceneDesc), C.POINTER(C.c_void_p)]
        lib.vref_scene_create.restype = C.c_int
        lib.vref_scene_describe.argtypes = [C.c_void_p, C.POINTER(SceneDesc)]
        lib.vref_scene_describe.restype = C.c_int
        lib.vref_scene_forget.argtypes = [C.c_void_p]
        lib.vref_dump_run.argtypes = [C.c_void_p, C.POINTER(RenderParams), C.POINTER(C.c_void_p)]
        lib.vref_dump_run.restype = C.c_int
        lib.vref_dump_array.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_uint64)]
        lib.vref_dump_array.restype = C.c_void_p
        lib.vref_dump_destroy.argtypes = [C.c_void_p]
        lib.vref_last_error.restype = C.c_char_p
        # the reference's own C API (reference veil.h)
        lib.veil_last_error.restype = C.c_char_p
        lib.veil_scene_load.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]
        lib.veil_scene_synthetic.argtypes = [C.c_char_p, C.c_uint64, C.c_int, C.c_int,
                                             C.POINTER(C.c_void_p)]
        lib.veil_scene_set_viewport.argtypes = [C.c_void_p, C.c_int, C.c_int]
        lib.veil_scene_set_camera.argtypes = [C.c_void_p, C.POINTER(C.c_double),
                                              C.POINTER(C.c_double)]
        lib.veil_scene_destroy.argtypes = [C.c_void_p]
        lib.veil_render_scene.argtypes = [C.c_void_p, C.POINTER(RenderParams), C.POINTER(C.c_void_p)]
        lib.veil_render_pixels.argtypes = [C.c_void_p]
        lib.veil_render_pixels.restype = C.POINTER(C.c_uint8)
        lib.veil_render_invalid_mask.argtypes = [C.c_void_p]
        lib.veil_render_invalid_mask.restype = C.POINTER(C.c_uint8)
        lib.veil_render_report_json.argtypes = [C.c_void_p]
        lib.veil_render_report_json.restype = C.c_char_p
        lib.veil_render_width.argtypes = [C.c_void_p]
        lib.veil_render_height.argtypes = [C.c_void_p]
        lib.veil_render_destroy.argtypes = [C.c_void_p]
        lib.veil_scene_group_quads.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
        _refs[lifted] = lib
    return _refs[lifted]


def _collect(getter, handle, names=None):
    out = {}
    for name, dt in DUMP_DTYPES.items():
        if names is not None and name not in names:
            continue
        n = C.c_uint64(0)
        ptr = getter(handle, name.encode(), C.byref(n))
        if not ptr:
            continue
        dt = np.dtype(dt)
        if n.value == 0:
            out[name] = np.zeros(0, dtype=dt)
            continue
        buf = (C.c_uint8 * (n.value * dt.itemsize)).from_address(ptr)
        out[name] = np.frombuffer(buf, dtype=dt).copy()
    return out


def oracle_render(scene: SceneArrays, params=None, extended=False, names=None):
    """Runs the C restatement; returns {name: ndarray}. Raises CheckerError."""
    lib = oracle_lib()
    params = params or default_params()
    desc = scene.desc()
    h = C.c_void_p()
    st = lib.vo_render(C.byref(desc), C.byref(params), int(bool(extended)), C.byref(h))
    try:
        if st != 0:
            raise CheckerError(st, lib.vo_message(h).decode())
        return _collect(lib.vo_array, h, names)
    finally:
        lib.vo_free(h)


class RefScene:
    """A scene inside the reference library."""

    def __init__(self, handle, lifted=False):
        self.h = C.c_void_p(handle)
        self.lib = ref_lib(lifted)

    def __del__(self):
        if getattr(self, "h", None) and getattr(self, "lib", None) is not None:
            self.lib.vref_scene_forget(self.h)
            self.lib.veil_scene_destroy(self.h)
            self.h = None

    @classmethod
    def from_arrays(cls, scene: SceneArrays, lifted=False):
        lib = ref_lib(lifted)
        desc = scene.desc()
        h = C.c_void_p()
        st = lib.vref_scene_create(C.byref(desc), C.byref(h))
        if st != 0:
            raise CheckerError(st, lib.vref_last_error().decode())
        return cls(h.value, lifted)

    @classmethod
    def load(cls, mesh, mtl=None, cam=None):
        lib = ref_lib()
        h = C.c_void_p()
        st = lib.veil_scene_load(mesh.encode(), mtl.encode() if mtl else None,
                                 cam.encode() if cam else None, C.byref(h))
        if st != 0:
            raise CheckerError(st, lib.veil_last_error().decode())
        return cls(h.value)

    @classmethod
    def synthetic(cls, kind, seed, width=0, height=0):
        lib = ref_lib()
        h = C.c_void_p()
        st = lib.veil_scene_synthetic(kind.encode(), seed, width, height, C.byref(h))
        if st != 0:
            raise CheckerError(st, lib.veil_last_error().decode())
        return cls(h.value)

    @classmethod
    def synthetic_params(cls, kind, seed, width, height, layers=0, triangles=0, sheets=0):
        """generate_synthetic_scene with SyntheticParams (acceptance.cpp:80-101)."""
        lib = ref_lib()
        lib.vref_scene_synthetic_params.argtypes = [C.c_char_p, C.c_uint64, C.c_int, C.c_int, C.c_int,
                                                    C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        h = C.c_void_p()
        st = lib.vref_scene_synthetic_params(kind.encode(), seed, width, height, layers, triangles,
                                             sheets, C.byref(h))
        if st != 0:
            raise CheckerError(st, lib.vref_last_error().decode())
        return cls(h.value)

    def measure_disorder(self, params=None):
        """RenderConfig::measure_disorder of the reference pipeline."""
        self.lib.vref_measure_disorder.argtypes = [C.c_void_p, C.POINTER(RenderParams), C.POINTER(C.c_int)]
        out = C.c_int(0)
        st = self.lib.vref_measure_disorder(self.h, C.byref(params or default_params()), C.byref(out))
        if st != 0:
            raise CheckerError(st, self.lib.vref_last_error().decode())
        return out.value

    def set_viewport(self, w, h):
        st = self.lib.veil_scene_set_viewport(self.h, w, h)
        if st != 0:
            raise CheckerError(st, self.lib.veil_last_error().decode())

    def set_camera(self, matrix, eye=None):
        m = (C.c_double * 16)(*[float(x) for x in np.asarray(matrix).reshape(16)])
        e = None if eye is None else (C.c_double * 3)(*[float(x) for x in eye])
        st = self.lib.veil_scene_set_camera(self.h, m, e)
        if st != 0:
            raise CheckerError(st, self.lib.veil_last_error().decode())

    def group_quads(self):
        d = C.c_double(0)
        st = self.lib.veil_scene_group_quads(self.h, C.byref(d))
        if st != 0:
            raise CheckerError(st, self.lib.veil_last_error().decode())
        return d.value

    def arrays(self) -> SceneArrays:
        d = SceneDesc()
        self.lib.vref_scene_describe(self.h, C.byref(d))
        return SceneArrays.from_desc(d)

    def dump(self, params=None, names=None):
        lib = self.lib
        params = params or default_params()
        h = C.c_void_p()
        st = lib.vref_dump_run(self.h, C.byref(params), C.byref(h))
        try:
            if st != 0:
                raise CheckerError(st, lib.vref_last_error().decode())
            return _collect(lib.vref_dump_array, h, names)
        finally:
            if h:
                lib.vref_dump_destroy(h)

    def render(self, params=None):
        """The reference's own C API render (veil_render_scene)."""
        lib = self.lib
        params = params or default_params()
        r = C.c_void_p()
        st = lib.veil_render_scene(self.h, C.byref(params), C.byref(r))
        if st != 0:
            raise CheckerError(st, lib.veil_last_error().decode())
        try:
            w, hh = lib.veil_render_width(r), lib.veil_render_height(r)
            img = np.ctypeslib.as_array(lib.veil_render_pixels(r), shape=(hh * w * 4,)).copy()
            mask = np.ctypeslib.as_array(lib.veil_render_invalid_mask(r), shape=(hh * w,)).copy()
            report = json.loads(lib.veil_render_report_json(r).decode())
            return img.reshape(hh, w, 4), mask.reshape(hh, w), report
        finally:
            lib.veil_render_destroy(r)


def ref_look_at(frm, at, up, fov_deg, near, far, width, height, lifted=False):
    """The reference's make_look_at_camera (scene.cpp:128-158) -> row-major 4x4."""
    lib = ref_lib(lifted)
    arr = lambda v: (C.c_double * 3)(*[float(x) for x in v])
    out = (C.c_double * 16)()
    lib.vref_look_at.restype = C.c_int
    lib.vref_look_at.argtypes = [C.c_double * 3] * 3 + [C.c_double] * 3 + [C.c_int] * 2 + [C.c_double * 16]
    st = lib.vref_look_at(arr(frm), arr(at), arr(up), fov_deg, near, far, width, height, out)
    if st != 0:
        raise CheckerError(st, lib.vref_last_error().decode())
    return np.array(list(out))


def ref_dump_arrays(scene: SceneArrays, params=None, names=None, lifted=False):
    return RefScene.from_arrays(scene, lifted).dump(params, names)
