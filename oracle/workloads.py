"""numpy generators of the BASELINE.json workloads. TEST / BASELINE INFRASTRUCTURE.

The reference arm of bench.py (and the CPU baseline leg) must build its input
arrays without mapping libveil.so, so the workload recipes of SURVEY.md 8(d)
are restated here in numpy: std::mt19937_64 (C++ [rand.eng.mers], the
engine the reference's synthetic scenes use, synthetic.cpp:29-43) is
vectorised one 312-word twist at a time, and the draws are consumed in the
strictly sequenced order libveil's workload_scene uses
(paper_2405_13364_b200/csrc/scene_io.cpp, stacked_quads / grid_mesh).
tests/test_workloads_cpu.py checks the arrays equal veil.Scene.workload's
byte for byte.
"""
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
)

_N, _M = 312, 156
_MATRIX_A = np.uint64(0xB5026F5AA96619E9)
_UPPER = np.uint64(0xFFFFFFFF80000000)
_LOWER = np.uint64(0x7FFFFFFF)
_M64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 with bulk output (identical sequence)."""

    def __init__(self, seed):
        mt = [seed & _M64]
        for i in range(1, _N):
            prev = mt[-1]
            mt.append((6364136223846793005 * (prev ^ (prev >> 62)) + i) & _M64)
        self.mt = np.array(mt, dtype=np.uint64)
        self.buf = np.zeros(0, dtype=np.uint64)

    def _twist(self):
        mt = self.mt
        one = np.uint64(1)

        def mix(hi, lo, far):
            x = (hi & _UPPER) | (lo & _LOWER)
            xa = x >> one
            xa ^= np.where((x & one) != 0, _MATRIX_A, np.uint64(0))
            return far ^ xa

        new = mt.copy()
        # i in [0, 156): far = old mt[i + 156], next = old mt[i + 1]
        new[0:156] = mix(mt[0:156], mt[1:157], mt[156:312])
        # i in [156, 311): far = new mt[i - 156], next = old mt[i + 1]
        new[156:311] = mix(mt[156:311], mt[157:312], new[0:155])
        # i = 311: next = new mt[0], far = new mt[155]
        new[311:312] = mix(mt[311:312], new[0:1], new[155:156])
        self.mt = new
        y = new.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        return y

    def draws(self, n):
        """The next n outputs of the engine."""
        parts = [self.buf]
        have = len(self.buf)
        while have < n:
            blk = self._twist()
            parts.append(blk)
            have += len(blk)
        allv = np.concatenate(parts)
        self.buf = allv[n:]
        return allv[:n]


def _unit(d):
    """(e() >> 11) * 2^-53, synthetic.cpp:34-37."""
    return (d >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def _uniform(d, lo, hi):
    return lo + (hi - lo) * _unit(d)


def _channel(d):
    """float(e() % 216 + 40) / 255.0f (colours on the 8-bit grid)."""
    return (d % np.uint64(216) + np.uint64(40)).astype(np.float32) / np.float32(255.0)


def _material():
    m = np.zeros(1, dtype=MATERIAL_DTYPE)
    m[0] = ((1.0, 1.0, 1.0, 1.0), 1.0, -1, MATERIAL_VERTEX_COLORS | MATERIAL_VERTEX_NORMALS)
    return m


def _vertices(n):
    v = np.zeros(n, dtype=VERTEX_DTYPE)
    v["normal"][:, 2] = -1.0
    return v


def stacked_quads(e, count, lo, hi, w, h):
    """Axis-aligned translucent quads, 9 draws each in this order: hx_px, hy_px,
    cx, cy, z, r, g, b, a (SURVEY.md 8(d) C2 recipe)."""
    d = e.draws(9 * count).reshape(count, 9)
    hx_px, hy_px = _uniform(d[:, 0], lo, hi), _uniform(d[:, 1], lo, hi)
    cx, cy = _uniform(d[:, 2], -1.0, 1.0), _uniform(d[:, 3], -1.0, 1.0)
    z = _uniform(d[:, 4], 0.05, 0.95)
    col = np.stack([_channel(d[:, 5]), _channel(d[:, 6]), _channel(d[:, 7]),
                    (d[:, 8] % np.uint64(151) + np.uint64(64)).astype(np.float32) / np.float32(255.0)],
                   axis=1)
    hx, hy = hx_px * 2.0 / w, hy_px * 2.0 / h
    xs = np.stack([cx - hx, cx + hx, cx + hx, cx - hx], axis=1)
    ys = np.stack([cy - hy, cy - hy, cy + hy, cy + hy], axis=1)
    v = _vertices(4 * count)
    v["position"][:, 0] = xs.reshape(-1).astype(np.float32)
    v["position"][:, 1] = ys.reshape(-1).astype(np.float32)
    v["position"][:, 2] = np.repeat(z, 4).astype(np.float32)
    v["color"] = np.repeat(col, 4, axis=0)
    return v


def grid_mesh(e, nx, ny):
    """Jittered grid over NDC [-1,1]^2: per vertex (row-major) two jitter draws
    when interior, then z, then r, g, b."""
    cw, ch = 2.0 / nx, 2.0 / ny
    jj, ii = np.meshgrid(np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    jj, ii = jj.reshape(-1), ii.reshape(-1)
    interior = (ii > 0) & (ii < nx) & (jj > 0) & (jj < ny)
    per = np.where(interior, 6, 4).astype(np.int64)
    start = np.concatenate([[0], np.cumsum(per)[:-1]])
    d = e.draws(int(per.sum()))
    x = -1.0 + cw * ii
    y = -1.0 + ch * jj
    k = start[interior]
    x[interior] += _uniform(d[k], -0.25, 0.25) * cw
    y[interior] += _uniform(d[k + 1], -0.25, 0.25) * ch
    zoff = start + np.where(interior, 2, 0)
    z = _uniform(d[zoff], 0.2, 0.8)
    v = _vertices(len(x))
    v["position"][:, 0] = x.astype(np.float32)
    v["position"][:, 1] = y.astype(np.float32)
    v["position"][:, 2] = z.astype(np.float32)
    v["color"][:, 0] = _channel(d[zoff + 1])
    v["color"][:, 1] = _channel(d[zoff + 2])
    v["color"][:, 2] = _channel(d[zoff + 3])
    v["color"][:, 3] = np.float32(128.0) / np.float32(255.0)
    jq, iq = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    v00 = (jq * (nx + 1) + iq).reshape(-1).astype(np.uint32)
    q = np.zeros(nx * ny, dtype=QUAD_DTYPE)
    q["v"] = np.stack([v00, v00 + 1, v00 + 1 + (nx + 1), v00 + (nx + 1)], axis=1)
    return v, q


def workload(name, seed, width=0, height=0):
    """SceneArrays of a BASELINE workload; same arrays as veil.Scene.workload."""
    e = MT19937_64(seed)
    flags = SCENE_HAS_COLORS | SCENE_HAS_NORMALS
    eye4 = np.eye(4).reshape(16)
    if name == "stack64k":
        w, h = width or 1920, height or 1080
        v = stacked_quads(e, 65536, 12.0, 20.0, w, h)
        q = np.zeros(65536, dtype=QUAD_DTYPE)
        q["v"] = np.arange(4 * 65536, dtype=np.uint32).reshape(-1, 4)
        return SceneArrays(v, q, _material(), flags, eye4, w, h)
    if name in ("tiny4m", "mixed16m"):
        w, h = (width or 3840, height or 2160) if name == "tiny4m" else (width or 7680, height or 4320)
        nx, ny = (2048, 2048) if name == "tiny4m" else (4096, 3840)
        v, q = grid_mesh(e, nx, ny)
        if name == "mixed16m":
            n = 1048576
            vs = stacked_quads(e, n, 4.0, 12.0, w, h)
            qs = np.zeros(n, dtype=QUAD_DTYPE)
            qs["v"] = len(v) + np.arange(4 * n, dtype=np.uint32).reshape(-1, 4)
            v, q = np.concatenate([v, vs]), np.concatenate([q, qs])
        return SceneArrays(v, q, _material(), flags, eye4, w, h)
    raise ValueError(f"unknown workload {name}")


def grid_scene(seed, nx, ny, width, height):
    """The tiny4m recipe (grid_mesh) at another grid size / viewport."""
    e = MT19937_64(seed)
    v, q = grid_mesh(e, nx, ny)
    return SceneArrays(v, q, _material(), SCENE_HAS_COLORS | SCENE_HAS_NORMALS, np.eye(4).reshape(16),
                       width, height)
