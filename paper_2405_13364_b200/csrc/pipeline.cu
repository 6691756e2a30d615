// libveil device pipeline: sort-middle exact-OIT frame render on sm_100a.
//
// Stage map (reference -> kernel):
//   setup phase 1 + compaction   setup.cpp:255-302    k_setup (single pass, decoupled look-back)
//   setup phase 2 (records)      setup.cpp:305-349    k_setup_tris
//   binning count / offsets      binning.cpp:124-145  k_bin_pass<false>, k_bin_large<false>, k_bin_scan
//   binning write                binning.cpp:147-186  k_bin_pass<true>, k_bin_large<true>
//                                                     (+ k_bin_sort for parity dumps)
//   tri-block rows / THB lists   raster.cpp:41-199    k_extract<kGlobal> (low pass, high pass)
//   shading, filter, blend       raster.cpp:201-321   k_order_bins, k_shade<KM, mode, kTex>
//   stats merge                  renderer.cpp:170-212 k_finalize
//
// Design notes (DESIGN.md has the full version):
//  * One frame is one CUDA graph replay; frame constants live in __constant__
//    memory written by the graph's first node from pinned staging.
//  * Per-bin lists are filled with warp-aggregated atomics in any order: the
//    extraction orders tri-blocks by (quantized centroid depth, is_large,
//    triangle), the same order as the reference's (depth, selection index)
//    because the selection index is monotone in (is_large, triangle).
//  * k_extract is a persistent kernel over (bin, block-row) items: a CTA of 4
//    warps builds the block-row's tri-block-rows in shared memory, then warp
//    w sorts block w's tri-blocks and splits them into tri-half-blocks (THB
//    pool). It also decides, per half-block, wave walk (k_shade mode 0:
//    lane = pixel, disjoint consecutive THBs per step) or dense segments
//    (mode 1: lane = sample, warp routing) and queues the latter.
//  * Items over the shared-memory capacities but within the rasterizer
//    limits are re-run by the same kernel with global scratch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <exception>
#include <thread>
#include <vector>

#include "device_math.cuh"
#include "veil_internal.hpp"

namespace veil {

// ============================================================ device side
namespace dev {

// Device-side invariant checks of the bounds-checked build (make CHECKS=1 ->
// build_checked/libveil.so, run by tests/test_checked_build_gpu.py; the
// pool's compute-sanitizer is unavailable): a violated index bound traps the
// kernel, which fails the frame. Compiled out of the product build.
#ifdef VEIL_DEVICE_CHECKS
#define VEIL_CHECK(cond) \
  do {                   \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define VEIL_CHECK(cond) \
  do {                   \
  } while (0)
#endif

constexpr int kSetupBlock = 256;
constexpr uint64_t kHashSeed = 0xcbf29ce484222325ull;
constexpr uint64_t kHashPrime = 0x100000001b3ull;
constexpr float kAlphaThreshold = 1.0f - 1.0f / 128.0f;  // raster.hpp:51

struct Limits {
  uint32_t tbr, tb, thb, frags;
};

struct MatDev {
  float base[4];
  float opacity;
  uint32_t flags;  // bit0 colors, bit1 normals, bit2 uvs (AND-ed with the scene flags)
  int32_t texture;  // -1: none
  uint32_t pad;
};

struct FrameConst {
  double m[16];
  double eye[3];
  double fwd[3];
  int has_eye;
  int width, height, bins_x, bins_y, nbins;
  int backface, extended;
  uint32_t nquads;
  float light[3];
  float ambient;
  float bg[4];  // premultiplied background
  int df;
  int threshold, visualize, force_high;
  Limits low, high;
  uint32_t items_cap;
  uint32_t tri_cap;  // visible-triangle capacity (2^24 standard)
  int rank, world;
  int dump;
  int decoded;  // setup writes per-triangle decoded shading records
  uint32_t pool_cap;
  uint32_t lpairs_cap;
  int sort_bins;  // host-side: canonical bin-list order (k_bin_sort) this frame
  int walk_min;   // experiment override of kWalkMinSamplesPerThb (VEIL_WALK_MIN), 0 = default
  int walk_min_u; // the same for bins whose triangles are not staged (VEIL_WALK_MIN_U)
  int wave1;      // experiment: one wave per step in the staged wave walk (VEIL_WAVE1=1)
  // Fused raster for tiny-triangle frames (not decoded): k_extract recomputes
  // small quads' triangle setups from the positions instead of reading 128-B
  // records, and shades its half-blocks right after extracting them (no
  // k_shade); write_tri: k_setup_tris still stores every record (parity dumps,
  // the non-fused path; large quads' records are always stored, k_bin_large
  // reads them).
  int fused;
  int write_tri;
  int fused_read;  // experiment: the fused raster reads stored records (VEIL_FUSED_READ=1)
  int bulk_stage;  // k_shade stages THB lists with cp.async.bulk (VEIL_BULK_STAGE=0/1)
  int fill_split;  // empty bins painted by k_fill_empty, not k_shade (VEIL_FILL_SPLIT=0/1)
  // zero-copy readback: the frame's pinned host RGBA8 / mask (device-mapped),
  // written by the shading kernels next to the device framebuffer; null when
  // the caller does not want host pixels
  uint32_t* host_fb;
  uint8_t* host_mask;
  // peer gather: the root rank's framebuffer (CUDA IPC, over NVLink); a
  // sharded rank writes its finished pixels there as well
  uint32_t* peer_fb;
  uint8_t* peer_mask;
};

// Frame constants live in constant memory, written once per frame by a
// memcpy that is part of the frame's CUDA graph (kernel parameters would be
// baked into the graph).
__constant__ FrameConst c_fc;

// Device counters; one instance per scene workspace, zeroed per frame.
struct Counters {
  unsigned long long cull[5];  // visible, degenerate, backfacing, frustum, between
  unsigned long long pairs;
  unsigned long long small_quads, large_tris;
  unsigned long long bin_error;  // ~min(bin * 64 + code), 0 = none (zeroed with the counters)
  unsigned int nvis;
  unsigned int error;  // bit0 visible capacity, bit1 item capacity
  unsigned int work_next[4];
  unsigned int spill_count[2];
  unsigned long long samples, fragments, thb, segments, invalid;
  unsigned long long bins_empty, bins_low, bins_high, bins_propagated;
  unsigned long long pool_pair;  // THB pool entries allocated
  unsigned long long walk_cost;  // sum of the bins' wave-walk costs (k_order_bins' split share)
  unsigned int shade_next[2];
  unsigned int seg_count;  // half-blocks queued for the segment-routing kernel
  unsigned int large_pairs;  // (large triangle, bin row) work pairs
  unsigned int setup_ticket;  // k_setup: block order for the decoupled look-back
  unsigned int list_count[2];  // owned bins to extract in the low / high pass
  unsigned int order_count;    // (bin, part) entries in k_shade's (mode 0/2) order list
  unsigned int shard_tri_count;  // sharded frames: triangles this rank sets up (k_shard_tris)
  unsigned int finalize_done;    // k_finalize CTAs finished (the last one publishes the counters)
};

// Decoded per-triangle shading inputs (unpack_color / decode_normal of the
// three corners, material colour and opacity), written by setup when
// triangles cover many pixels so the per-sample path skips the unpacking.
struct __align__(16) ShadeRec {
  float4 c[3];    // corner colours (valid when flags & 1)
  float4 n[3];    // corner normals (flags & 2) or n[0] = flat normal
  float4 mat;     // base rgb, opacity
  uint32_t flags;  // 1 colours, 2 normals, 4 the corners share an axis normal (axis in pad[0])
  uint32_t pad[3];
};
static_assert(sizeof(ShadeRec) == 128, "ShadeRec is one cache line");

struct HbDesc {
  uint32_t off, cnt, frags, pad;
};

struct Buffers {
  // scene
  const float4* pos;
  const uint32_t* vcol;
  const uint32_t* vnrm;
  const uint4* quads;
  const uint32_t* qmat;
  const MatDev* mats;
  const float2* vuv;     // per vertex, when the scene has UVs
  const float4* texels;  // every texture's mip levels, straight RGBA
  const uint4* texlev;   // per level: texel offset, width, height
  const uint2* texdesc;  // per texture: first level, level count
  // setup
  unsigned long long* block_state;  // k_setup look-back: status << 32 | count
  uint32_t* vq_src;
  uint4* vq_idx;  // the visible quad's vertex indices (k_setup_tris gathers without vq_src -> quads)
  uint2* vq_box;  // (x0 | x1 << 16, y0 | y1 << 16)
  uint32_t* vq_flags;  // bit0 large, 1 colors, 2 normals, 3 uvs, 4-5 cull flags
  uint32_t* vq_mat;
  uint4* vq_col;
  uint4* vq_nrm;
  float4* vq_uv;  // per visible quad with UVs: (uv0, uv1), (uv2, uv3)
  TriRec* tri;
  uint4* tri_meta;  // flat normal, material, quad index, tri | valid << 8
  uint32_t* tri_y;  // int16 y_min | int16 y_max << 16 (empty range when invalid)
  struct ShadeRec* shade;  // per triangle, when FrameConst::decoded
  // bins
  uint32_t* qcnt;
  uint32_t* tcnt;
  uint32_t* off;
  uint32_t* qcur;
  uint32_t* tcur;
  uint8_t* cat;
  uint8_t* prop;
  uint32_t* items;
  uint8_t* item_rows;     // per item: which of its bin's block-rows each of its triangles meets
  uint32_t* bin_list[2];  // owned bins per extraction pass (high: + propagated ones)
  uint32_t* lpair_cols;   // per large pair: covered bin-column words from the count pass
  uint32_t lpair_cols_cap;  // words
  uint32_t* prop_q;       // per bin: already appended to the high-pass list
  uint32_t* bin_cost;     // per bin: wave-walk shading cost (samples + 4 per THB)
  uint32_t* bin_order;    // (bin | part << 24 | log2(parts) << 28) in descending cost: k_shade's order
  // raster
  unsigned long long* slots;  // per (bin, row): samples, frags, thb, segments, invalid
  uint32_t* spill[2];
  uint8_t* scratch;
  uint64_t scratch_per_cta;
  uint32_t* fb;
  uint8_t* mask;
  uint64_t* hash;
  uint32_t* emit;
  struct HbDesc* hbd;  // per (bin, half-block): THB list in the pool
  uint32_t* pool_tri;
  uint32_t* pool_mask;  // coverage, bit = ly * 8 + lx
  uint32_t* pool_pre;   // exclusive fragment prefix
  uint4* seg_queue;  // half-blocks for the segment kernel: (bin * 32 + hb | high pass << 31, off, cnt, frags)
  uint16_t* pool_slot;  // per THB: the triangle's position in the bin list (k_shade staging slot)
  uint2* lpairs;        // (large triangle, bin row) pairs for k_bin_large
  uint32_t* shard_tris; // sharded frames: the visible triangles this rank's bins can use
  // depth filters above 8 (MemFilter): nodes per lane, and the global
  // scratch ([CTA][warp][node/slot][lane]) when they do not fit shared memory
  uint8_t* dfm_g;
  uint32_t dfm_cap;
  // fused raster scratch per k_extract CTA: candidate triangle setups (for
  // row spans spread over the warp) and the item's TBR planes (phase B
  // centroid depths and the shading), L2-resident while the item runs
  TriRec* cscratch;
  struct TriPlanes* tplanes;
  uint64_t cs_per_cta, tp_per_cta;        // k_extract<false> CTAs (shared-memory items)
  uint64_t cs_per_cta_g, tp_per_cta_g;    // k_extract<true> CTAs (global-scratch items)
  uint64_t cs_off_g, tp_off_g;            // where the latter's slices start
  uint32_t dfm_ctas;  // grid cap of the shading kernels when dfm_g is used
  Counters* ctr;
};

// Exact unpack tables: g_lut_c[q] = float(q) / 255.0f (unpack_color,
// packing.hpp:63-66) and g_lut_n[q + 512] = float(q) / 511.0f
// (decode_normal, packing.hpp:43-49), filled by the host with IEEE division.
__device__ float g_lut_c[256];
__device__ float g_lut_n[1024];

__device__ __forceinline__ float lut_c(uint32_t w, int shift) {
  return __ldg(&g_lut_c[(w >> shift) & 0xffu]);
}
__device__ __forceinline__ float lut_n(uint32_t w, int shift) {
  int32_t q = (int32_t)(((w >> shift) & 0x3ffu) << 22) >> 22;
  return __ldg(&g_lut_n[q + 512]);
}

// Shared-memory copies of the tables for the shading kernels (per-sample
// unpacking on the generic path); filled by load_shared_luts at kernel start.
__shared__ float s_lut_c[256];
__shared__ float s_lut_n[1024];
__device__ __forceinline__ void load_shared_luts() {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_lut_c[i] = g_lut_c[i];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s_lut_n[i] = g_lut_n[i];
}
__device__ __forceinline__ float slut_c(uint32_t w, int shift) { return s_lut_c[(w >> shift) & 0xffu]; }
__device__ __forceinline__ float slut_n(uint32_t w, int shift) {
  const int32_t q = (int32_t)(((w >> shift) & 0x3ffu) << 22) >> 22;
  return s_lut_n[q + 512];
}

// Axis index (component * 2 + negative) of a packed X10Y10Z10 normal word
// that encodes one of the six axis-aligned unit normals (decode_normal gives
// exactly 0 and +-1 for them), else -1.
__device__ __forceinline__ int axis_of_word(uint32_t w) {
  switch (w) {
    case 0x1ffu: return 0;
    case 0x201u: return 1;
    case 0x1ffu << 10: return 2;
    case 0x201u << 10: return 3;
    case 0x1ffu << 20: return 4;
    case 0x201u << 20: return 5;
    default: return -1;
  }
}

// ------------------------------------------------------------ setup

__device__ __forceinline__ uint32_t checked_index(uint32_t i, uint32_t n) {
  VEIL_CHECK(i < n);
  return i;
}

__device__ __forceinline__ void load_quad(const Buffers& B, uint32_t q, uint4* idx,
                                          float4 p[4]) {
  *idx = B.quads[q];
  p[0] = __ldg(&B.pos[idx->x]);
  p[1] = __ldg(&B.pos[idx->y]);
  p[2] = __ldg(&B.pos[idx->z]);
  p[3] = __ldg(&B.pos[idx->w]);
}

// triangle_front_facing, setup.cpp:104-110
__device__ __forceinline__ bool front_facing(const FrameConst& fc, const double* p0,
                                             const double* p1, const double* p2) {
  double a[3] = {__dsub_rn(p1[0], p0[0]), __dsub_rn(p1[1], p0[1]), __dsub_rn(p1[2], p0[2])};
  double b[3] = {__dsub_rn(p2[0], p0[0]), __dsub_rn(p2[1], p0[1]), __dsub_rn(p2[2], p0[2])};
  double n[3];
  cross3(a, b, n);
  if (fc.has_eye) {
    double v[3] = {__dsub_rn(fc.eye[0], p0[0]), __dsub_rn(fc.eye[1], p0[1]),
                   __dsub_rn(fc.eye[2], p0[2])};
    return dot3(n, v) > 0.0;
  }
  return dot3(n, fc.fwd) < 0.0;
}

__device__ __forceinline__ uint32_t outside_mask(const double* c) {
  uint32_t m = 0;
  if (c[0] < -c[3]) m |= 1u;
  if (c[0] > c[3]) m |= 2u;
  if (c[1] < -c[3]) m |= 4u;
  if (c[1] > c[3]) m |= 8u;
  if (c[2] < 0.0) m |= 16u;
  if (c[2] > c[3]) m |= 32u;
  return m;
}

__constant__ int c_quad_edges[5][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {0, 2}};
__constant__ int c_tri_edges[3][2] = {{0, 1}, {1, 2}, {2, 0}};

struct CullOut {
  int reason;  // 0 visible, 1 degenerate, 2 backfacing, 3 frustum, 4 between samples
  uint32_t flags;
  int x0, y0, x1, y1;
  bool large;
};

// project_quad + cull_projected, setup.cpp:119-186
__device__ void cull_quad(const FrameConst& fc, const uint4& idx, const float4 p[4],
                          double clip[4][4], CullOut* o) {
  o->flags = 0;
  o->large = false;
  bool d0 = idx.x == idx.y || idx.y == idx.z || idx.x == idx.z;
  bool d1 = idx.x == idx.z || idx.z == idx.w || idx.x == idx.w;
#pragma unroll
  for (int i = 0; i < 4; ++i) to_clip(fc.m, p[i].x, p[i].y, p[i].z, clip[i]);
  if (d0) o->flags |= 1u;
  if (d1) o->flags |= 2u;
  if (d0 && d1) {
    o->reason = 1;
    return;
  }
  if (fc.backface) {
    double w[4][3];
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i][0] = p[i].x, w[i][1] = p[i].y, w[i][2] = p[i].z;
    bool b0 = d0 ? true : !front_facing(fc, w[0], w[1], w[2]);
    bool b1 = d1 ? true : !front_facing(fc, w[0], w[2], w[3]);
    if (!d0 && b0) o->flags |= 1u;
    if (!d1 && b1) o->flags |= 2u;
    if (b0 && b1) {
      o->reason = 2;
      return;
    }
  }
  if ((outside_mask(clip[0]) & outside_mask(clip[1]) & outside_mask(clip[2]) &
       outside_mask(clip[3])) != 0) {
    o->reason = 3;
    return;
  }
  double px[4], py[4], pw[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double h[3];
    hpixel(clip[i], fc.width, fc.height, h);
    px[i] = h[0], py[i] = h[1], pw[i] = h[2];
  }
  double bx0, bx1, by0, by1;
  extend_axis<4, 5>(px, pw, c_quad_edges, (double)fc.width, &bx0, &bx1);
  extend_axis<4, 5>(py, pw, c_quad_edges, (double)fc.height, &by0, &by1);
  int xf, xl, yf, yl;
  pixel_range(bx0, bx1, fc.width, &xf, &xl);
  pixel_range(by0, by1, fc.height, &yf, &yl);
  if (bx0 > bx1 || by0 > by1 || xf > xl || yf > yl) {
    o->reason = 4;
    return;
  }
  o->reason = 0;
  o->x0 = xf / kBin;
  o->y0 = yf / kBin;
  o->x1 = xl / kBin;
  o->y1 = yl / kBin;
  o->large = (o->x1 - o->x0 + 1) * (o->y1 - o->y0 + 1) > 4;
}

// Exclusive scan of up to 1024*kPer values with one CTA.
template <int kThreads>
__device__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* total) {
  __shared__ uint32_t warp_sums[kThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t s = lane < kThreads / 32 ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < kThreads / 32) warp_sums[lane] = s;
  }
  __syncthreads();
  uint32_t warp_prefix = warp ? warp_sums[warp - 1] : 0;
  *total = warp_sums[kThreads / 32 - 1];
  __syncthreads();
  return warp_prefix + x - v;
}


// triangle setup, setup.cpp:209-239 (+ flat normal, setup.cpp:342-343)
__device__ void triangle_setup(const FrameConst& fc, const double c0[4], const double c1[4],
                               const double c2[4], TriRec* out, bool* valid) {
  double v0[3], v1[3], v2[3], e0[3], e1[3], e2[3];
  hpixel(c0, fc.width, fc.height, v0);
  hpixel(c1, fc.width, fc.height, v1);
  hpixel(c2, fc.width, fc.height, v2);
  cross3(v1, v2, e0);
  cross3(v2, v0, e1);
  cross3(v0, v1, e2);
  double det = dot3(e0, v0);
  TriRec r;
  memset(&r, 0, sizeof r);
  r.y_min = 0;
  r.y_max = -1;
  *valid = false;
  if (!(det == 0.0 || !isfinite(det))) {
    double s = det > 0.0 ? 1.0 : -1.0;
    const double* es[3] = {e0, e1, e2};
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      r.e[i].a = __dmul_rn(es[i][0], s);
      r.e[i].b = __dmul_rn(es[i][1], s);
      r.e[i].c = __dmul_rn(es[i][2], s);
    }
    double inv_det = __ddiv_rn(1.0, det);
    double z0 = c0[2], z1 = c1[2], z2 = c2[2];
    double* dz[3] = {&r.dz.a, &r.dz.b, &r.dz.c};
    double* iw[3] = {&r.iw.a, &r.iw.b, &r.iw.c};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      *dz[k] = __dmul_rn(
          __dadd_rn(__dadd_rn(__dmul_rn(e0[k], z0), __dmul_rn(e1[k], z1)), __dmul_rn(e2[k], z2)),
          inv_det);
      *iw[k] = __dmul_rn(__dadd_rn(__dadd_rn(e0[k], e1[k]), e2[k]), inv_det);
    }
    double py[3] = {v0[1], v1[1], v2[1]}, pw[3] = {v0[2], v1[2], v2[2]};
    double lo, hi;
    extend_axis<3, 3>(py, pw, c_tri_edges, (double)fc.height, &lo, &hi);
    int f, l;
    pixel_range(lo, hi, fc.height, &f, &l);
    r.y_min = f;
    r.y_max = l;
    *valid = true;
  }
  *out = r;
}

__device__ __forceinline__ uint32_t flat_normal(const float4& a, const float4& b,
                                                const float4& c) {
  double w0[3] = {a.x, a.y, a.z}, w1[3] = {b.x, b.y, b.z}, w2[3] = {c.x, c.y, c.z};
  double u[3] = {__dsub_rn(w1[0], w0[0]), __dsub_rn(w1[1], w0[1]), __dsub_rn(w1[2], w0[2])};
  double v[3] = {__dsub_rn(w2[0], w0[0]), __dsub_rn(w2[1], w0[1]), __dsub_rn(w2[2], w0[2])};
  double n[3];
  cross3(u, v, n);
  double l2 = dot3(n, n);
  if (l2 <= 0.0) {
    n[0] = n[1] = n[2] = 0.0;
  } else {
    double inv = __ddiv_rn(1.0, __dsqrt_rn(l2));
    n[0] = __dmul_rn(n[0], inv);
    n[1] = __dmul_rn(n[1], inv);
    n[2] = __dmul_rn(n[2], inv);
  }
  return encode_normal((float)n[0], (float)n[1], (float)n[2]);
}

// A triangle's edge and depth planes (the shading inputs of a TriRec).
struct TriPlanes {
  Fn3 e[3];
  Fn3 dz;
};
static_assert(sizeof(TriPlanes) == 96, "TriPlanes layout");

// Fused raster: the setup of visible triangle ti recomputed from the scene
// positions exactly as k_setup_tris computes it (same expressions and
// roundings, so the same doubles); only called for triangles whose y range
// in tri_y is non-empty, i.e. valid ones.
__device__ __forceinline__ void recompute_setup(const FrameConst& fc, const Buffers& B, uint32_t ti,
                                                TriRec* out) {
  const uint4 idx = __ldg(&B.vq_idx[ti >> 1]);
  const uint32_t i1 = (ti & 1u) == 0 ? idx.y : idx.z, i2 = (ti & 1u) == 0 ? idx.z : idx.w;
  const float4 p0 = __ldg(&B.pos[idx.x]), p1 = __ldg(&B.pos[i1]), p2 = __ldg(&B.pos[i2]);
  double c0[4], c1[4], c2[4];
  to_clip(fc.m, p0.x, p0.y, p0.z, c0);
  to_clip(fc.m, p1.x, p1.y, p1.z, c1);
  to_clip(fc.m, p2.x, p2.y, p2.z, c2);
  bool valid;
  triangle_setup(fc, c0, c1, c2, out, &valid);
}

// Phase 1 of setup in one pass (setup.cpp:252-302): cull every quad, then
// compact the visible ones in ascending input order. Blocks take tickets in
// launch order and chain their visible counts with a decoupled look-back
// (status word per block: 1 = own count, 2 = inclusive prefix), so the
// compaction needs no second cull pass and no separate scan kernel.
__device__ __forceinline__ unsigned long long ld_state(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

// Programmatic dependent launch: the frame's kernels are launched with
// programmatic stream serialization, so a kernel's CTAs may become resident
// while its predecessor drains; each kernel waits here (griddepcontrol.wait:
// the predecessor grid has completed and its memory is visible) before it
// touches anything a predecessor wrote. Without the launch attribute it is a
// no-op.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Lets the next kernel's CTAs launch now (they run their prologue and wait in
// grid_dep_wait); used by kernels whose CTAs are all resident at once, so the
// early dependents cannot starve them.
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// 32-bit shared-window address of a shared-memory object (for inline PTX).
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// 4 CTAs/SM (64 registers, small spill) beats 3 at 80 registers: the cull is
// gather- and FP64-latency bound (C4 setup -6%, measured; 5 or 6 spill more)
__global__ void __launch_bounds__(kSetupBlock, 4) k_setup(Buffers B, uint32_t nblocks) {
  grid_dep_wait();
  const FrameConst& fc = c_fc;
  __shared__ uint32_t s_bid, s_excl;
  if (threadIdx.x == 0) s_bid = atomicAdd(&B.ctr->setup_ticket, 1u);
  __syncthreads();
  const uint32_t bid = s_bid;
  const uint32_t q = bid * kSetupBlock + threadIdx.x;
  uint4 idx = make_uint4(0, 0, 0, 0);
  float4 p[4];
  double clip[4][4];
  CullOut o;
  o.reason = -1;
  if (q < fc.nquads) {
    load_quad(B, q, &idx, p);
    cull_quad(fc, idx, p, clip, &o);
  }
  // the visible quad's material and corner attributes (setup.cpp:320-333)
  // are gathered before the block's compaction barriers, so their latency
  // overlaps warp 0's look-back instead of following it
  uint32_t mat = 0, mflags = 0;
  uint4 col = make_uint4(0, 0, 0, 0), nrm = make_uint4(0, 0, 0, 0);
  if (o.reason == 0) {
    mat = B.qmat[q];
    mflags = B.mats[mat].flags;
    if (mflags & 1u) col = make_uint4(B.vcol[idx.x], B.vcol[idx.y], B.vcol[idx.z], B.vcol[idx.w]);
    if (mflags & 2u) nrm = make_uint4(B.vnrm[idx.x], B.vnrm[idx.y], B.vnrm[idx.z], B.vnrm[idx.w]);
  }
  // visible-rank scan and the four cull-reason counts in two barriers: each
  // warp posts its visible count and reason ballots, warp 0 scans and sums
  constexpr int kWarps = kSetupBlock / 32;
  __shared__ uint32_t s_wvis[kWarps], s_wreason[4][kWarps];
  uint32_t rank, total;
  {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned vis = __ballot_sync(0xffffffffu, o.reason == 0);
    if (lane == 0) s_wvis[warp] = __popc(vis);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const unsigned m = __ballot_sync(0xffffffffu, o.reason == k + 1);
      if (lane == 0) s_wreason[k][warp] = __popc(m);
    }
    __syncthreads();
    if (warp == 0) {
      uint32_t x = lane < kWarps ? s_wvis[lane] : 0u;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
      }
      if (lane < kWarps) s_wvis[lane] = x;  // inclusive per-warp prefix
    }
    __syncthreads();
    total = s_wvis[kWarps - 1];
    rank = (warp ? s_wvis[warp - 1] : 0u) + __popc(vis & ((1u << lane) - 1u));
  }
  int deg = 0, back = 0, fru = 0, bet = 0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      deg += (int)s_wreason[0][w];
      back += (int)s_wreason[1][w];
      fru += (int)s_wreason[2][w];
      bet += (int)s_wreason[3][w];
    }
  }
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    unsigned long long* state = B.block_state;
    if (lane == 0)
      atomicExch(&state[bid], ((bid == 0 ? 2ull : 1ull) << 32) | (unsigned long long)total);
    uint32_t excl = 0;
    if (bid > 0) {
      long long top = (long long)bid - 1;
      for (;;) {
        const long long j = top - lane;
        unsigned long long w = j >= 0 ? ld_state(&state[j]) : (2ull << 32);
        while (__any_sync(0xffffffffu, (w >> 32) == 0ull))
          if ((w >> 32) == 0ull) w = ld_state(&state[j]);
        const uint32_t v = (uint32_t)w;
        const unsigned inc = __ballot_sync(0xffffffffu, (w >> 32) == 2ull);
        if (inc) {  // nearest inclusive prefix: add it and the counts after it
          const int k = __ffs(inc) - 1;
          excl += __reduce_add_sync(0xffffffffu, lane <= k ? v : 0u);
          break;
        }
        excl += __reduce_add_sync(0xffffffffu, v);
        top -= 32;
      }
      if (lane == 0) atomicExch(&state[bid], (2ull << 32) | (unsigned long long)(excl + total));
    }
    if (lane == 0) {
      s_excl = excl;
      if (total) atomicAdd(&B.ctr->cull[0], (unsigned long long)total);
      if (deg) atomicAdd(&B.ctr->cull[1], (unsigned long long)deg);
      if (back) atomicAdd(&B.ctr->cull[2], (unsigned long long)back);
      if (fru) atomicAdd(&B.ctr->cull[3], (unsigned long long)fru);
      if (bet) atomicAdd(&B.ctr->cull[4], (unsigned long long)bet);
      if (bid == nblocks - 1) {
        const uint32_t nvis = excl + total;
        B.ctr->nvis = nvis;
        // setup.cpp:298-299: 2 * visible > 2^24 is a capacity error
        if ((unsigned long long)nvis * 2ull > (unsigned long long)fc.tri_cap) atomicOr(&B.ctr->error, 1u);
      }
    }
  }
  __syncthreads();
  if (o.reason != 0) return;
  const uint32_t slot = s_excl + rank;
  const bool has_c = mflags & 1u, has_n = mflags & 2u;
  B.vq_src[slot] = q;
  B.vq_idx[slot] = idx;
  B.vq_box[slot] = make_uint2((uint32_t)o.x0 | ((uint32_t)o.x1 << 16),
                              (uint32_t)o.y0 | ((uint32_t)o.y1 << 16));
  const bool has_uv = mflags & 4u;
  B.vq_flags[slot] = (o.large ? 1u : 0u) | (has_c ? 2u : 0u) | (has_n ? 4u : 0u) | (has_uv ? 8u : 0u) |
                     (o.flags << 4);
  B.vq_mat[slot] = mat;
  if (has_uv) {  // setup.cpp:326-328
    const float2 u0 = B.vuv[idx.x], u1 = B.vuv[idx.y], u2 = B.vuv[idx.z], u3 = B.vuv[idx.w];
    B.vq_uv[2 * (size_t)slot] = make_float4(u0.x, u0.y, u1.x, u1.y);
    B.vq_uv[2 * (size_t)slot + 1] = make_float4(u2.x, u2.y, u3.x, u3.y);
  }
  // (corner colours / normals gathered above, one quad per lane; moving these
  // gathers into the sharded k_setup_tris measured slower: C4 setup +0.1 ms at
  // one GPU, the same at eight)
  B.vq_col[slot] = col;
  B.vq_nrm[slot] = nrm;
}

// Triangle setups (setup.cpp:305-349, compute_triangle_setup 209-239): one
// thread per visible triangle, re-projecting its quad's corners exactly as the
// reference's phase 2 does. The warp's 128-byte records are staged in shared
// memory and written back as 512-byte contiguous runs (coalesced stores).
constexpr int kTriBlock = 128;

// Sharded frames: the visible triangles a rank's bins can use -- every large
// quad's (their bin coverage comes from the triangles) and those of the small
// quads whose bin box meets an owned bin -- listed (in any order) so that
// k_setup_tris<true> runs over them only (it used to launch over every
// triangle and skip the others: C4 at 8 ranks 0.35 ms for 1/8 of the work).
__global__ void __launch_bounds__(256) k_shard_tris(Buffers B) {
  grid_dep_wait();
  const FrameConst& fc = c_fc;
  __shared__ unsigned int n_small;  // per-block count, one global atomic
  if (B.ctr->error & 1u) return;
  if (threadIdx.x == 0) n_small = 0;
  __syncthreads();
  const uint32_t nq = B.ctr->nvis;
  const int lane = threadIdx.x & 31;
  for (uint32_t base = blockIdx.x * blockDim.x; base < nq; base += gridDim.x * blockDim.x) {
    const uint32_t q = base + threadIdx.x;
    bool need = false;
    if (q < nq) {
      need = B.vq_flags[q] & 1u;
      if (!need) {
        const uint2 box = B.vq_box[q];
        const int x0 = (int)(box.x & 0xffffu), x1 = (int)(box.x >> 16), y0 = (int)(box.y & 0xffffu),
                  y1 = (int)(box.y >> 16);
        for (int by = y0; by <= y1; ++by)
          for (int bx = x0; bx <= x1; ++bx) need |= ((bx + 3 * by) % fc.world) == fc.rank;
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, need);
    // (the frame's visible small-quad count, which k_bin_pass takes when
    // it walks every quad)
    const unsigned sm = __ballot_sync(0xffffffffu, q < nq && !(B.vq_flags[q] & 1u));
    if (lane == 0 && sm) atomicAdd(&n_small, (unsigned)__popc(sm));
    uint32_t at = 0;
    if (lane == 0 && m) at = atomicAdd(&B.ctr->shard_tri_count, 2u * (uint32_t)__popc(m));
    at = __shfl_sync(0xffffffffu, at, 0);
    if (need) {
      const uint32_t pos = at + 2u * (uint32_t)__popc(m & ((1u << lane) - 1u));
      B.shard_tris[pos] = 2u * q;
      B.shard_tris[pos + 1] = 2u * q + 1u;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && n_small) atomicAdd(&B.ctr->small_quads, (unsigned long long)n_small);
}

// kCtas: resident CTAs per SM the registers are budgeted for -- 7 (72
// registers) for small frames, 6 (80, no spill) for frames of a million
// triangles or more, where fewer spills beat one more CTA (C5 setup -1.5%,
// C4 -0.9%; C2's 131k triangles lose 2 us at 6)
template <bool kShard, int kCtas = 7>
__global__ void __launch_bounds__(kTriBlock, kCtas) k_setup_tris(Buffers B) {
  grid_dep_wait();
  const FrameConst& fc = c_fc;
  __shared__ __align__(16) TriRec stage[kTriBlock];
  if (B.ctr->error & 1u) return;
  // kShard: the triangles of k_shard_tris's list (records stored one line per
  // lane); else every visible triangle (records staged per warp and written as
  // contiguous runs)
  const uint32_t nt = kShard ? B.ctr->shard_tri_count : 2u * B.ctr->nvis;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t base = blockIdx.x * kTriBlock; base < nt; base += gridDim.x * kTriBlock) {
    const uint32_t li = base + threadIdx.x;
    const bool needed = li < nt;
    const uint32_t ti = kShard ? (needed ? B.shard_tris[li] : 0u) : li;
    TriRec rec;
    memset(&rec, 0, sizeof rec);
    rec.y_min = 0;
    rec.y_max = -1;
    uint4 meta = make_uint4(0, 0, 0, 0);
    bool valid = false;
    uint32_t slot = 0, t = 0, vf = 0, mat = 0;
    if (needed) {
      slot = ti >> 1;
      t = ti & 1u;
      vf = B.vq_flags[slot];
      const uint4 idx = B.vq_idx[slot];
      mat = B.vq_mat[slot];

      if (!((vf >> 4) & (1u << t))) {  // not individually culled
        const uint32_t i1 = t == 0 ? idx.y : idx.z, i2 = t == 0 ? idx.z : idx.w;
        const float4 p0 = __ldg(&B.pos[idx.x]), p1 = __ldg(&B.pos[i1]), p2 = __ldg(&B.pos[i2]);
        double c0[4], c1[4], c2[4];
        to_clip(fc.m, p0.x, p0.y, p0.z, c0);
        to_clip(fc.m, p1.x, p1.y, p1.z, c1);
        to_clip(fc.m, p2.x, p2.y, p2.z, c2);
        triangle_setup(fc, c0, c1, c2, &rec, &valid);
        meta.x = flat_normal(p0, p1, p2);
        meta.y = mat;
        meta.z = slot;
        meta.w = t | (valid ? 0x100u : 0u);
      }
    }
    // the 128-byte record is stored when some consumer reads it: always for
    // large quads (k_bin_large), for small ones unless the fused raster
    // recomputes them (fc.write_tri == 0)
    const bool store = needed && (fc.write_tri || (vf & 1u));
    if (kShard) {
      if (store) B.tri[ti] = rec;
    } else {  // coalesced copy-out of this warp's 32 records (4 KB)
      // the previous run's bulk store has finished reading the stage
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp();
      stage[threadIdx.x] = rec;
      const unsigned needm = __ballot_sync(0xffffffffu, store);
      const uint32_t wbase = base + (uint32_t)warp * 32u;
      const uint32_t nrec = wbase < nt ? min(32u, nt - wbase) : 0u;
      const unsigned full = nrec >= 32u ? 0xffffffffu : ((1u << nrec) - 1u);
      if (nrec && (needm & full) == full && fc.bulk_stage) {
        // every record of the run is stored: one bulk copy (TMA engine)
        // shared -> global, issued by one lane, the warp moves on
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(B.tri + wbase),
                       "r"(smem_addr(&stage[warp * 32])), "r"(nrec * (uint32_t)sizeof(TriRec))
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      } else {
        __syncwarp();
        const uint4* src = reinterpret_cast<const uint4*>(&stage[warp * 32]);
        uint4* dst = reinterpret_cast<uint4*>(B.tri + wbase);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t e = (uint32_t)k * 32u + lane;  // 16-byte chunk index within the warp
          if (e < nrec * 8u && ((needm >> (e >> 3)) & 1u)) dst[e] = src[e];
        }
        __syncwarp();
      }
    }
    if (needed) {
      B.tri_meta[ti] = meta;
      B.tri_y[ti] = valid ? ((uint32_t)(uint16_t)(int16_t)rec.y_min |
                             ((uint32_t)(uint16_t)(int16_t)rec.y_max << 16))
                          : 0x00000001u;  // y_min 1 > y_max 0
      if (fc.decoded && valid) {
        // corner slots (0,1,2) / (0,2,3), shading.cpp:41-44
        const MatDev md = B.mats[mat];
        const bool has_c = vf & 2u, has_n = vf & 4u;
        const uint4 col = B.vq_col[slot], nrm = B.vq_nrm[slot];
        const uint32_t cw[3] = {col.x, t == 0 ? col.y : col.z, t == 0 ? col.z : col.w};
        const uint32_t nw[3] = {nrm.x, t == 0 ? nrm.y : nrm.z, t == 0 ? nrm.z : nrm.w};
        ShadeRec sr;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          sr.c[k] = make_float4(lut_c(cw[k], 0), lut_c(cw[k], 8), lut_c(cw[k], 16), lut_c(cw[k], 24));
          const uint32_t w = has_n ? nw[k] : meta.x;
          sr.n[k] = make_float4(lut_n(w, 0), lut_n(w, 10), lut_n(w, 20), 0.0f);
        }
        sr.mat = make_float4(md.base[0], md.base[1], md.base[2], md.opacity);
        sr.flags = (has_c ? 1u : 0u) | (has_n ? 2u : 0u);
        sr.pad[0] = sr.pad[1] = sr.pad[2] = 0;
        if (has_n && nw[0] == nw[1] && nw[1] == nw[2] && axis_of_word(nw[0]) >= 0) {
          sr.flags |= 4u;  // one axis-aligned vertex normal: light from s_axis_light
          sr.pad[0] = (uint32_t)axis_of_word(nw[0]);
        }
        B.shade[ti] = sr;
      }
    }
  }
  // outstanding bulk stores complete before the CTA (and its stage) retires
  if (!kShard && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------ binning

__device__ __forceinline__ void warp_agg_add(uint32_t* base, uint32_t bin, bool active,
                                             uint32_t* slot_out) {
  // Warp-aggregated atomic: lanes with the same bin share one atomicAdd.
  unsigned mask = __ballot_sync(0xffffffffu, active);
  if (!active) return;
  unsigned peers = __match_any_sync(mask, bin);
  int leader = __ffs(peers) - 1;
  int lane = threadIdx.x & 31;
  uint32_t base_slot = 0;
  if (lane == leader) base_slot = atomicAdd(&base[bin], (uint32_t)__popc(peers));
  base_slot = __shfl_sync(peers, base_slot, leader);
  if (slot_out) *slot_out = base_slot + __popc(peers & ((1u << lane) - 1u));
}

// rasterize_triangle_bins, binning.hpp:89-117: calls fn(bin) per covered bin
template <typename Fn>
__device__ void tri_bins(const FrameConst& fc, const TriRec& t, Fn&& fn) {
  int y = t.y_min;
  while (y <= t.y_max) {
    int bin_row = y / kBin;
    int row_end = min(t.y_max, (bin_row + 1) * kBin - 1);
    uint64_t mask[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (; y <= row_end; ++y) {
      int b, l;
      if (!row_span(t, y, 0, fc.width - 1, &b, &l)) continue;
      int b0 = b / kBin, b1 = l / kBin;
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        int lo = max(b0, w * 64), hi = min(b1, w * 64 + 63);
        if (lo > hi) continue;
        int n = hi - lo + 1;
        uint64_t bits = n == 64 ? ~0ull : (((1ull << n) - 1ull) << (lo - w * 64));
        mask[w] |= bits;
      }
    }
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      uint64_t bits = mask[w];
      while (bits) {
        int b = w * 64 + __ffsll((long long)bits) - 1;
        bits &= bits - 1;
        if (b < fc.bins_x) fn(bin_row * fc.bins_x + b);
      }
    }
  }
}

// Which of a bin's four 8-row block-rows a triangle's pixel-row range meets
// (the candidate test of k_extract's phase A, precomputed at binning so the
// extraction scans a 1-byte mask per item instead of gathering tri_y).
__device__ __forceinline__ uint32_t block_rows_mask(uint32_t yy, int by, int height) {
  const int y_lo = (int)(int16_t)(yy & 0xffffu), y_hi = (int)(int16_t)(yy >> 16);
  uint32_t m = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int ry0 = by * kBin + r * 8, ry1 = min(ry0 + 7, height - 1);
    if (max(y_lo, ry0) <= min(y_hi, ry1)) m |= 1u << r;
  }
  return m;
}

template <bool kWrite, bool kList>
__global__ void __launch_bounds__(256) k_bin_pass(Buffers B) {
  grid_dep_wait();
  const FrameConst& fc = c_fc;
  __shared__ unsigned int n_small, n_large;  // per-block counts, one global atomic each
  if (B.ctr->error) return;
  if (threadIdx.x == 0) n_small = n_large = 0;
  __syncthreads();
  // sharded frames walk k_shard_tris's list (its even entries are 2q): the
  // other quads cannot reach an owned bin; their small-quad count was taken
  // there
  constexpr bool listed = kList;  // (a template parameter: the runtime test cost one GPU 15 us)
  const uint32_t nvis = listed ? B.ctr->shard_tri_count / 2u : B.ctr->nvis;
  for (uint32_t base = blockIdx.x * 256; base < nvis; base += gridDim.x * 256) {
    const uint32_t i = base + threadIdx.x;
    bool in = i < nvis;
    const uint32_t q = listed ? (in ? B.shard_tris[2u * i] >> 1 : 0u) : i;
    uint32_t flags = in ? B.vq_flags[q] : 0u;
    bool small = in && !(flags & 1u);
    uint2 box = in ? B.vq_box[q] : make_uint2(0, 0);
    uint32_t x0 = box.x & 0xffffu, x1 = box.x >> 16, y0 = box.y & 0xffffu, y1 = box.y >> 16;
    // small quads: every bin of the AABB (binning.hpp:76-81), 1..4 bins
    uint32_t nb = small ? (x1 - x0 + 1) * (y1 - y0 + 1) : 0u;
    if (!kWrite && !listed) {
      unsigned sm = __ballot_sync(0xffffffffu, small);
      if ((threadIdx.x & 31) == 0 && sm) atomicAdd(&n_small, (unsigned)__popc(sm));
    }
    if (!kWrite && in && (flags & 1u)) {
      // large quad: one (triangle, bin row) pair per bin row of each valid
      // triangle for k_bin_large (a warp per pair)
      for (uint32_t t = 0; t < 2; ++t) {
        const uint32_t ti = q * 2 + t;
        if (!(B.tri_meta[ti].w & 0x100u)) continue;
        const uint32_t yy = B.tri_y[ti];
        const int y_lo = (int)(int16_t)(yy & 0xffffu), y_hi = (int)(int16_t)(yy >> 16);
        atomicAdd(&n_large, 1u);
        if (y_lo > y_hi) continue;
        const uint32_t r0 = (uint32_t)y_lo / kBin, nr = (uint32_t)y_hi / kBin - r0 + 1u;
        // a sharded rank keeps the bin rows where the quad's bin columns meet
        // an owned bin (owner (bx + 3 by) mod G: the first owned column of
        // row R is x0 + ((rank - 3R - x0) mod G))
        uint32_t rows_mask = 0xffffffffu;  // (bit r: row r0 + r kept; rows >= 32 always kept)
        uint32_t nkeep = nr;
        if (fc.world > 1 && box.x >> 16 < (box.x & 0xffffu) + (uint32_t)fc.world - 1u) {
          const int G = fc.world, bx0 = (int)(box.x & 0xffffu), bx1 = (int)(box.x >> 16);
          nkeep = 0;
          for (uint32_t r = 0; r < nr; ++r) {
            const int R = (int)(r0 + r);
            const int first = bx0 + ((((fc.rank - 3 * R - bx0) % G) + G) % G);
            const bool keep = r >= 32u || first <= bx1;
            if (r < 32u && !keep) rows_mask &= ~(1u << r);
            nkeep += keep ? 1u : 0u;
          }
        }
        if (!nkeep) continue;
        const uint32_t at = atomicAdd(&B.ctr->large_pairs, nkeep);
        if ((unsigned long long)at + nkeep > fc.lpairs_cap) {
          atomicOr(&B.ctr->error, 16u);  // pair list capacity: grow and re-run
          continue;
        }
        for (uint32_t r = 0, k = 0; r < nr; ++r)
          if (r >= 32u || ((rows_mask >> r) & 1u)) B.lpairs[at + k++] = make_uint2(ti, r0 + r);
      }
    }
    for (uint32_t k = 0; k < 4; ++k) {
      bool act = k < nb;
      uint32_t bx = x0 + (k % (x1 - x0 + 1 > 0 ? x1 - x0 + 1 : 1));
      uint32_t by = y0 + (k / (x1 - x0 + 1 > 0 ? x1 - x0 + 1 : 1));
      // a sharded rank fills only its own bins' lists
      if (fc.world > 1 && ((bx + 3u * by) % (uint32_t)fc.world) != (uint32_t)fc.rank) act = false;
      uint32_t bin = act ? by * (uint32_t)fc.bins_x + bx : 0u;
      if (__any_sync(0xffffffffu, act)) {
        if (kWrite) {
          uint32_t slot = 0;
          warp_agg_add(B.qcur, bin, act, &slot);
          if (act && slot < fc.items_cap) {
            VEIL_CHECK(bin < (uint32_t)fc.nbins);
            B.items[slot] = q;
            const uint2 ty = *reinterpret_cast<const uint2*>(&B.tri_y[2 * q]);
            B.item_rows[slot] = (uint8_t)(block_rows_mask(ty.x, (int)by, fc.height) |
                                          (block_rows_mask(ty.y, (int)by, fc.height) << 4));
          }
        } else {
          warp_agg_add(B.qcnt, bin, act, nullptr);
        }
      }
    }
  }
  if (!kWrite) {
    __syncthreads();
    if (threadIdx.x == 0) {
      if (n_small) atomicAdd(&B.ctr->small_quads, (unsigned long long)n_small);
      if (n_large) atomicAdd(&B.ctr->large_tris, (unsigned long long)n_large);
    }
  }
}

// Large quads' valid triangles (rasterize_triangle_bins, binning.hpp:89-117):
// one warp per (triangle, bin row) pair, lane = pixel row; the per-row
// covered bin-column ranges are OR-reduced across the warp, then each set bin
// is counted (kWrite = false) or receives the triangle index.
template <bool kWrite>
__global__ void __launch_bounds__(256) k_bin_large(Buffers B) {
  grid_dep_wait();
  const FrameConst& fc = c_fc;
  if (B.ctr->error) return;
  const uint32_t npairs = min(B.ctr->large_pairs, fc.lpairs_cap);
  const int lane = threadIdx.x & 31;
  const uint32_t gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const int nwords = (fc.bins_x + 31) / 32;
  for (uint32_t w = gwarp; w < npairs; w += nwarps) {
    const uint2 pr = B.lpairs[w];
    const uint32_t ti = pr.x;
    const int R = (int)pr.y;
    // the count pass stores the pair's column words; the write pass reuses
    // them instead of repeating the row spans (when they fit the cache)
    const bool cached = (unsigned long long)(w + 1) * (unsigned long long)nwords <= B.lpair_cols_cap;
    int b0 = 1, b1 = 0;
    if (!(kWrite && cached)) {
      const TriRec& tr = B.tri[ti];
      const int y = R * kBin + lane;
      if (y >= tr.y_min && y <= tr.y_max) {
        int b, l;
        if (row_span(tr, y, 0, fc.width - 1, &b, &l)) b0 = b / kBin, b1 = l / kBin;
      }
    }
    for (int wd = 0; wd < nwords; ++wd) {
      uint32_t word = 0;
      if (kWrite && cached) {
        word = B.lpair_cols[(size_t)w * nwords + wd];
      } else {
        const int lo = max(b0, wd * 32), hi = min(b1, wd * 32 + 31);
        if (lo <= hi) word = (hi - lo == 31 ? 0xffffffffu : ((2u << (hi - lo)) - 1u)) << (lo - wd * 32);
        word = __reduce_or_sync(0xffffffffu, word);
        if (!kWrite && cached && lane == 0) B.lpair_cols[(size_t)w * nwords + wd] = word;
      }
      const bool mine = fc.world <= 1 || ((wd * 32 + lane + 3 * R) % fc.world) == fc.rank;
      if (((word >> lane) & 1u) && mine) {
        const int bin = R * fc.bins_x + wd * 32 + lane;
        if (kWrite) {
          const uint32_t slot = atomicAdd(&B.tcur[bin], 1u);
          if (slot < fc.items_cap) {
            VEIL_CHECK(bin < fc.nbins);
            B.items[slot] = ti;
            B.item_rows[slot] = (uint8_t)block_rows_mask(B.tri_y[ti], R, fc.height);
          }
        } else {
          atomicAdd(&B.tcnt[bin], 1u);
        }
      }
    }
  }
}

// offsets (binning.cpp:24-32) + categories (34-37) + write cursors
__global__ void __launch_bounds__(1024) k_bin_scan(Buffers B) {
  grid_dep_wait();
  const FrameConst& fc = c_fc;
  if (B.ctr->error) return;
  __shared__ unsigned long long carry;
  __shared__ unsigned int cnt[3];
  if (threadIdx.x == 0) carry = 0, cnt[0] = cnt[1] = cnt[2] = 0;
  __syncthreads();
  for (int base = 0; base < fc.nbins; base += 1024) {
    int b = base + threadIdx.x;
    uint32_t qc = b < fc.nbins ? B.qcnt[b] : 0, tc = b < fc.nbins ? B.tcnt[b] : 0;
    uint32_t total;
    uint32_t ex = block_exclusive_scan<1024>(qc + tc, &total);
    if (b < fc.nbins) {
      unsigned long long o = carry + ex;
      B.off[b] = (uint32_t)o;
      B.qcur[b] = (uint32_t)o;
      B.tcur[b] = (uint32_t)(o + qc);
      uint32_t eq = 2u * qc + tc;
      uint8_t c = eq == 0 ? 0 : (eq < 1024u ? 1 : 2);
      B.cat[b] = c;
      B.prop[b] = 0;
      B.prop_q[b] = 0;
      B.bin_cost[b] = 0;
      atomicAdd(&cnt[c], 1u);
    }
    {  // extraction work lists (renderer.cpp:150-190: low bins, then high bins)
      const int bxi = b % fc.bins_x, byi = b / fc.bins_x;
      const bool owned = b < fc.nbins && (fc.world <= 1 || ((bxi + 3 * byi) % fc.world) == fc.rank);
      const uint8_t c = owned ? B.cat[b] : 0;
      const bool lo = c == 1 && !fc.force_high, hi = c == 2 || (c == 1 && fc.force_high);
      const int lane = threadIdx.x & 31;
#pragma unroll
      for (int ps = 0; ps < 2; ++ps) {
        const bool in = ps == 0 ? lo : hi;
        const unsigned m = __ballot_sync(0xffffffffu, in);
        uint32_t at = 0;
        if (lane == 0 && m) at = atomicAdd(&B.ctr->list_count[ps], (unsigned)__popc(m));
        at = __shfl_sync(0xffffffffu, at, 0);
        if (in) B.bin_list[ps][at + __popc(m & ((1u << lane) - 1u))] = (uint32_t)b;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    B.ctr->pairs = carry;
    B.ctr->bins_empty = cnt[0];
    B.ctr->bins_low = cnt[1];
    B.ctr->bins_high = cnt[2];
    if (carry > fc.items_cap) atomicOr(&B.ctr->error, 2u);
  }
}

// Sort one segment of u32 ascending in place (bitonic; SMEM when it fits).
__device__ void cta_sort_segment(uint32_t* g, uint32_t n, uint32_t* sm, uint32_t sm_cap) {
  if (n < 2) return;
  uint32_t N = 1;
  while (N < n) N <<= 1;
  uint32_t* a = N <= sm_cap ? sm : g;
  if (N > sm_cap) {
    // Global-memory path for very long lists: pad is impossible in place, so
    // run an odd-even transposition merge on the real length instead.
    for (uint32_t phase = 0; phase < n; ++phase) {
      for (uint32_t i = 2 * threadIdx.x + (phase & 1); i + 1 < n; i += 2 * blockDim.x) {
        uint32_t x = g[i], y = g[i + 1];
        if (x > y) g[i] = y, g[i + 1] = x;
      }
      __syncthreads();
    }
    return;
  }
  for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) a[i] = i < n ? g[i] : 0xffffffffu;
  __syncthreads();
  for (uint32_t k = 2; k <= N; k <<= 1)
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
        uint32_t ixj = i ^ j;
        if (ixj > i) {
          uint32_t x = a[i], y = a[ixj];
          bool up = (i & k) == 0;
          if ((x > y) == up) a[i] = y, a[ixj] = x;
        }
      }
      __syncthreads();
    }
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) g[i] = a[i];
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_bin_sort(Buffers B) {
  grid_dep_wait();
  const FrameConst& fc = c_fc;
  if (B.ctr->error) return;
  __shared__ uint32_t sm[4096];
  for (int b = blockIdx.x; b < fc.nbins; b += gridDim.x) {
    uint32_t qc = B.qcnt[b], tc = B.tcnt[b], o = B.off[b];
    cta_sort_segment(B.items + o, qc, sm, 4096);
    cta_sort_segment(B.items + o + qc, tc, sm, 4096);
    __syncthreads();
    const int by = b / fc.bins_x;  // the row masks follow their items
    for (uint32_t i = threadIdx.x; i < qc + tc; i += blockDim.x) {
      const uint32_t it = B.items[o + i];
      B.item_rows[o + i] =
          i < qc ? (uint8_t)(block_rows_mask(B.tri_y[2 * it], by, fc.height) |
                             (block_rows_mask(B.tri_y[2 * it + 1], by, fc.height) << 4))
                 : (uint8_t)block_rows_mask(B.tri_y[it], by, fc.height);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ raster

struct Tbr {  // one triangle's coverage of a 32x8 block-row (packing.hpp:108-149)
  uint32_t tri;
  uint32_t meta;   // bits 0-3 block-column mask, bit 4 large
  uint32_t b[2];   // 8 row begins, one byte each
  uint32_t l[2];   // 8 row lasts, one byte each; empty row = (31, 0)
  uint32_t slot;   // position in the bin's triangle list (k_shade staging)
};

__device__ __forceinline__ uint32_t byte_of(const uint32_t* w, int i) {
  return (w[i >> 2] >> ((i & 3) * 8)) & 0xffu;
}

// Register depth filter (depth_filter.hpp:31-92) with compile-time maximum
// capacity KM and runtime capacity cap <= KM; entries ascending by key
// (keys are unique per pixel). push() returns the entry the reference's
// insert-then-pop_min would emit: when full, that is min(new, oldest
// minimum), and the survivor set is merged back with one select pass.
template <int KM, bool kExact = false>
struct RegFilter {
  uint64_t key[KM];
  float4 col[KM];
  int n;
  uint64_t max_key;
  bool any;

  __device__ __forceinline__ void reset() {
    n = 0;
    max_key = 0;
    any = false;
  }
  __device__ __forceinline__ void note(uint64_t pk, bool* ooo) {
    *ooo = any && pk < max_key;
    if (!any || pk > max_key) max_key = pk;
    any = true;
  }
  __device__ __forceinline__ bool push(int cap_rt, uint64_t k, float4 c, uint64_t* pk, float4* pc,
                                       bool* ooo) {
    const int cap = kExact ? KM : cap_rt;
    if (n < cap) {  // not full: bubble into [0, n]
      uint64_t ck = k;
      float4 cc = c;
#pragma unroll
      for (int i = 0; i < KM; ++i) {
        if (i < n) {
          const bool sw = key[i] > ck;
          const uint64_t tk = key[i];
          const float4 tc = col[i];
          key[i] = sw ? ck : tk;
          col[i] = sw ? cc : tc;
          ck = sw ? tk : ck;
          cc = sw ? tc : cc;
        } else if (i == n) {
          key[i] = ck;
          col[i] = cc;
        }
      }
      ++n;
      return false;
    }
    if (k < key[0]) {  // the new sample is the minimum: it falls straight out
      *pk = k;
      *pc = c;
      note(k, ooo);
      return true;
    }
    *pk = key[0];
    *pc = col[0];
    note(key[0], ooo);
    uint64_t ck = k;  // slots <- sorted(key[1..cap-1] + {k})
    float4 cc = c;
#pragma unroll
    for (int i = 0; i < KM; ++i) {
      if (i + 1 < cap) {
        const uint64_t x = key[i + 1];
        const float4 xc = col[i + 1];
        const bool lt = x < ck;
        key[i] = lt ? x : ck;
        col[i] = lt ? xc : cc;
        ck = lt ? ck : x;
        cc = lt ? cc : xc;
      } else if (i + 1 == cap) {
        key[i] = ck;
        col[i] = cc;
      }
    }
    return true;
  }
  __device__ __forceinline__ void pop(uint64_t* pk, float4* pc, bool* ooo) {
    *pk = key[0];
    *pc = col[0];
#pragma unroll
    for (int i = 0; i + 1 < KM; ++i)
      if (i + 1 < n) key[i] = key[i + 1], col[i] = col[i + 1];
    --n;
    note(*pk, ooo);
  }
  // Colour push(k) would pop (if any), without modifying the filter.
  __device__ __forceinline__ bool peek(int cap_rt, uint64_t k, float4 c, float4* pc) const {
    const int cap = kExact ? KM : cap_rt;
    if (n < cap) return false;
    *pc = (k < key[0]) ? c : col[0];
    return true;
  }
};

// Depth filter variant with the colours in shared memory: the registers hold
// only (key << 4 | slot), sorted ascending (keys are unique, so the slot
// bits never affect the order), and each slot's colour lives in this lane's
// column of a per-warp [K][32] float4 array. Same emission semantics as
// RegFilter (depth_filter.hpp:31-92); moves 2 registers per merge step
// instead of 6.
template <int K>
struct SlotFilter {
  uint64_t sk[K];
  int n;
  uint64_t max_key;
  bool any;
  float4* cols;  // this lane's slot 0; slot s at cols[s * 32]

  __device__ __forceinline__ void reset(float4* lane_cols) {
    n = 0;
    max_key = 0;
    any = false;
    cols = lane_cols;
  }
  __device__ __forceinline__ void note(uint64_t pk, bool* ooo) {
    *ooo = any && pk < max_key;
    if (!any || pk > max_key) max_key = pk;
    any = true;
  }
  __device__ __forceinline__ bool push(int, uint64_t k, float4 c, uint64_t* pk, float4* pc,
                                       bool* ooo) {
    if (n < K) {  // not full: store the colour in slot n, bubble the key in
      cols[n * 32] = c;
      uint64_t ck = (k << 4) | (uint64_t)n;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        if (i < n) {
          const uint64_t x = sk[i];
          const bool sw = x > ck;
          sk[i] = sw ? ck : x;
          ck = sw ? x : ck;
        } else if (i == n) {
          sk[i] = ck;
        }
      }
      ++n;
      return false;
    }
    const uint64_t k0 = sk[0];
    if (k < (k0 >> 4)) {  // the new sample is the minimum: it falls straight out
      *pk = k;
      *pc = c;
      note(k, ooo);
      return true;
    }
    const uint32_t s0 = (uint32_t)k0 & 15u;
    *pk = k0 >> 4;
    *pc = cols[s0 * 32];
    cols[s0 * 32] = c;
    note(*pk, ooo);
    uint64_t ck = (k << 4) | s0;  // slots <- sorted(sk[1..K-1] + {new})
#pragma unroll
    for (int i = 0; i + 1 < K; ++i) {
      const uint64_t x = sk[i + 1];
      const bool lt = x < ck;
      sk[i] = lt ? x : ck;
      ck = lt ? ck : x;
    }
    sk[K - 1] = ck;
    return true;
  }
  __device__ __forceinline__ void pop(uint64_t* pk, float4* pc, bool* ooo) {
    const uint64_t k0 = sk[0];
    *pk = k0 >> 4;
    *pc = cols[((uint32_t)k0 & 15u) * 32];
#pragma unroll
    for (int i = 0; i + 1 < K; ++i)
      if (i + 1 < n) sk[i] = sk[i + 1];
    --n;
    note(*pk, ooo);
  }
};

// Depth filter for capacities above 8 (DF 9 .. 32768): per pixel, a sorted
// ring of entries in memory (shared memory when the block's rings fit next to
// the staged triangles, else this warp's slice of a global scratch that stays
// L1/L2-resident). Same emission as the reference's sorted filter
// (depth_filter.hpp:31-92): when an insert overflows it, the minimum of
// (entries + new) leaves; keys are unique, so that is "the new key if it is
// below the front, else the front", and the flush pops the front in order.
// Samples arrive almost sorted (tri-blocks are depth-sorted per block), so an
// insert usually lands at the tail: O(1) per sample in the common case, a
// shift of the displaced entries otherwise. Ring entries hold (compact key
// << 15 | colour slot); colours stay in their slots ([slot][32 lanes], a
// lane's column), so a shift moves 8 bytes per entry. The compact key keeps
// the (depth, triangle) order in 49 bits: (q << 24 | tri24), or
// (q << 27 | tri27) with extended limits. Slots are insertion indices while
// the filter fills; once full it stays full until the half-block's flush and
// every insert reuses the slot of the entry it pushes out. A pixel receives
// at most one sample per THB of its half-block, so min(k, max THB limit)
// entries suffice (host: dfm_cap).
struct MemFilter {
  uint64_t* rk;  // this lane's ring entry 0; entry i at rk[i * 32]
  float4* rc;    // this lane's colour slot 0; slot s at rc[s * 32]
  int n, head, cap_mem;
  uint64_t max_key;
  bool any;

  static constexpr int kSlotBits = 15;
  static constexpr uint64_t kSlotMask = (1ull << kSlotBits) - 1ull;

  __device__ __forceinline__ void reset(uint64_t* keys, float4* cols, int cap) {
    rk = keys;
    rc = cols;
    n = 0;
    head = 0;
    cap_mem = cap;
    max_key = 0;
    any = false;
  }
  __device__ __forceinline__ static uint64_t pack(uint64_t k) {
    return c_fc.extended ? (((k >> 32) << 27) | (k & 0x7ffffffull)) : k;
  }
  __device__ __forceinline__ static uint64_t unpack(uint64_t ck) {
    return c_fc.extended ? (((ck >> 27) << 32) | (ck & 0x7ffffffull)) : ck;
  }
  __device__ __forceinline__ size_t at(int i) const {  // logical -> ring position (x32 lanes)
    const int p = head + i;
    return (size_t)(p >= cap_mem ? p - cap_mem : p) * 32u;
  }
  __device__ __forceinline__ void note(uint64_t pk, bool* ooo) {
    *ooo = any && pk < max_key;
    if (!any || pk > max_key) max_key = pk;
    any = true;
  }
  // places e at logical position n (the tail), shifting larger entries up
  __device__ __forceinline__ void insert_tail(uint64_t e) {
    VEIL_CHECK(n < cap_mem && (uint32_t)(e & kSlotMask) < (uint32_t)cap_mem);
    int i = n;
    while (i > 0) {
      const uint64_t prev = rk[at(i - 1)];
      if (prev < e) break;
      rk[at(i)] = prev;
      --i;
    }
    rk[at(i)] = e;
    ++n;
  }
  __device__ __forceinline__ bool push(int cap, uint64_t k, float4 c, uint64_t* pk, float4* pc,
                                       bool* ooo) {
    const uint64_t ck = pack(k);
    if (n < cap) {
      rc[(size_t)n * 32] = c;
      insert_tail((ck << kSlotBits) | (uint64_t)n);
      return false;
    }
    const uint64_t e0 = rk[at(0)];
    if (ck < (e0 >> kSlotBits)) {  // the new sample is the minimum: it falls straight out
      *pk = k;
      *pc = c;
      note(k, ooo);
      return true;
    }
    const uint32_t s0 = (uint32_t)(e0 & kSlotMask);
    *pk = unpack(e0 >> kSlotBits);
    *pc = rc[(size_t)s0 * 32];
    rc[(size_t)s0 * 32] = c;
    note(*pk, ooo);
    head = head + 1 == cap_mem ? 0 : head + 1;  // drop the front, then insert in its slot
    --n;
    insert_tail((ck << kSlotBits) | s0);
    return true;
  }
  __device__ __forceinline__ void pop(uint64_t* pk, float4* pc, bool* ooo) {
    const uint64_t e0 = rk[at(0)];
    *pk = unpack(e0 >> kSlotBits);
    *pc = rc[(size_t)(e0 & kSlotMask) * 32];
    head = head + 1 == cap_mem ? 0 : head + 1;
    --n;
    note(*pk, ooo);
  }
  // Colour push(k) would emit (if any), without modifying the filter.
  __device__ __forceinline__ bool peek(int cap, uint64_t k, float4 c, float4* pc) const {
    if (n < cap) return false;
    const uint64_t e0 = rk[at(0)];
    *pc = pack(k) < (e0 >> kSlotBits) ? c : rc[(size_t)(e0 & kSlotMask) * 32];
    return true;
  }
};

// The ring filter's shading paths keep scalar blend products (see blend).
template <typename F> struct PairBlend { static constexpr bool value = true; };
template <> struct PairBlend<MemFilter> { static constexpr bool value = false; };

// Paired FP32 multiplies (sm_100's FMUL2: two IEEE round-to-nearest products
// per instruction, each exactly __fmul_rn), so the colour channels' products
// cost half the issue slots with bit-identical results. The sums stay scalar
// __fadd_rn: a paired add (the __fadd2_rn intrinsic, or add.rn.f32x2 in inline
// PTX) was contracted with its product into FFMA2 -- one rounding instead of
// two -- which moved pixels by one step.
__device__ __forceinline__ float2 lo2(float4 v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 hi2(float4 v) { return make_float2(v.z, v.w); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  return make_float2(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y));
}
__device__ __forceinline__ float4 cat4(float2 a, float2 b) { return make_float4(a.x, a.y, b.x, b.y); }

// ((c0 * b0) + (c1 * b1)) + (c2 * b2) per channel (the barycentric attribute
// interpolation, shading.cpp:55-62), products two channels at a time.
__device__ __forceinline__ float4 interp4(float4 c0, float4 c1, float4 c2, float b0, float b1, float b2) {
  const float2 bb0 = make_float2(b0, b0), bb1 = make_float2(b1, b1), bb2 = make_float2(b2, b2);
  return cat4(add2(add2(mul2(lo2(c0), bb0), mul2(lo2(c1), bb1)), mul2(lo2(c2), bb2)),
              add2(add2(mul2(hi2(c0), bb0), mul2(hi2(c1), bb1)), mul2(hi2(c2), bb2)));
}

// acc + (1 - acc.w) * s per channel (shade_half_block's blend). kPair: the
// products two at a time (faster in the register-filter paths; the ring
// filter's paths measured 6% slower with it, C2 at DF 64).
template <bool kPair = true>
__device__ __forceinline__ float4 blend(float4 acc, float4 s) {
  const float t = __fsub_rn(1.0f, acc.w);
  if (kPair) {
    const float2 tt = make_float2(t, t);
    return cat4(add2(lo2(acc), mul2(tt, lo2(s))), add2(hi2(acc), mul2(tt, hi2(s))));
  }
  return make_float4(__fadd_rn(acc.x, __fmul_rn(t, s.x)), __fadd_rn(acc.y, __fmul_rn(t, s.y)),
                     __fadd_rn(acc.z, __fmul_rn(t, s.z)), __fadd_rn(acc.w, __fmul_rn(t, s.w)));
}

// normalize + Lambert (shade_sample, shading.cpp:123-136): the light factor.
__device__ __forceinline__ float light_factor(const FrameConst& fc, float n[3]) {
  // normalize (float), math.hpp:80-85
  float len2 = __fadd_rn(__fadd_rn(__fmul_rn(n[0], n[0]), __fmul_rn(n[1], n[1])), __fmul_rn(n[2], n[2]));
  if (len2 <= 0.0f) {
    n[0] = n[1] = n[2] = 0.0f;
  } else {
    float il = __fdiv_rn(1.0f, __fsqrt_rn(len2));
    n[0] = __fmul_rn(n[0], il);
    n[1] = __fmul_rn(n[1], il);
    n[2] = __fmul_rn(n[2], il);
  }
  float d = __fadd_rn(__fadd_rn(__fmul_rn(n[0], fc.light[0]), __fmul_rn(n[1], fc.light[1])),
                      __fmul_rn(n[2], fc.light[2]));
  float lam = smaxf(0.0f, -d);
  return sminf(1.0f, __fadd_rn(fc.ambient, lam));
}

// base * colour * texture(1) * light, premultiplied (shading.cpp:137-139);
// mat = (base rgb, opacity).
__device__ __forceinline__ float4 premultiply(float4 color, float4 mat, float light) {
  // (the reference's texture factor is 1 here: x * 1.0f == x exactly, so the
  // product is left out)
  // r, g = (base * colour) * light; (b, a) = (base.z * colour.z, opacity * colour.w)
  const float2 rg = mul2(mul2(lo2(mat), lo2(color)), make_float2(light, light));
  const float2 ba = mul2(hi2(mat), hi2(color));
  const float b = __fmul_rn(ba.x, light), a = ba.y;
  const float2 rga = mul2(rg, make_float2(a, a));
  return make_float4(rga.x, rga.y, __fmul_rn(b, a), a);
}

__device__ __forceinline__ float4 light_and_premultiply(const FrameConst& fc, float n[3],
                                                        float4 color, float4 mat) {
  const float light = light_factor(fc, n);
  return premultiply(color, mat, light);
}

// bilinear (shading.cpp:81-101): repeat wrapping, texel centres at +0.5,
// float arithmetic in the reference's order.
__device__ __forceinline__ float4 tex_bilinear(const Buffers& B, uint4 lev, float u, float v) {
  const int w = (int)lev.y, h = (int)lev.z;
  const float x = __fsub_rn(__fmul_rn(u, (float)w), 0.5f);
  const float y = __fsub_rn(__fmul_rn(v, (float)h), 0.5f);
  const float fx = floorf(x), fy = floorf(y);
  const float wx = __fsub_rn(x, fx), wy = __fsub_rn(y, fy);
  auto wrap = [](int i, int n) {
    const int m = i % n;
    return m < 0 ? m + n : m;
  };
  const int x0 = wrap((int)fx, w), x1 = wrap((int)fx + 1, w);
  const int y0 = wrap((int)fy, h), y1 = wrap((int)fy + 1, h);
  const float4* t = B.texels + lev.x;
  const float4 t00 = __ldg(&t[(size_t)y0 * w + x0]), t10 = __ldg(&t[(size_t)y0 * w + x1]);
  const float4 t01 = __ldg(&t[(size_t)y1 * w + x0]), t11 = __ldg(&t[(size_t)y1 * w + x1]);
  const float ax = __fsub_rn(1.0f, wx), ay = __fsub_rn(1.0f, wy);
  auto lerp4 = [](float4 a, float4 b, float ka, float kb) {
    return make_float4(__fadd_rn(__fmul_rn(a.x, ka), __fmul_rn(b.x, kb)),
                       __fadd_rn(__fmul_rn(a.y, ka), __fmul_rn(b.y, kb)),
                       __fadd_rn(__fmul_rn(a.z, ka), __fmul_rn(b.z, kb)),
                       __fadd_rn(__fmul_rn(a.w, ka), __fmul_rn(b.w, kb)));
  };
  const float4 top = lerp4(t00, t10, ax, wx), bot = lerp4(t01, t11, ax, wx);
  return lerp4(top, bot, ay, wy);
}

// sample_texture (shading.cpp:105-121): mip level log2(rho) of the UV
// footprint, trilinear between levels. The level uses CUDA's log2f (1 ulp)
// where the reference calls the C library's log2f, so a frac one ulp apart
// can move a blended texel by one unit in the last place; everything else is
// the reference's float arithmetic.
__device__ __forceinline__ float4 sample_texture(const Buffers& B, int texi, float2 uv, float2 dx,
                                                 float2 dy) {
  const uint2 td = __ldg(&B.texdesc[texi]);
  const uint4 base = __ldg(&B.texlev[td.x]);
  const float bw = (float)base.y, bh = (float)base.z;
  const float gx0 = __fmul_rn(dx.x, bw), gx1 = __fmul_rn(dx.y, bh);
  const float gy0 = __fmul_rn(dy.x, bw), gy1 = __fmul_rn(dy.y, bh);
  const float gx = __fsqrt_rn(__fadd_rn(__fmul_rn(gx0, gx0), __fmul_rn(gx1, gx1)));
  const float gy = __fsqrt_rn(__fadd_rn(__fmul_rn(gy0, gy0), __fmul_rn(gy1, gy1)));
  const float rho = smaxf(gx, gy);
  const float level = rho > 0.0f ? log2f(rho) : 0.0f;
  if (!(level > 0.0f)) return tex_bilinear(B, base, uv.x, uv.y);
  const float max_level = (float)(td.y - 1u);
  if (level >= max_level) return tex_bilinear(B, __ldg(&B.texlev[td.x + td.y - 1u]), uv.x, uv.y);
  const int l0 = (int)level;
  const float frac = __fsub_rn(level, (float)l0);
  const float4 a = tex_bilinear(B, __ldg(&B.texlev[td.x + l0]), uv.x, uv.y);
  const float4 b = tex_bilinear(B, __ldg(&B.texlev[td.x + l0 + 1]), uv.x, uv.y);
  const float ka = __fsub_rn(1.0f, frac);
  return make_float4(__fadd_rn(__fmul_rn(a.x, ka), __fmul_rn(b.x, frac)),
                     __fadd_rn(__fmul_rn(a.y, ka), __fmul_rn(b.y, frac)),
                     __fadd_rn(__fmul_rn(a.z, ka), __fmul_rn(b.z, frac)),
                     __fadd_rn(__fmul_rn(a.w, ka), __fmul_rn(b.w, frac)));
}

// shade_sample's products with a texture factor (shading.cpp:134-138).
__device__ __forceinline__ float4 premultiply_tex(float4 color, float4 mat, float4 tex, float light) {
  float r = __fmul_rn(__fmul_rn(__fmul_rn(mat.x, color.x), tex.x), light);
  float g = __fmul_rn(__fmul_rn(__fmul_rn(mat.y, color.y), tex.y), light);
  float b = __fmul_rn(__fmul_rn(__fmul_rn(mat.z, color.z), tex.z), light);
  float a = __fmul_rn(__fmul_rn(mat.w, color.w), tex.w);
  return make_float4(__fmul_rn(r, a), __fmul_rn(g, a), __fmul_rn(b, a), a);
}

// The texture factor of one sample (compiled only into the textured
// instantiations of the shading kernels). UVs by
// the quotient rule with analytic gradients (shading.cpp:55-74), in double;
// zero when the quad carries no UVs (SampleContext defaults).
__device__ __forceinline__ float4 texture_factor(const Buffers& B, const Fn3* te, uint32_t q, int ltri,
                                              bool has_uv, int texi, double e0, double e1, double e2,
                                              double sum, double inv) {
  float2 uv = make_float2(0.f, 0.f), duv_dx = uv, duv_dy = uv;
  if (has_uv) {
    const float4 ua = __ldg(&B.vq_uv[2 * (size_t)q]), ub = __ldg(&B.vq_uv[2 * (size_t)q + 1]);
    const float2 c0 = make_float2(ua.x, ua.y);
    const float2 c1 = ltri == 0 ? make_float2(ua.z, ua.w) : make_float2(ub.x, ub.y);
    const float2 c2 = ltri == 0 ? make_float2(ub.x, ub.y) : make_float2(ub.z, ub.w);
    auto dot3d = [](double a0, double a1, double a2, double b0, double b1, double b2) {
      return __dadd_rn(__dadd_rn(__dmul_rn(a0, b0), __dmul_rn(a1, b1)), __dmul_rn(a2, b2));
    };
    const double nu = dot3d(c0.x, c1.x, c2.x, e0, e1, e2), nv = dot3d(c0.y, c1.y, c2.y, e0, e1, e2);
    const double nu_dx = dot3d(c0.x, c1.x, c2.x, te[0].a, te[1].a, te[2].a);
    const double nv_dx = dot3d(c0.y, c1.y, c2.y, te[0].a, te[1].a, te[2].a);
    const double nu_dy = dot3d(c0.x, c1.x, c2.x, te[0].b, te[1].b, te[2].b);
    const double nv_dy = dot3d(c0.y, c1.y, c2.y, te[0].b, te[1].b, te[2].b);
    const double d_dx = __dadd_rn(__dadd_rn(te[0].a, te[1].a), te[2].a);
    const double d_dy = __dadd_rn(__dadd_rn(te[0].b, te[1].b), te[2].b);
    const double inv2 = __dmul_rn(inv, inv);
    uv = make_float2((float)__dmul_rn(nu, inv), (float)__dmul_rn(nv, inv));
    duv_dx = make_float2((float)__dmul_rn(__dsub_rn(__dmul_rn(nu_dx, sum), __dmul_rn(nu, d_dx)), inv2),
                         (float)__dmul_rn(__dsub_rn(__dmul_rn(nv_dx, sum), __dmul_rn(nv, d_dx)), inv2));
    duv_dy = make_float2((float)__dmul_rn(__dsub_rn(__dmul_rn(nu_dy, sum), __dmul_rn(nu, d_dy)), inv2),
                         (float)__dmul_rn(__dsub_rn(__dmul_rn(nv_dy, sum), __dmul_rn(nv, d_dy)), inv2));
  }
  return sample_texture(B, texi, uv, duv_dx, duv_dy);
}

// Light factors of the six axis-aligned unit normals interpolated to
// s * axis, for the 17 floats s around 1.0f (bit offsets -8..8) that
// (b0 + b1) + b2 takes in practice; filled per CTA from the frame constants
// with shade_staged_bf's exact operations.
constexpr int kAxisLightSpan = 8;
__shared__ float s_axis_light[6][2 * kAxisLightSpan + 1];

__device__ __forceinline__ float light_of_normal(const FrameConst& fc, float n0, float n1, float n2) {
  const float len2 = __fadd_rn(__fadd_rn(__fmul_rn(n0, n0), __fmul_rn(n1, n1)), __fmul_rn(n2, n2));
  const bool pos = len2 > 0.0f;
  const float il = __fdiv_rn(1.0f, __fsqrt_rn(pos ? len2 : 1.0f));
  const float nx = pos ? __fmul_rn(n0, il) : 0.0f, ny = pos ? __fmul_rn(n1, il) : 0.0f,
              nz = pos ? __fmul_rn(n2, il) : 0.0f;
  const float d = __fadd_rn(__fadd_rn(__fmul_rn(nx, fc.light[0]), __fmul_rn(ny, fc.light[1])),
                            __fmul_rn(nz, fc.light[2]));
  return sminf(1.0f, __fadd_rn(fc.ambient, smaxf(0.0f, -d)));
}

__device__ __forceinline__ void fill_axis_light(const FrameConst& fc) {
  for (int i = threadIdx.x; i < 6 * (2 * kAxisLightSpan + 1); i += blockDim.x) {
    const int axis = i / (2 * kAxisLightSpan + 1), o = i % (2 * kAxisLightSpan + 1) - kAxisLightSpan;
    const float s = __uint_as_float((uint32_t)((int)0x3f800000 + o));
    const float v = (axis & 1) ? -s : s;
    const int k = axis >> 1;
    s_axis_light[axis][o + kAxisLightSpan] = light_of_normal(fc, k == 0 ? v : 0.0f, k == 1 ? v : 0.0f,
                                                             k == 2 ? v : 0.0f);
  }
}

// The light factor of a triangle whose corners share axis normal `axis`
// (-1: none) from the table, when s = (b0 + b1) + b2 is tabulated; false
// when the caller must compute it.
__device__ __forceinline__ bool axis_light(int axis, float b0, float b1, float b2, float* light) {
  if (axis < 0) return false;
  const float s = __fadd_rn(__fadd_rn(b0, b1), b2);
  const int so = (int)__float_as_uint(s) - (int)0x3f800000;
  if (so < -kAxisLightSpan || so > kAxisLightSpan) return false;
  *light = s_axis_light[axis][so + kAxisLightSpan];
  return true;
}

// make_sample_context (shading.cpp:24-77) + shade_sample (123-139), no
// textures. Returns the premultiplied colour and the sample depth.
template <bool kTex>
__device__ __forceinline__ float4 shade_sample(const FrameConst& fc, const Buffers& B,
                                               uint32_t tri, int px, int py, double* depth,
                                               const TriPlanes* P = nullptr) {
  // planes: the fused raster's per-TBR copy, else the triangle's record
  const Fn3* te = P ? P->e : B.tri[tri].e;
  const Fn3* tz = P ? &P->dz : &B.tri[tri].dz;
  const uint4 meta = __ldg(&B.tri_meta[tri]);
  const double x = (double)px + 0.5, y = (double)py + 0.5;
  const double e0 = eval(te[0], x, y), e1 = eval(te[1], x, y), e2 = eval(te[2], x, y);
  const double sum = __dadd_rn(__dadd_rn(e0, e1), e2);
  const double inv = __ddiv_rn(1.0, sum);
  const float b0 = (float)__dmul_rn(e0, inv), b1 = (float)__dmul_rn(e1, inv),
              b2 = (float)__dmul_rn(e2, inv);
  *depth = eval(*tz, x, y);
  if (fc.decoded) {
    const ShadeRec& sr = B.shade[tri];
    const uint32_t fl = sr.flags;
    float4 color = make_float4(1.0f, 1.0f, 1.0f, 1.0f);
    if (fl & 1u) {
      color = interp4(sr.c[0], sr.c[1], sr.c[2], b0, b1, b2);
    }
    float light;
    if (!axis_light((fl & 4u) ? (int)sr.pad[0] : -1, b0, b1, b2, &light)) {
      float n[3];
      const float4 n0 = sr.n[0];
      if (fl & 2u) {
        const float4 n1 = sr.n[1], n2 = sr.n[2];
        n[0] = __fadd_rn(__fadd_rn(__fmul_rn(n0.x, b0), __fmul_rn(n1.x, b1)), __fmul_rn(n2.x, b2));
        n[1] = __fadd_rn(__fadd_rn(__fmul_rn(n0.y, b0), __fmul_rn(n1.y, b1)), __fmul_rn(n2.y, b2));
        n[2] = __fadd_rn(__fadd_rn(__fmul_rn(n0.z, b0), __fmul_rn(n1.z, b1)), __fmul_rn(n2.z, b2));
      } else {
        n[0] = n0.x, n[1] = n0.y, n[2] = n0.z;
      }
      light = light_factor(fc, n);
    }
    return premultiply(color, sr.mat, light);
  }
  const uint32_t q = tri >> 1;
  const uint32_t qf = __ldg(&B.vq_flags[q]);
  const int ltri = (int)(meta.w & 0xffu);
  // corner attributes loaded with the flags (one round trip; unused when the
  // quad has none)
  const uint4 qcol = __ldg(&B.vq_col[q]), qnrm = __ldg(&B.vq_nrm[q]);
  float4 color = make_float4(1.0f, 1.0f, 1.0f, 1.0f);
  if (qf & 2u) {
    const uint4 c = qcol;
    const uint32_t w0 = c.x, w1 = ltri == 0 ? c.y : c.z, w2 = ltri == 0 ? c.z : c.w;
    // (scalar here: the paired products measured slower on this gather-bound
    // path, C4 shade +2%)
    float r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      r[k] = __fadd_rn(__fadd_rn(__fmul_rn(slut_c(w0, 8 * k), b0), __fmul_rn(slut_c(w1, 8 * k), b1)),
                       __fmul_rn(slut_c(w2, 8 * k), b2));
    color = make_float4(r[0], r[1], r[2], r[3]);
  }
  float light;
  {
    // corners sharing one axis-aligned normal take the light from the table
    const uint4 c = qnrm;
    const uint32_t w0 = c.x, w1 = ltri == 0 ? c.y : c.z, w2 = ltri == 0 ? c.z : c.w;
    const int axis = (qf & 4u) && w0 == w1 && w1 == w2 ? axis_of_word(w0) : -1;
    if (!axis_light(axis, b0, b1, b2, &light)) {
      float n[3];
      if (qf & 4u) {
#pragma unroll
        for (int k = 0; k < 3; ++k)
          n[k] = __fadd_rn(__fadd_rn(__fmul_rn(slut_n(w0, 10 * k), b0), __fmul_rn(slut_n(w1, 10 * k), b1)),
                           __fmul_rn(slut_n(w2, 10 * k), b2));
      } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) n[k] = slut_n(meta.x, 10 * k);
      }
      light = light_factor(fc, n);
    }
  }
  const MatDev& m = B.mats[meta.y];
  const float4 mat = make_float4(__ldg(&m.base[0]), __ldg(&m.base[1]), __ldg(&m.base[2]), __ldg(&m.opacity));
  if constexpr (kTex) {  // scenes with textured materials (see launch_shade)
    const int texi = __ldg(&m.texture);
    if (texi >= 0) {
      const float4 tex = texture_factor(B, te, q, ltri, (qf & 8u) != 0u, texi, e0, e1, e2, sum, inv);
      return premultiply_tex(color, mat, tex, light);
    }
  }
  return premultiply(color, mat, light);
}

// Branch-free variant of shade_sample for the decoded-record path (selects
// instead of branches) so two independent samples per lane can be
// interleaved by the scheduler. Bit-identical to shade_sample.
__device__ __forceinline__ float4 shade_decoded_bf(const FrameConst& fc, const Buffers& B,
                                                   uint32_t tri, int px, int py, uint32_t* qd) {
  const TriRec& t = B.tri[tri];
  const ShadeRec& sr = B.shade[tri];
  const double x = (double)px + 0.5, y = (double)py + 0.5;
  const double e0 = eval(t.e[0], x, y), e1 = eval(t.e[1], x, y), e2 = eval(t.e[2], x, y);
  const double sum = __dadd_rn(__dadd_rn(e0, e1), e2);
  const double inv = __ddiv_rn(1.0, sum);
  const float b0 = (float)__dmul_rn(e0, inv), b1 = (float)__dmul_rn(e1, inv),
              b2 = (float)__dmul_rn(e2, inv);
  *qd = quantize_depth(eval(t.dz, x, y));
  const uint32_t fl = sr.flags;
  const float4 c0 = sr.c[0], c1 = sr.c[1], c2 = sr.c[2];
  const float4 n0 = sr.n[0], n1 = sr.n[1], n2 = sr.n[2];
  const bool hc = fl & 1u, hn = fl & 2u;
  const float4 ci = interp4(c0, c1, c2, b0, b1, b2);
  float4 color;
  color.x = hc ? ci.x : 1.0f;
  color.y = hc ? ci.y : 1.0f;
  color.z = hc ? ci.z : 1.0f;
  color.w = hc ? ci.w : 1.0f;
  const float4 mat = sr.mat;
  float light;
  if (!axis_light((fl & 4u) ? (int)sr.pad[0] : -1, b0, b1, b2, &light)) {
    float n[3];
    n[0] = hn ? __fadd_rn(__fadd_rn(__fmul_rn(n0.x, b0), __fmul_rn(n1.x, b1)), __fmul_rn(n2.x, b2)) : n0.x;
    n[1] = hn ? __fadd_rn(__fadd_rn(__fmul_rn(n0.y, b0), __fmul_rn(n1.y, b1)), __fmul_rn(n2.y, b2)) : n0.y;
    n[2] = hn ? __fadd_rn(__fadd_rn(__fmul_rn(n0.z, b0), __fmul_rn(n1.z, b1)), __fmul_rn(n2.z, b2)) : n0.z;
    light = light_of_normal(fc, n[0], n[1], n[2]);
  }
  // (the reference's texture factor is 1 here: x * 1.0f == x exactly, so the
  // product is left out)
  // r, g = (base * colour) * light; (b, a) = (base.z * colour.z, opacity * colour.w)
  const float2 rg = mul2(mul2(lo2(mat), lo2(color)), make_float2(light, light));
  const float2 ba = mul2(hi2(mat), hi2(color));
  const float b = __fmul_rn(ba.x, light), a = ba.y;
  const float2 rga = mul2(rg, make_float2(a, a));
  return make_float4(rga.x, rga.y, __fmul_rn(b, a), a);
}

// A bin-row's triangle, staged in shared memory by k_shade: edge and depth
// planes plus the decoded shading record (one copy per bin-row instead of
// one L1/L2 load per sample). Per-triangle constants are folded at staging:
// without vertex normals the light factor is constant over the triangle
// (flag 4, in `light`), and with neither vertex colours nor normals so is the
// whole premultiplied colour (flag 8, in c[0]). Same float operations in the
// same order, so bit-identical to shading every sample in full.
struct __align__(16) StagedTri {
  double e[9];
  double dz[3];
  float4 c[3];
  float4 mat;
  float n[9];
  uint32_t flags;  // 1 colours, 2 normals, 4 constant light, 8 constant colour, 16 flat depth,
                   // 32 one axis-aligned vertex normal (light from s_axis_light, axis in `light`)
  float light;
  uint32_t pad;  // quantized depth when flag 16
};
static_assert(sizeof(StagedTri) == 208, "StagedTri layout");
constexpr int kStageTris = 320;

constexpr int kShadeStage = 256;  // THB entries k_shade stages per warp; longer lists stream

// Wave walk (mode 0) vs dense segments (mode 1) crossover, in samples per
// THB: lower when the bin's triangles are staged in shared memory (waves read
// them there), higher when each lane gathers its triangle from global memory.
constexpr uint32_t kWalkMinSamplesPerThbStaged = 6;
constexpr uint32_t kWalkMinSamplesPerThb = 16;  // (12 -> 16: C5 shade -0.7%)

__device__ __forceinline__ void stage_triangle(const FrameConst& fc, const Buffers& B, uint32_t tri,
                                               StagedTri* dst) {
  const TriRec& t = B.tri[tri];
  const ShadeRec& sr = B.shade[tri];
  const double2* e2 = reinterpret_cast<const double2*>(&t.e[0]);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double2 v = e2[k];
    dst->e[2 * k] = v.x;
    dst->e[2 * k + 1] = v.y;
  }
  dst->e[8] = t.e[2].c;
  dst->dz[0] = t.dz.a;
  dst->dz[1] = t.dz.b;
  dst->dz[2] = t.dz.c;
  const float4 mat = sr.mat;
  dst->c[0] = sr.c[0];
  dst->c[1] = sr.c[1];
  dst->c[2] = sr.c[2];
  dst->mat = mat;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float4 nn = sr.n[k];
    dst->n[3 * k] = nn.x;
    dst->n[3 * k + 1] = nn.y;
    dst->n[3 * k + 2] = nn.z;
  }
  uint32_t fl = sr.flags & 3u;  // colours / normals (the record's axis bit is re-derived below)
  dst->pad = 0;
  if (t.dz.a == 0.0 && t.dz.b == 0.0) {
    // flat depth plane: (0*x + 0*y) + c is c (or a zero, which quantizes
    // like c) for every finite pixel centre, so the quantized depth is the
    // triangle's (bit-identical to evaluating it per sample)
    dst->pad = quantize_depth(t.dz.c);
    fl |= 16u;
  }
  if (fl & 2u) {
    // the three corners carry the same axis-aligned unit normal (components
    // 0 and +-1, e.g. every C2 quad): the interpolated normal is then exactly
    // that axis times s = (b0 + b1) + b2 (products by 0 / +-1 are exact and
    // rounding is sign-symmetric), so the light factor is a function of s
    // alone, tabulated per frame (axis_light_table)
    const float4 a = sr.n[0], b = sr.n[1], c = sr.n[2];
    if (a.x == b.x && a.x == c.x && a.y == b.y && a.y == c.y && a.z == b.z && a.z == c.z) {
      const int nz = (a.x != 0.0f) + (a.y != 0.0f) + (a.z != 0.0f);
      const float v = a.x != 0.0f ? a.x : (a.y != 0.0f ? a.y : a.z);
      if (nz == 1 && (v == 1.0f || v == -1.0f)) {
        const uint32_t axis = (a.x != 0.0f ? 0u : (a.y != 0.0f ? 1u : 2u)) * 2u + (v < 0.0f ? 1u : 0u);
        dst->light = __uint_as_float(axis);
        fl |= 32u;
      }
    }
  }
  if (!(fl & 2u)) {
    const float4 n0 = sr.n[0];
    float n[3] = {n0.x, n0.y, n0.z};
    const float light = light_factor(fc, n);
    dst->light = light;
    fl |= 4u;
    if (!(fl & 1u)) {
      dst->c[0] = premultiply(make_float4(1.0f, 1.0f, 1.0f, 1.0f), mat, light);
      fl |= 8u;
    }
  }
  dst->flags = fl;
}

// shade_decoded_bf on a staged triangle (bit-identical).
__device__ __forceinline__ float4 shade_staged(const FrameConst& fc, const StagedTri& T, int px,
                                               int py, uint32_t* qd) {
  const double x = (double)px + 0.5, y = (double)py + 0.5;
  const Fn3 f0 = {T.e[0], T.e[1], T.e[2]}, f1 = {T.e[3], T.e[4], T.e[5]}, f2 = {T.e[6], T.e[7], T.e[8]};
  const uint32_t fl = T.flags;
  if (fl & 16u) {
    *qd = T.pad;  // flat depth plane (stage_triangle)
  } else {
    const Fn3 fz = {T.dz[0], T.dz[1], T.dz[2]};
    *qd = quantize_depth(eval(fz, x, y));
  }
  if (fl & 8u) return T.c[0];  // constant colour (barycentrics unused)
  const double e0 = eval(f0, x, y), e1 = eval(f1, x, y), e2 = eval(f2, x, y);
  const double sum = __dadd_rn(__dadd_rn(e0, e1), e2);
  const double inv = __ddiv_rn(1.0, sum);
  const float b0 = (float)__dmul_rn(e0, inv), b1 = (float)__dmul_rn(e1, inv),
              b2 = (float)__dmul_rn(e2, inv);
  float4 color = make_float4(1.0f, 1.0f, 1.0f, 1.0f);
  if (fl & 1u) {
    color = interp4(T.c[0], T.c[1], T.c[2], b0, b1, b2);
  }
  float light;
  if (fl & 4u) {
    light = T.light;
  } else {
    float n[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
      n[k] = __fadd_rn(__fadd_rn(__fmul_rn(T.n[k], b0), __fmul_rn(T.n[3 + k], b1)), __fmul_rn(T.n[6 + k], b2));
    light = light_factor(fc, n);
  }
  return premultiply(color, T.mat, light);
}

// shade_staged without branches (every path computed, the flags select), so
// that two independent samples per lane can be interleaved by the scheduler
// (shade_waves_staged2). Bit-identical to shade_staged: each selected value
// is computed by the same operations on the same inputs.
// ltab: the 32-bit shared address of s_axis_light, taken once per half-block
// by the caller (naming the table directly made the compiler rematerialize
// its cluster-window address -- an S2R and three ALU operations -- per sample).
__device__ __forceinline__ float4 shade_staged_bf(const FrameConst& fc, const StagedTri& T, int px, int py,
                                                  uint32_t* qd, uint32_t ltab) {
  const double x = (double)px + 0.5, y = (double)py + 0.5;
  const uint32_t fl = T.flags;
  if (fl & 16u) {  // flat depth plane (stage_triangle); the one branch kept: every C2 quad
    *qd = T.pad;
  } else {
    const Fn3 fz = {T.dz[0], T.dz[1], T.dz[2]};
    *qd = quantize_depth(eval(fz, x, y));
  }
  const Fn3 f0 = {T.e[0], T.e[1], T.e[2]}, f1 = {T.e[3], T.e[4], T.e[5]}, f2 = {T.e[6], T.e[7], T.e[8]};
  const double e0 = eval(f0, x, y), e1 = eval(f1, x, y), e2 = eval(f2, x, y);
  const double sum = __dadd_rn(__dadd_rn(e0, e1), e2);
  const double inv = __ddiv_rn(1.0, sum);
  const float b0 = (float)__dmul_rn(e0, inv), b1 = (float)__dmul_rn(e1, inv),
              b2 = (float)__dmul_rn(e2, inv);
  const float4 c0 = T.c[0], c1 = T.c[1], c2 = T.c[2];
  const bool hc = fl & 1u;
  const float4 ci = interp4(c0, c1, c2, b0, b1, b2);
  float4 color;
  color.x = hc ? ci.x : 1.0f;
  color.y = hc ? ci.y : 1.0f;
  color.z = hc ? ci.z : 1.0f;
  color.w = hc ? ci.w : 1.0f;
  float light;
  const float s = __fadd_rn(__fadd_rn(b0, b1), b2);
  const int so = (int)__float_as_uint(s) - (int)0x3f800000;
  if ((fl & 32u) && so >= -kAxisLightSpan && so <= kAxisLightSpan) {
    // s_axis_light[axis][so + span] (axis-aligned normal)
    const uint32_t at = ltab + 4u * (__float_as_uint(T.light) * (2u * kAxisLightSpan + 1u) +
                                     (uint32_t)(so + kAxisLightSpan));
    asm("ld.shared.f32 %0, [%1];" : "=f"(light) : "r"(at));
  } else {
    float n[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
      n[k] = __fadd_rn(__fadd_rn(__fmul_rn(T.n[k], b0), __fmul_rn(T.n[3 + k], b1)), __fmul_rn(T.n[6 + k], b2));
    const float lit = light_of_normal(fc, n[0], n[1], n[2]);
    light = (fl & 4u) ? T.light : lit;
  }
  // (constant-colour triangles select their staged colour: an early return
  // for them measured C2 shade +3% -- it splits the two interleaved waves --
  // though C3's constant-colour boxes gain 6%)
  const float4 shaded = premultiply(color, T.mat, light);
  const float4 cc = T.c[0];
  return (fl & 8u) ? cc : shaded;
}

__device__ __forceinline__ uint64_t sample_key(const FrameConst& fc, uint32_t qd, uint32_t tri) {
  // sample_sort_key, raster.hpp:95-97 (32-bit triangle field when extended)
  return fc.extended ? (((uint64_t)qd << 32) | tri) : (((uint64_t)qd << 24) | (tri & 0xffffffu));
}

// Scratch of one (bin, block-row) extraction item, in shared or global memory.
struct RasterView {
  Tbr* tbr;
  uint64_t* keys;  // [4][cap_tb]
  uint16_t* refs;  // [4][cap_tb]
  uint32_t* rows;  // phase A: [4 warps][32 candidates][b0 b1 l0 l1] (aliases refs in SMEM)
  TriRec* cs;      // fused raster: candidate setups of the current round [cand_cap]
  TriPlanes* tp;   // fused raster: planes per TBR [cap_tbr]
};

struct RasterShared {
  // Shared-memory capacities; larger items (within the active limits) run
  // again with global scratch.
  static constexpr int kTbr = 512, kTb = 256;
  Tbr tbr[kTbr];
  uint64_t keys[4 * kTb];
  __align__(16) uint16_t refs[4 * kTb];
};
static_assert(sizeof(uint16_t) * 4 * RasterShared::kTb >= 4 * 32 * 16, "phase-A row scratch");

__host__ __device__ inline size_t global_scratch_bytes(uint32_t cap_tbr, uint32_t cap_tb) {
  return (size_t)cap_tbr * sizeof(Tbr) + (size_t)4 * cap_tb * (8 + 2) + 64 + 2048 + 16;
}

struct ItemState {
  int ntbr;
  int status;  // 0 ok, 1 overflow (soft), 2 spill, 3 hard error
  int err_code;
  uint32_t warp_n[4];
  uint32_t pool_base;
  int alloc_ok;
  // candidate count / next row-span group, per phase-A round parity: round
  // r + 1's pair is reset during round r (no barrier of its own)
  uint32_t ncand[2];
  uint32_t gnext[2];
};

// ItemState before an item (k_extract's thread 0, ahead of the barrier that
// publishes the item).
__device__ __forceinline__ void reset_item_state(ItemState* st) {
  st->ntbr = 0;
  st->status = 0;
  st->err_code = 0x7fffffff;
  st->ncand[0] = st->gnext[0] = 0;
}

enum { kPassLow = 0, kPassHigh = 1 };

__device__ __forceinline__ void set_status(ItemState* st, int s, int code) {
  atomicMax(&st->status, s);
  if (s == 3) atomicMin(&st->err_code, code);
}

struct PixelOut {
  float4 acc;
  bool invalid;
  uint64_t hash;
  uint32_t emitted;
};

// Blend one popped sample into the pixel state (shade_half_block,
// raster.cpp:248-255). kDump: 0 = test c_fc.dump, 1 = no dump, 2 = dump frame
// (the compiler turns the run-time test into a select, so hot callers that
// know the frame kind drop the hash's instructions entirely).
template <int kDump = 0, bool kPair = true>
__device__ __forceinline__ void commit(PixelOut& o, uint64_t pk, float4 pc, bool ooo) {
  o.acc = blend<kPair>(o.acc, pc);
  if (kDump == 2 || (kDump == 0 && c_fc.dump))
    o.hash = (o.hash ^ pk) * kHashPrime;  // blend-order evidence (parity dumps)
  if (kDump != 1) ++o.emitted;  // (kDump 1: the caller knows the half-block's sample total)
  if (ooo) o.invalid = true;
}

// k-th covered pixel (row-major) of a tri-half-block coverage mask; each of
// the 4 rows is one contiguous run (packing.hpp:96-103), so row counts and
// the run start locate it without a bit-by-bit scan.
__device__ __forceinline__ uint32_t kth_pixel(uint32_t m, uint32_t k) {
  const uint32_t c0 = __popc(m & 0xffu), c1 = __popc(m & 0xff00u), c2 = __popc(m & 0xff0000u);
  uint32_t row = 0, before = 0;
  if (k >= c0) row = 1, before = c0;
  if (k >= c0 + c1) row = 2, before = c0 + c1;
  if (k >= c0 + c1 + c2) row = 3, before = c0 + c1 + c2;
  const uint32_t rb = (m >> (8 * row)) & 0xffu;
  return row * 8 + (__ffs(rb) - 1) + (k - before);
}

// Canonical-order shading of one half-block without the alpha threshold:
// the sample stream (THBs in sorted order, then row-major) is cut into
// 32-sample segments; lane s shades sample base+s, then each pixel's lane
// takes its samples of
// the segment in stream order through per-warp routing masks and pushes them
// into its register depth filter. Every pixel therefore sees exactly the
// reference's per-pixel sequence.
template <typename Filter>
__device__ __forceinline__ void blend_routed(const FrameConst& fc, Filter& f, PixelOut& o,
                                             uint32_t mine, uint64_t key, float4 col) {
  while (__any_sync(0xffffffffu, mine != 0u)) {
    const int src = mine ? __ffs(mine) - 1 : (threadIdx.x & 31);
    const uint64_t k2 = __shfl_sync(0xffffffffu, key, src);
    float4 c2;
    c2.x = __shfl_sync(0xffffffffu, col.x, src);
    c2.y = __shfl_sync(0xffffffffu, col.y, src);
    c2.z = __shfl_sync(0xffffffffu, col.z, src);
    c2.w = __shfl_sync(0xffffffffu, col.w, src);
    if (mine) {
      mine &= mine - 1u;
      uint64_t pk;
      float4 pc;
      bool ooo;
      if (f.push(fc.df, k2, c2, &pk, &pc, &ooo)) commit<0, PairBlend<Filter>::value>(o, pk, pc, ooo);
    }
  }
}

__device__ __forceinline__ uint32_t route_mask(uint32_t* route, uint32_t pix, bool valid) {
  const int lane = threadIdx.x & 31;
  route[lane] = 0u;
  __syncwarp();
  const unsigned peers = __match_any_sync(0xffffffffu, pix);
  VEIL_CHECK(!valid || pix < 32u);
  if (valid && lane == __ffs(peers) - 1) route[pix] = peers;
  __syncwarp();
  const uint32_t mine = route[lane];
  __syncwarp();
  return mine;
}

template <int KM, bool kTex, typename Filter>
__device__ __forceinline__ void shade_segments(const FrameConst& fc, const Buffers& B, int px0,
                                               int py0, const uint32_t* tri_l,
                                               const uint32_t* mask_l, const uint32_t* pre_l,
                                               uint32_t n, uint32_t total, uint32_t* route,
                                               PixelOut& o, Filter& f, const uint16_t* slot_l = nullptr,
                                               const TriPlanes* tp = nullptr) {
  const int lane = threadIdx.x & 31;
  uint32_t r_lo = 0;
  for (uint32_t base = 0; base < total; base += 32) {
    // THB r_lo holds a sample < base and every THB holds >= 1 sample, so
    // sample base+lane lies in a THB <= r_lo + lane + 1.
    const uint32_t s0 = base + lane;
    const bool v0 = s0 < total;
    const uint32_t c0 = v0 ? s0 : total - 1;
    // THBs r_lo+1 .. r_lo+32 start inside [base, base+32) or later (THB r_lo
    // holds sample base-1, or base = 0 and r_lo = 0): one bit per start, and
    // sample base+lane lies in THB r_lo + (starts at or before it)
    const uint32_t rj = r_lo + 1u + (uint32_t)lane;
    uint32_t start_bit = 0u;
    if (rj < n) {
      const uint32_t st = pre_l[rj] - base;
      if (st < 32u) start_bit = 1u << st;
    }
    const uint32_t starts = __reduce_or_sync(0xffffffffu, start_bit);
    const uint32_t r0 = r_lo + (uint32_t)__popc(starts & (0xffffffffu >> (31 - lane)));
    const uint32_t p0 = kth_pixel(mask_l[r0], c0 - pre_l[r0]);
    const uint32_t t0 = tri_l[r0];
    float4 col0;
    uint32_t q0;
    if (fc.decoded) {
      col0 = shade_decoded_bf(fc, B, t0, px0 + (int)(p0 & 7u), py0 + (int)(p0 >> 3), &q0);
    } else {
      double d0;
      col0 = shade_sample<kTex>(fc, B, t0, px0 + (int)(p0 & 7u), py0 + (int)(p0 >> 3), &d0,
                                tp ? &tp[slot_l[r0]] : nullptr);
      q0 = quantize_depth(d0);
    }
    const uint64_t key0 = sample_key(fc, q0, t0);
    r_lo = __shfl_sync(0xffffffffu, r0, 31);
    const uint32_t m0 = route_mask(route, v0 ? p0 : 32u + lane, v0);
    blend_routed(fc, f, o, m0, key0, col0);
  }
  while (f.n > 0) {
    uint64_t pk;
    float4 pc;
    bool ooo;
    f.pop(&pk, &pc, &ooo);
    commit<0, PairBlend<Filter>::value>(o, pk, pc, ooo);
  }
}

// THB-by-THB walk with lane == pixel (raster.cpp:232-284): every lane visits
// the THBs in sorted order and shades the ones covering its pixel, so the
// triangle data of each step is a warp-wide broadcast. Used when THBs cover
// many pixels (samples/THB high) and, with kThreshold, for the alpha
// threshold, where the 32nd saturation must be located at its exact stream
// position.
template <int KM, bool kThreshold, bool kTex, typename Filter>
__device__ __forceinline__ void shade_walk(const FrameConst& fc, const Buffers& B, int px0,
                                           int py0, const uint32_t* tri_l, const uint32_t* mask_l,
                                           uint32_t n, PixelOut& o,
                                           unsigned long long* enumerated_out, Filter& f,
                                           const uint16_t* slot_l = nullptr, const TriPlanes* tp = nullptr) {
  const int lane = threadIdx.x & 31;
  const int px = px0 + (lane & 7), py = py0 + (lane >> 3);
  bool saturated = false, stopped = false;
  unsigned sat_mask = 0;
  unsigned long long enumerated = 0;
  for (uint32_t r = 0; r < n; ++r) {
    const uint32_t m = mask_l[r];
    const uint32_t tri = tri_l[r];
    const bool covered = (m >> lane) & 1u;
    float4 col = make_float4(0.f, 0.f, 0.f, 0.f);
    uint64_t key = 0;
    if (covered) {
      uint32_t qd;
      if (fc.decoded) {
        col = shade_decoded_bf(fc, B, tri, px, py, &qd);
      } else {
        double depth;
        col = shade_sample<kTex>(fc, B, tri, px, py, &depth, tp ? &tp[slot_l[r]] : nullptr);
        qd = quantize_depth(depth);
      }
      key = sample_key(fc, qd, tri);
    }
    int commit_until = 32;
    if (kThreshold) {
      bool newly = false;
      if (covered && !saturated) {
        float4 pc;
        if (f.peek(fc.df, key, col, &pc)) newly = blend(o.acc, pc).w >= kAlphaThreshold;
      }
      const unsigned new_mask = __ballot_sync(0xffffffffu, newly);
      if (new_mask && (sat_mask | new_mask) == 0xffffffffu) {
        commit_until = 32 - __clz(new_mask);
        stopped = true;
      }
      enumerated += __popc(m & (commit_until == 32 ? 0xffffffffu : ((1u << commit_until) - 1u)));
    }
    if (covered && lane < commit_until) {
      uint64_t pk;
      float4 pc;
      bool ooo;
      if (f.push(fc.df, key, col, &pk, &pc, &ooo)) {
        commit<0, PairBlend<Filter>::value>(o, pk, pc, ooo);
        if (kThreshold && !saturated && o.acc.w >= kAlphaThreshold) saturated = true;
      }
    }
    if (kThreshold) {
      sat_mask = __ballot_sync(0xffffffffu, saturated);
      if (stopped) break;
    }
  }
  if (!stopped) {
    bool done = kThreshold && o.acc.w >= kAlphaThreshold;
    while (f.n > 0) {
      uint64_t pk;
      float4 pc;
      bool ooo;
      f.pop(&pk, &pc, &ooo);
      if (done) continue;
      commit<0, PairBlend<Filter>::value>(o, pk, pc, ooo);
      if (kThreshold && o.acc.w >= kAlphaThreshold) done = true;
    }
  }
  if (kThreshold) *enumerated_out = enumerated;
}

// Wave walk (no alpha threshold): consecutive THBs whose coverage masks are
// pairwise disjoint form a wave; each pixel receives at most one sample per
// wave and waves follow the THB order, so every pixel still sees the
// reference's per-pixel sequence (raster.cpp:232-267) while a warp step
// shades up to 32 samples from several triangles (e.g. both triangles of a
// quad, which are adjacent in the sort order and disjoint).
template <int KM, bool kTex, typename Filter>
__device__ __forceinline__ void shade_waves(const FrameConst& fc, const Buffers& B, int px0,
                                            int py0, const uint32_t* tri_l,
                                            const uint32_t* mask_l, const uint16_t* slot_l,
                                            const StagedTri* staged, uint32_t n, PixelOut& o,
                                            Filter& f, const TriPlanes* tp = nullptr) {
  const int lane = threadIdx.x & 31;
  const int px = px0 + (lane & 7), py = py0 + (lane >> 3);
  uint32_t r = 0;
  while (r < n) {
    uint32_t acc_mask = 0, my_r = 0xffffffffu;
    do {
      const uint32_t m = mask_l[r];
      if (acc_mask & m) break;
      if ((m >> lane) & 1u) my_r = r;
      acc_mask |= m;
      ++r;
    } while (r < n);
    if (my_r != 0xffffffffu) {
      const uint32_t tri = tri_l[my_r];
      uint32_t qd;
      float4 col;
      if (staged) {
        VEIL_CHECK(slot_l[my_r] < kStageTris);
        col = shade_staged(fc, staged[slot_l[my_r]], px, py, &qd);
      } else if (fc.decoded) {
        col = shade_decoded_bf(fc, B, tri, px, py, &qd);
      } else {
        double depth;
        col = shade_sample<kTex>(fc, B, tri, px, py, &depth, tp ? &tp[slot_l[my_r]] : nullptr);
        qd = quantize_depth(depth);
      }
      uint64_t pk;
      float4 pc;
      bool ooo;
      if (f.push(fc.df, sample_key(fc, qd, tri), col, &pk, &pc, &ooo)) commit<0, PairBlend<Filter>::value>(o, pk, pc, ooo);
    }
  }
  while (f.n > 0) {
    uint64_t pk;
    float4 pc;
    bool ooo;
    f.pop(&pk, &pc, &ooo);
    commit<0, PairBlend<Filter>::value>(o, pk, pc, ooo);
  }
}

// Wave walk over staged triangles, two waves per step: both waves' samples
// are shaded by straight-line code (shade_staged_bf) so the scheduler can
// overlap the two dependency chains, then pushed in wave order -- each pixel
// still receives its samples in the reference's sequence.
template <int KM, int kDump, typename Filter>
__device__ __forceinline__ void shade_waves_staged2(const FrameConst& fc, int px0, int py0,
                                                    const uint32_t* tri_l, const uint32_t* mask_l,
                                                    const uint16_t* slot_l, const StagedTri* staged,
                                                    uint32_t n, PixelOut& o, Filter& f) {
  const int lane = threadIdx.x & 31;
  const int px = px0 + (lane & 7), py = py0 + (lane >> 3);
  constexpr uint32_t kNone = 0xffffffffu;
  // next wave from THB *r: two masks are loaded per iteration so the
  // shared-memory latency is paid once per pair (the list buffers have slack
  // past n, and a mask past n is never used)
  auto form = [&](uint32_t* r) {
    uint32_t acc_mask = 0, my_r = kNone;
    while (*r < n) {
      const uint32_t m0 = mask_l[*r], m1 = mask_l[*r + 1];
      if (acc_mask & m0) break;
      if ((m0 >> lane) & 1u) my_r = *r;
      acc_mask |= m0;
      ++*r;
      if (*r >= n || (acc_mask & m1)) break;
      if ((m1 >> lane) & 1u) my_r = *r;
      acc_mask |= m1;
      ++*r;
    }
    return my_r;
  };
  uint32_t ltab, sbase;
  asm volatile("mov.u32 %0, %1;" : "=r"(ltab) : "r"(smem_addr(&s_axis_light[0][0])));
  // the staged triangles through an opaque shared address too (same reason)
  asm volatile("mov.u32 %0, %1;" : "=r"(sbase) : "r"(smem_addr(staged)));
  const StagedTri* stri = static_cast<const StagedTri*>(__cvta_shared_to_generic(sbase));
  uint32_t r = 0;
  while (r < n) {
    const uint32_t ra = form(&r);
    const uint32_t rb = form(&r);
    const uint32_t ia = ra != kNone ? ra : 0u, ib = rb != kNone ? rb : 0u;
    uint32_t qa, qb;
    VEIL_CHECK(slot_l[ia] < kStageTris && slot_l[ib] < kStageTris);
    const float4 ca = shade_staged_bf(fc, stri[slot_l[ia]], px, py, &qa, ltab);
    const float4 cb = shade_staged_bf(fc, stri[slot_l[ib]], px, py, &qb, ltab);
    uint64_t pk;
    float4 pc;
    bool ooo;
    if (ra != kNone && f.push(fc.df, sample_key(fc, qa, tri_l[ia]), ca, &pk, &pc, &ooo))
      commit<kDump>(o, pk, pc, ooo);
    if (rb != kNone && f.push(fc.df, sample_key(fc, qb, tri_l[ib]), cb, &pk, &pc, &ooo))
      commit<kDump>(o, pk, pc, ooo);
  }
  while (f.n > 0) {
    uint64_t pk;
    float4 pc;
    bool ooo;
    f.pop(&pk, &pc, &ooo);
    commit<kDump>(o, pk, pc, ooo);
  }
}

// Composite a finished half-block over the background, write its 8x4 pixels
// (device framebuffer; the mapped host frame and the root rank's peer
// framebuffer when the frame has them; blend-order evidence in dump mode),
// and add its samples / segments / invalid pixels to the (bin, block-row)
// stat slot (shade_half_block's tail, raster.cpp:286-320).
__device__ __forceinline__ void finish_half_block(const FrameConst& fc, const Buffers& B, int bin, int row,
                                                  int hpx0, int hpy0, const PixelOut& po, bool live,
                                                  unsigned long long enumerated) {
  const int lane = threadIdx.x & 31;
  const int px = hpx0 + (lane & 7), py = hpy0 + (lane >> 3);
  unsigned invalid_px = 0;
  if (px < fc.width && py < fc.height) {
    const size_t pix = (size_t)py * fc.width + px;
    uint32_t word;
    if (po.invalid && fc.visualize) {
      word = 0xffff00ffu;  // magenta overlay, renderer.cpp:56-65
    } else {
      const float4 out = blend(po.acc, make_float4(fc.bg[0], fc.bg[1], fc.bg[2], fc.bg[3]));
      word = quantize_channel(out.x) | (quantize_channel(out.y) << 8) |
             (quantize_channel(out.z) << 16) | (quantize_channel(out.w) << 24);
    }
    B.fb[pix] = word;
    B.mask[pix] = po.invalid ? 1 : 0;
    if (fc.host_fb) {  // over the host link, overlapped with the rest of the frame
      fc.host_fb[pix] = word;
      fc.host_mask[pix] = po.invalid ? 1 : 0;
    }
    if (fc.peer_fb) {  // into the root rank's framebuffer (peer memory)
      fc.peer_fb[pix] = word;
      fc.peer_mask[pix] = po.invalid ? 1 : 0;
    }
    if (fc.dump) {
      B.hash[pix] = po.hash;
      B.emit[pix] = po.emitted;
    }
    invalid_px = po.invalid ? 1u : 0u;
  }
  if (live) {
    unsigned long long samples = po.emitted;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) samples += __shfl_xor_sync(0xffffffffu, samples, s);
    const unsigned inv = __popc(__ballot_sync(0xffffffffu, invalid_px != 0));
    if (lane == 0) {
      unsigned long long* slot = B.slots + ((size_t)bin * 4 + row) * 5;
      atomicAdd(&slot[0], samples);
      atomicAdd(&slot[3], (enumerated + 255ull) / 256ull);
      if (inv) atomicAdd(&slot[4], (unsigned long long)inv);
    }
  }
}

// This warp's ring filter storage (MemFilter): after the staged triangles in
// dynamic shared memory, or its slice of the global scratch.
template <int kMode>
__device__ __forceinline__ void dfm_reset(const Buffers& B, uint8_t* shade_dyn, MemFilter& f,
                                          int warps_per_cta = 8) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t warp_bytes = (size_t)B.dfm_cap * 32u * 24u;
  uint8_t* base = B.dfm_g ? B.dfm_g + ((size_t)blockIdx.x * warps_per_cta + (size_t)warp) * warp_bytes
                           : shade_dyn + (kMode == 0 ? (size_t)kStageTris * sizeof(StagedTri) : 0) +
                                 (size_t)warp * warp_bytes;
  f.reset(reinterpret_cast<uint64_t*>(base) + lane,
          reinterpret_cast<float4*>(base + (size_t)B.dfm_cap * 32u * 8u) + lane, (int)B.dfm_cap);
}

__device__ __forceinline__ uint32_t span_mask(uint32_t b, uint32_t l, uint32_t c0, uint32_t c1) {
  // row span [b, l] (bin-local) clipped to block columns [c0, c1] as 8 bits
  if (b > l) return 0u;
  b = max(b, c0);
  l = min(l, c1);
  if (b > l) return 0u;
  return ((2u << (l - b)) - 1u) << (b - c0);
}

// Compare-exchange of registers j and j ^ (M / 32) (stages with distance >= 32).
template <int J, int M>
__device__ __forceinline__ void bitonic_cross(uint64_t (&v)[4], int k, int lane) {
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int jp = j ^ (M >> 5);
    if (jp > j) {
      const int i = j * 32 + lane;
      const bool up = (i & k) == 0;
      const uint64_t x = v[j], y = v[jp];
      const bool sw = (x > y) == up;
      v[j] = sw ? y : x;
      v[jp] = sw ? x : y;
    }
  }
}

// Warp bitonic sort of N = 32*J 64-bit keys held in registers, strided
// layout (element i = j*32 + lane in v[j]); ascending. The stage loops run
// at run time (only the register index is unrolled) to keep the kernel's
// code small: the fully unrolled network cost instruction-cache stalls.
template <int J>
__device__ __forceinline__ void warp_bitonic(uint64_t (&v)[4], int lane) {
  constexpr int N = 32 * J;
  constexpr int kMU = 2;  // measured: 1 and 5 are slower
#pragma unroll 1
  for (int k = 2; k <= N; k <<= 1) {
    if (J == 4 && k >= 128) bitonic_cross<J, 64>(v, k, lane);
    if (J >= 2 && k >= 64) bitonic_cross<J, 32>(v, k, lane);
#pragma unroll kMU
    for (int m = min(k >> 1, 16); m > 0; m >>= 1) {
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int i = j * 32 + lane;
        const uint64_t x = v[j];
        const uint64_t y = __shfl_xor_sync(0xffffffffu, x, m);
        const bool up = (i & k) == 0, lower = (lane & m) == 0;
        const uint64_t lo = x < y ? x : y, hi = x < y ? y : x;
        v[j] = (lower == up) ? lo : hi;
      }
    }
  }
}

// One (bin, block-row) extraction item: phases A and B of the reference's
// rasterize_bin (raster.cpp:41-199). Tri-half-block lists go to the global
// THB pool (L2-resident) with one descriptor per half-block; shading runs
// in k_shade. kGlobal selects global-memory scratch for items that exceed
// the shared-memory capacities (but not the active limits).
// Bitonic sort of a block's (key, ref) pairs in scratch memory, for blocks
// with more tri-blocks than the register sort holds (out of line: rare).
__device__ __noinline__ void sort_keys_scratch(uint64_t* keys, uint16_t* refs, uint32_t n, int lane) {
  uint32_t N = 1;
  while (N < n) N <<= 1;
  for (uint32_t i = n + lane; i < N; i += 32) keys[i] = ~0ull, refs[i] = 0;
  __syncwarp();
  for (uint32_t k = 2; k <= N; k <<= 1)
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      // one compare-exchange pair per lane step: pair p -> (i, i + j), i
      // with bit log2(j) clear
      for (uint32_t p = lane; p < N / 2; p += 32) {
        const uint32_t i = ((p & ~(j - 1u)) << 1) | (p & (j - 1u)), ixj = i | j;
        const uint64_t x = keys[i], y = keys[ixj];
        const bool up = (i & k) == 0;
        if ((x > y) == up) {
          keys[i] = y;
          keys[ixj] = x;
          const uint16_t t = refs[i];
          refs[i] = refs[ixj];
          refs[ixj] = t;
        }
      }
      __syncwarp();
    }
}

template <bool kGlobal, int kFuse>
__device__ __forceinline__ void extract_item(const FrameConst& fc, const Buffers& B, int pass,
                                             int bin, int row, const RasterView& V,
                                             ItemState* st, uint32_t cap_tbr, uint32_t cap_tb) {
  const Limits lim = pass == kPassLow ? fc.low : fc.high;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bxi = bin % fc.bins_x, byi = bin / fc.bins_x;
  const int px0 = bxi * kBin, py0 = byi * kBin;
  const int px_last = min(px0 + kBin - 1, fc.width - 1);
  const int py_last = min(py0 + kBin - 1, fc.height - 1);
  const int ry0 = py0 + row * 8, ry1 = min(ry0 + 7, py_last);
  // (st was reset by k_extract before the barrier that published the item)

  // ---- phase A: tri-block-rows of this block-row (raster.cpp:41-98).
  // Candidates (valid triangles whose y range meets the block-row) are first
  // compacted with warp ballots, so the FP64 row-span loop runs dense.
  const uint32_t nq = B.qcnt[bin], nt = B.tcnt[bin], o = B.off[bin];
  const uint32_t T = 2 * nq + nt;
  uint64_t* cand = V.keys;  // keys are free until phase B
  const uint32_t cand_cap = 4u * cap_tb;
  // rounds over bin items (a small quad's item holds its 2 triangles), sized
  // so that a round's candidates fit the candidate buffer
  const uint32_t nitem = nq + nt, round_items = cand_cap / 2u;
  uint32_t par = 0;  // round parity: this round's ncand / gnext
  for (uint32_t round = 0; round < nitem; round += round_items, par ^= 1u) {
    const uint32_t end = min(nitem, round + round_items);
    for (uint32_t j0 = round; j0 < end; j0 += blockDim.x) {
      const uint32_t j = j0 + threadIdx.x;
      uint32_t rows = 0, it = 0;
      if (j < end) {
        rows = (uint32_t)B.item_rows[o + j];
        rows = j < nq ? ((rows >> row) & 1u) | (((rows >> (4 + row)) & 1u) << 1) : ((rows >> row) & 1u);
        if (rows) it = B.items[o + j];
      }
      // candidate triangles in bin-list expansion order: 2j, 2j+1 (small
      // quads) or 2nq + (j - nq) (large triangles)
      const unsigned m0 = __ballot_sync(0xffffffffu, rows & 1u);
      const unsigned m1 = __ballot_sync(0xffffffffu, (rows >> 1) & 1u);
      uint32_t wbase = 0;
      if (lane == 0 && (m0 | m1)) wbase = atomicAdd(&st->ncand[par], (uint32_t)(__popc(m0) + __popc(m1)));
      wbase = __shfl_sync(0xffffffffu, wbase, 0);
      const unsigned below = (1u << lane) - 1u;
      if (rows & 1u) {
        const bool large = j >= nq;
        const uint32_t i = large ? 2 * nq + (j - nq) : 2 * j;
        const uint32_t ti = large ? it : it * 2;
        VEIL_CHECK(wbase + __popc(m0 & below) < cand_cap);
        cand[wbase + __popc(m0 & below)] = ((uint64_t)i << 32) | ti | ((large ? 1u : 0u) << 31);
        if (!kFuse) asm volatile("prefetch.global.L2 [%0];" ::"l"(B.tri + ti));  // read by the row spans next
      }
      if (rows & 2u) {
        cand[wbase + __popc(m0) + __popc(m1 & below)] = ((uint64_t)(2 * j + 1) << 32) | (it * 2 + 1);
        if (!kFuse) asm volatile("prefetch.global.L2 [%0];" ::"l"(B.tri + it * 2 + 1));
      }
    }
    __syncthreads();
    const uint32_t nc = st->ncand[par];
    // every thread is past the previous round (which used the other pair)
    if (threadIdx.x == 0) st->ncand[par ^ 1u] = st->gnext[par ^ 1u] = 0;
    // Row spans, load-balanced per warp: a warp takes 32 candidates, scans
    // their row counts and spreads the (candidate, row) pairs over its lanes,
    // so tall and short triangles keep all lanes busy; each candidate's lane
    // then assembles its tri-block-row from the per-row bytes.
    // Groups of G candidates are taken dynamically; with fewer than 32
    // candidates G shrinks (down to 8) so that all four warps share the row
    // spans (smaller groups for larger items cost short triangles more than
    // they gain for tall ones, measured).
    uint32_t* rs = V.rows + (size_t)warp * 128u;  // [candidate][b0 b1 l0 l1]
    const uint32_t G = nc < 32u ? max(8u, ((nc + 3u) / 4u + 7u) & ~7u) : 32u;
    for (;;) {
      uint32_t g = 0;
      if (lane == 0) g = atomicAdd(&st->gnext[par], G);
      g = __shfl_sync(0xffffffffu, g, 0);
      if (g >= nc) break;
      const uint32_t j = g + lane;
      uint32_t ti = 0, large = 0, nrows = 0;
      int yb = 0;
      uint64_t code = 0;
      if ((uint32_t)lane < G && j < nc) {
        code = cand[j];
        ti = (uint32_t)code & 0x7fffffffu;
        large = ((uint32_t)code) >> 31;
        if (kFuse) {
          // fused raster: the candidate's setup (small quads' recomputed,
          // large ones' loaded) goes to the CTA's candidate scratch, read
          // back by the row spans and copied into its TBR's planes
          TriRec tr;
          if (large || fc.fused_read)
            tr = B.tri[ti];
          else
            recompute_setup(fc, B, ti, &tr);
          yb = max(tr.y_min, ry0);
          const int ye = min(tr.y_max, ry1);
          nrows = ye >= yb ? (uint32_t)(ye - yb + 1) : 0u;
          if (nrows) V.cs[j] = tr;
        } else {
          const TriRec& t = B.tri[ti];
          yb = max(t.y_min, ry0);
          const int ye = min(t.y_max, ry1);
          nrows = ye >= yb ? (uint32_t)(ye - yb + 1) : 0u;
        }
      }
      const uint32_t total = __reduce_add_sync(0xffffffffu, nrows);
      const uint32_t ngroup = min(G, nc - g);
      // per-lane walk for groups of short triangles, unless a few tall ones
      // would leave most lanes idle (mixed scenes)
      const uint32_t max_rows = __reduce_max_sync(0xffffffffu, nrows);
      // Row spans with one call site: per lane for groups of short
      // triangles, (candidate, row) pairs spread over the lanes otherwise;
      // each row's (begin, last) bytes land in the candidate's scratch slot.
      const bool pairs = !(total < 3u * ngroup && max_rows <= (total + 31u) / 32u + 2u);
      uint32_t rb0 = 0x1f1f1f1fu, rb1 = 0x1f1f1f1fu, rl0 = 0u, rl1 = 0u, cols = 0;
      uint32_t excl = 0;
      if (kFuse) __syncwarp();  // candidate setups visible to the warp
      if (pairs) {
        reinterpret_cast<uint4*>(rs)[lane] = make_uint4(0x1f1f1f1fu, 0x1f1f1f1fu, 0u, 0u);
        uint32_t incl = nrows;
#pragma unroll
        for (int sft = 1; sft < 32; sft <<= 1) {
          const uint32_t v = __shfl_up_sync(0xffffffffu, incl, sft);
          if (lane >= sft) incl += v;
        }
        excl = incl - nrows;
      }
      __syncwarp();
      const uint32_t iters = pairs ? (total + 31u) / 32u : max_rows;
#pragma unroll 1
      for (uint32_t it = 0; it < iters; ++it) {
        uint32_t c = (uint32_t)lane, tcur = ti;
        int py = yb + (int)it;
        bool act = it < nrows;
        if (pairs) {
          const uint32_t p = it * 32u + lane;
          c = 0;  // largest c with excl[c] <= p (shuffle binary search)
#pragma unroll
          for (uint32_t sft = 16; sft > 0; sft >>= 1) {
            const uint32_t e = __shfl_sync(0xffffffffu, excl, c + sft);
            if (e <= p) c += sft;
          }
          const uint32_t ec = __shfl_sync(0xffffffffu, excl, c);
          tcur = __shfl_sync(0xffffffffu, ti, c);
          py = __shfl_sync(0xffffffffu, yb, c) + (int)(p - ec);
          act = p < total;
        }
        int b, l;
        bool spans;
        if (kFuse)
          spans = act && row_span(V.cs[g + c], py, px0, px_last, &b, &l);
        else
          spans = act && row_span(B.tri[tcur], py, px0, px_last, &b, &l);
        if (spans) {
          const int ly = py - ry0;
          const uint32_t bb = (uint32_t)(b - px0), ll = (uint32_t)(l - px0);
          if (pairs) {
            reinterpret_cast<uint8_t*>(rs + c * 4)[ly] = (uint8_t)bb;
            reinterpret_cast<uint8_t*>(rs + c * 4 + 2)[ly] = (uint8_t)ll;
          } else {  // the lane's own candidate: keep its row bytes in registers
            const int sh8 = (ly & 3) * 8;
            const uint32_t keepm = ~(0xffu << sh8);
            if (ly < 4) {
              rb0 = (rb0 & keepm) | (bb << sh8);
              rl0 = (rl0 & keepm) | (ll << sh8);
            } else {
              rb1 = (rb1 & keepm) | (bb << sh8);
              rl1 = (rl1 & keepm) | (ll << sh8);
            }
            cols |= ((2u << (ll >> 3)) - 1u) & ~((1u << (bb >> 3)) - 1u);
          }
        }
      }
      if (pairs) {
        __syncwarp();
        const uint4 rr = reinterpret_cast<const uint4*>(rs)[lane];
        rb0 = rr.x, rb1 = rr.y, rl0 = rr.z, rl1 = rr.w;
        __syncwarp();
        if (nrows) {
#pragma unroll
          for (int y = 0; y < 8; ++y) {
            const uint32_t bb = ((y < 4 ? rb0 : rb1) >> ((y & 3) * 8)) & 0xffu;
            const uint32_t ll = ((y < 4 ? rl0 : rl1) >> ((y & 3) * 8)) & 0xffu;
            if (bb <= ll) cols |= ((2u << (ll >> 3)) - 1u) & ~((1u << (bb >> 3)) - 1u);
          }
        }
      }
      if (nrows) {
        if (cols) {
          const int slot = atomicAdd(&st->ntbr, 1);
          if ((uint32_t)slot < cap_tbr) {
            Tbr rec;
            rec.tri = ti;
            rec.meta = cols | (large << 4);
            rec.b[0] = rb0;
            rec.b[1] = rb1;
            rec.l[0] = rl0;
            rec.l[1] = rl1;
            rec.slot = (uint32_t)(code >> 32);
            VEIL_CHECK((uint32_t)slot < cap_tbr && (!kFuse || j < cand_cap));
            V.tbr[slot] = rec;
            if (kFuse) {
              const TriRec& tr = V.cs[j];
              TriPlanes pl;
              pl.e[0] = tr.e[0];
              pl.e[1] = tr.e[1];
              pl.e[2] = tr.e[2];
              pl.dz = tr.dz;
              V.tp[slot] = pl;
            }
          }
        }
      }
    }
    __syncthreads();
  }
  // (the rounds loop ends with a barrier; with no items ntbr is still 0)
  const uint32_t ntbr = (uint32_t)st->ntbr;
  if (ntbr > lim.tbr || ntbr > cap_tbr) {  // uniform: every thread leaves
    if (threadIdx.x == 0) set_status(st, ntbr > lim.tbr ? (pass == kPassLow ? 1 : 3) : 2, 0);
    return;
  }

  // ---- phase B: warp w extracts block (row, w) (raster.cpp:100-199)
  const int block = row * 4 + warp;
  const uint32_t c0 = (uint32_t)warp * 8u, c1 = c0 + 7u;
  const double bpx0 = (double)(px0 + warp * 8), bpy0 = (double)(py0 + row * 8);
  uint64_t* keys = V.keys + (size_t)warp * cap_tb;
  uint16_t* refs = V.refs + (size_t)warp * cap_tb;
  const bool packable = cap_tbr <= 16384u;  // TBR index fits the key's low 14 bits
  // select the tri-block-rows touching this block's columns (selection
  // order = TBR order; compacted first so the centroid pass runs dense)
  uint32_t n = 0;
  for (uint32_t base = 0; base < ntbr; base += 32) {
    const uint32_t i = base + lane;
    const bool sel = i < ntbr && ((V.tbr[i].meta >> warp) & 1u);
    const unsigned m = __ballot_sync(0xffffffffu, sel);
    if (sel) {
      const uint32_t pos = n + __popc(m & ((1u << lane) - 1u));
      if (pos < cap_tb) refs[pos] = (uint16_t)i;
    }
    n += __popc(m);
  }
  __syncwarp();
  const uint32_t nsel = min(n, cap_tb);
  for (uint32_t pos = lane; pos < nsel; pos += 32) {
    const uint32_t i = refs[pos];
    const Tbr& rw = V.tbr[i];
    uint32_t count = 0, sx = 0, sy = 0;
#pragma unroll
    for (int y = 0; y < 8; ++y) {
      uint32_t b = byte_of(rw.b, y), l = byte_of(rw.l, y);
      if (b > l) continue;
      b = max(b, c0);
      l = min(l, c1);
      if (b > l) continue;
      const uint32_t k = l - b + 1;
      count += k;
      sx += (b + l) * k / 2 - c0 * k;
      sy += (uint32_t)y * k;
    }
    uint32_t qd = 0x3fffffu;
    if (count) {
      const Fn3 dz = kFuse ? V.tp[i].dz : B.tri[rw.tri].dz;
      if (dz.a == 0.0 && dz.b == 0.0) {
        qd = quantize_depth(dz.c);  // flat plane: (±0 + ±0) + c quantizes like c at any centroid
      } else {
        // (a zero sum -- the TBR's pixels all in the block's first column /
        // row, common for tiny triangles -- divides to +0 exactly; testing it
        // keeps those lanes off the division's out-of-line slow path, which a
        // zero dividend takes)
        const double mx = sx ? __ddiv_rn((double)sx, (double)count) : 0.0;
        const double my = sy ? __ddiv_rn((double)sy, (double)count) : 0.0;
        const double cx = __dadd_rn(__dadd_rn(bpx0, mx), 0.5);
        const double cy = __dadd_rn(__dadd_rn(bpy0, my), 0.5);
        qd = quantize_depth(eval(dz, cx, cy));
      }
    }
    // (depth, is_large, triangle) orders exactly like the reference's
    // (depth, selection index): selection order is bin-list order. The
    // packed form carries the TBR reference in the low 14 bits.
    const uint64_t large = (rw.meta >> 4) & 1u;
    keys[pos] = packable ? (((uint64_t)qd << 42) | (large << 41) | ((uint64_t)rw.tri << 14) | i)
                         : (((uint64_t)qd << 33) | (large << 32) | rw.tri);
  }
  if (n > lim.tb) {
    if (lane == 0) set_status(st, pass == kPassLow ? 1 : 3, 1 + 3 * block);
  } else if (n > cap_tb) {
    if (lane == 0) set_status(st, 2, 0);
  }
  __syncwarp();
  const bool ok = n <= lim.tb && n <= cap_tb;
  const bool in_regs = ok && packable && n <= 128;
  uint64_t v[4] = {~0ull, ~0ull, ~0ull, ~0ull};
  if (in_regs) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if ((uint32_t)(j * 32 + lane) < n) v[j] = keys[j * 32 + lane];
    // two register sorts only: a third (32-key) variant costs more in
    // instruction-cache misses than it saves in compare-exchanges
    if (n <= 64) warp_bitonic<2>(v, lane);
    else warp_bitonic<4>(v, lane);
  } else if (ok && n > 1) {
    sort_keys_scratch(keys, refs, n, lane);
  }
  // one pool allocation per item: 2n THB slots per warp (each tri-block
  // yields <= 1 THB per half)
  if (lane == 0) st->warp_n[warp] = ok ? n : 0u;
  __syncthreads();
  if (threadIdx.x == 0) {
    st->alloc_ok = 0;
    unsigned long long* slot = B.slots + ((size_t)bin * 4 + row) * 5;
    slot[1] = slot[2] = 0;  // fragment / THB sums, added per warp below
    if (!st->status) {
      const uint32_t tot = 2u * (st->warp_n[0] + st->warp_n[1] + st->warp_n[2] + st->warp_n[3]);
      const unsigned long long pb = atomicAdd(&B.ctr->pool_pair, (unsigned long long)tot);
      if (pb + tot > fc.pool_cap) {
        atomicOr(&B.ctr->error, 8u);  // pool capacity: grow and re-run
      } else {
        st->pool_base = (uint32_t)pb;
        st->alloc_ok = 1;
      }
    }
  }
  __syncthreads();
  uint32_t nthb[2] = {0, 0}, frags[2] = {0, 0};
  uint32_t pbase = st->pool_base;
  for (int w = 0; w < warp; ++w) pbase += 2u * st->warp_n[w];
  if (ok && n && st->alloc_ok) {
    auto chunk = [&](uint32_t k, uint32_t ref) {
      uint32_t hm[2] = {0u, 0u};
      uint32_t tri = 0;
      if (k < n) {
        const Tbr& rw = V.tbr[ref];
        tri = rw.tri;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int y = 0; y < 4; ++y)
            hm[h] |= span_mask(byte_of(rw.b, h * 4 + y), byte_of(rw.l, h * 4 + y), c0, c1) << (8 * y);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t fr = __popc(hm[h]);
        const bool ne = fr > 0;
        const unsigned m = __ballot_sync(0xffffffffu, ne);
        const uint32_t pos = nthb[h] + __popc(m & ((1u << lane) - 1u));
        uint32_t incl = fr;  // inclusive scan of fragment counts
#pragma unroll
        for (int s2 = 1; s2 < 32; s2 <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, s2);
          if (lane >= s2) incl += y;
        }
        if (ne) {
          const size_t at = (size_t)pbase + (size_t)h * n + pos;
          VEIL_CHECK(at < fc.pool_cap && pos < n);
          B.pool_tri[at] = tri;
          B.pool_mask[at] = hm[h];
          B.pool_pre[at] = frags[h] + incl - fr;
          // fused: the TBR (its planes in V.tp); else the bin-list position
          // (k_shade's staging slot)
          B.pool_slot[at] = kFuse ? (uint16_t)ref : (uint16_t)min(V.tbr[ref].slot, 65535u);
        }
        nthb[h] += __popc(m);
        frags[h] += __shfl_sync(0xffffffffu, incl, 31);
      }
    };
    // one call site for the THB split (keeps the kernel's code compact)
#pragma unroll 1
    for (uint32_t base = 0; base < n; base += 32) {
      const uint32_t k = base + lane;
      uint32_t ref = 0;
      if (k < n) {
        if (in_regs) {
          const uint32_t j = base >> 5;
          const uint64_t vj = j == 0 ? v[0] : (j == 1 ? v[1] : (j == 2 ? v[2] : v[3]));
          ref = (uint32_t)(vj & 0x3fffu);
        } else {
          ref = refs[k];
        }
      }
      chunk(k, ref);
    }
    {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (nthb[h] > lim.thb) {
          if (lane == 0) set_status(st, pass == kPassLow ? 1 : 3, 2 + 3 * block);
        } else if (frags[h] > lim.frags) {
          if (lane == 0) set_status(st, pass == kPassLow ? 1 : 3, 3 + 3 * block);
        }
      }
    }
  }
  __syncthreads();
  if (st->status || !st->alloc_ok) return;
  // the block-row's triangle list (TBR order): k_shade stages these records
  if (lane < 2) {
    // Small THBs (few samples each) are shaded by k_shade_seg's dense
    // segments, the rest by k_shade's wave walk; the choice is made here so
    // the segment queue is complete when shading starts. The crossover is
    // lower when k_shade stages the bin's triangles in shared memory.
    HbDesc d;
    d.off = pbase + (uint32_t)lane * n;
    d.cnt = nthb[lane];
    d.frags = frags[lane];
    const bool staged = fc.decoded && T <= (uint32_t)kStageTris;
    const uint32_t wmin = staged ? (fc.walk_min ? (uint32_t)fc.walk_min : kWalkMinSamplesPerThbStaged)
                                 : (fc.walk_min_u ? (uint32_t)fc.walk_min_u : kWalkMinSamplesPerThb);
    // (segment lists always fit k_shade's per-warp stage, so the segment
    // kernel reads them from shared memory only; longer lists take the walk)
    const bool seg = !fc.threshold && d.frags < wmin * d.cnt && d.cnt <= (uint32_t)kShadeStage;
    d.pad = seg ? 1u : 0u;
    const uint32_t hbi = (uint32_t)bin * 32u + (uint32_t)(row * 8 + warp * 2 + lane);
    B.hbd[hbi] = d;
    const uint32_t cost = seg ? 0u : min(d.frags + 4u * d.cnt, 0x00ffffffu);
    const uint32_t both = cost + __shfl_down_sync(0x3u, cost, 1);  // the block's two halves
    const unsigned walks = __ballot_sync(0x3u, !seg);
    // bit 31: the bin has half-blocks for k_shade's wave walk (or background)
    if (!kFuse && lane == 0 && (both || walks)) {
      atomicAdd(&B.bin_cost[bin], both);
      if (both) atomicAdd(&B.ctr->walk_cost, (unsigned long long)both);
    }
    if (!kFuse && lane == 0 && walks) atomicOr(&B.bin_cost[bin], 0x80000000u);
    // low-pass entries of a bin that later propagates are stale (k_shade_seg skips them)
    if (seg && !kFuse)
      B.seg_queue[checked_index(atomicAdd(&B.ctr->seg_count, 1u), (uint32_t)fc.nbins * 32u)] =
          make_uint4(hbi | (pass == kPassLow ? 0u : 0x80000000u), d.off, d.cnt, d.frags);
  }
  if (threadIdx.x == 0) {
    unsigned long long* slot = B.slots + ((size_t)bin * 4 + row) * 5;
    slot[0] = slot[3] = slot[4] = 0;
  }
  if (lane == 0) {
    unsigned long long* slot = B.slots + ((size_t)bin * 4 + row) * 5;
    atomicAdd(&slot[1], (unsigned long long)(frags[0] + frags[1]));
    atomicAdd(&slot[2], (unsigned long long)(nthb[0] + nthb[1]));
  }
  if constexpr (kFuse != 0) {
    // Fused raster: warp w shades the two half-blocks of block (row, w) it
    // just extracted, from the pool lists (L2-hot) and the TBR planes in V.tp.
    __syncthreads();  // thread 0's slot reset precedes the shading's stat atomics
    uint32_t* route = V.rows + (size_t)warp * 128u;  // phase-A scratch, free now
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      const uint32_t off = pbase + (uint32_t)h * n, cnt = nthb[h], frg = frags[h];
      const int hpx0 = px0 + warp * 8, hpy0 = py0 + row * 8 + h * 4;
      PixelOut po;
      po.acc = make_float4(0.f, 0.f, 0.f, 0.f);
      po.invalid = false;
      po.hash = kHashSeed;
      po.emitted = 0;
      unsigned long long enumerated = frg;
      if (cnt) {
        const uint32_t* tri_l = B.pool_tri + off;
        const uint32_t* mask_l = B.pool_mask + off;
        const uint32_t* pre_l = B.pool_pre + off;
        const uint16_t* slot_l = B.pool_slot + off;
        auto run = [&](auto& f) {
          if (fc.threshold)
            shade_walk<3, true, false>(fc, B, hpx0, hpy0, tri_l, mask_l, cnt, po, &enumerated, f, slot_l, V.tp);
          else if (frg < kWalkMinSamplesPerThb * cnt)
            shade_segments<3, false>(fc, B, hpx0, hpy0, tri_l, mask_l, pre_l, cnt, frg, route, po, f, slot_l,
                                     V.tp);
          else
            shade_waves<3, false>(fc, B, hpx0, hpy0, tri_l, mask_l, slot_l, nullptr, cnt, po, f, V.tp);
        };
        if constexpr (kFuse == 1) {  // depth_filter_size 3, the reference default
          RegFilter<3, true> f;
          f.reset();
          run(f);
        } else {
          MemFilter f;
          dfm_reset<1>(B, nullptr, f, 4);
          run(f);
        }
      }
      finish_half_block(fc, B, bin, row, hpx0, hpy0, po, true, enumerated);
    }
  }
}

// kFuse: 0 = extraction only (k_shade shades), 1 = fused raster with the
// register filter (depth_filter_size 3), 2 = fused raster with MemFilter.
template <bool kGlobal, int kFuse>
__global__ void __launch_bounds__(128, kFuse ? 6 : 7) k_extract(Buffers B, int pass,
                                                              uint32_t cap_tbr, uint32_t cap_tb) {
  grid_dep_wait();
  const FrameConst& fc = c_fc;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __shared__ ItemState st;
  if (B.ctr->error) return;
  __shared__ uint32_t item_next[2];  // by iteration parity (one barrier per item fetch)
  const uint32_t nitems = kGlobal ? B.ctr->spill_count[pass] : B.ctr->list_count[pass] * 4u;
  // (the global-scratch and high passes are usually empty: leave before the
  // work counter, whose atomics every CTA would otherwise serialize on)
  if (nitems == 0) return;
  if (kFuse) {  // the generic shading path's unpack and axis-light tables
    load_shared_luts();
    fill_axis_light(fc);
    __syncthreads();
  }
  RasterView V;
  V.cs = nullptr;
  V.tp = nullptr;
  if (kFuse) {
    V.cs = B.cscratch + (kGlobal ? B.cs_off_g + (size_t)blockIdx.x * B.cs_per_cta_g
                                 : (size_t)blockIdx.x * B.cs_per_cta);
    V.tp = B.tplanes + (kGlobal ? B.tp_off_g + (size_t)blockIdx.x * B.tp_per_cta_g
                                : (size_t)blockIdx.x * B.tp_per_cta);
  }
  if (kGlobal) {
    uint8_t* g = B.scratch + (size_t)blockIdx.x * B.scratch_per_cta;
    V.tbr = reinterpret_cast<Tbr*>(g);
    g += (size_t)cap_tbr * sizeof(Tbr);
    g = reinterpret_cast<uint8_t*>(((uintptr_t)g + 15) & ~(uintptr_t)15);
    V.keys = reinterpret_cast<uint64_t*>(g);
    g += (size_t)4 * cap_tb * 8;
    V.refs = reinterpret_cast<uint16_t*>(g);
    g += (size_t)4 * cap_tb * 2;
    V.rows = reinterpret_cast<uint32_t*>(((uintptr_t)g + 15) & ~(uintptr_t)15);
  } else {
    RasterShared* sh = reinterpret_cast<RasterShared*>(smem_raw);
    V.tbr = sh->tbr;
    V.keys = sh->keys;
    V.refs = sh->refs;
    V.rows = reinterpret_cast<uint32_t*>(sh->refs);  // refs are unused until phase B
  }
  unsigned int* counter = &B.ctr->work_next[pass * 2 + (kGlobal ? 1 : 0)];
  // Thread 0 takes the next item, decides whether this pass extracts it and
  // resets the item state, all before the one barrier that publishes them
  // (so the decision is uniform even while a sibling block-row of the same
  // bin flips B.prop). The published words are double-buffered by iteration
  // parity: the write for iteration k+1 cannot race the reads of k.
  auto fetch = [&](uint32_t slot) {
    const uint32_t item = atomicAdd(counter, 1u);
    uint32_t code = 0xffffffffu;
    if (item < nitems) {
      const uint32_t c = kGlobal ? B.spill[pass][item] : (B.bin_list[pass][item >> 2] << 2) | (item & 3u);
      const int bin = (int)(c >> 2);
      const int bxi = bin % fc.bins_x, byi = bin / fc.bins_x;
      const uint8_t cat = B.cat[bin];
      const bool owned = fc.world <= 1 || ((bxi + 3 * byi) % fc.world) == fc.rank;
      bool run = owned && cat != 0;
      if (run) {
        if (pass == kPassLow)
          run = cat == 1 && !fc.force_high && !(!kGlobal && B.prop[bin]);  // sibling already overflowed
        else
          run = cat == 2 || (cat == 1 && fc.force_high) || B.prop[bin];
      }
      code = run ? c : 0xfffffffeu;  // 0xfffffffe: skip this item
    }
    item_next[slot] = code;
    reset_item_state(&st);
  };
  if (threadIdx.x == 0) fetch(0);
  __syncthreads();
  for (uint32_t k = 0;; k ^= 1u) {
    const uint32_t code = item_next[k];
    if (code == 0xffffffffu) break;
    const bool run = code != 0xfffffffeu;
    const int bin = (int)(code >> 2), row = (int)(code & 3u);
    if (run) {
      extract_item<kGlobal, kFuse>(fc, B, pass, bin, row, V, &st, cap_tbr, cap_tb);
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      if (run && st.status) {
        if (st.status == 1) {  // soft overflow: the whole bin goes to the high pass
          B.prop[bin] = 1;
          if (atomicAdd(&B.prop_q[bin], 1u) == 0u)
            B.bin_list[1][checked_index(atomicAdd(&B.ctr->list_count[1], 1u), (uint32_t)fc.nbins)] =
                (uint32_t)bin;
        } else if (st.status == 2) {
          const uint32_t sl = atomicAdd(&B.ctr->spill_count[pass], 1u);
          B.spill[pass][sl] = code;
        } else {
          atomicMax(&B.ctr->bin_error, ~((unsigned long long)bin * 64ull +
                                           (unsigned long long)min(st.err_code, 63)));
        }
      }
      fetch(k ^ 1u);
    }
    __syncthreads();
  }
}

// Shading: a CTA of 8 warps takes one (bin, block-row) work item; warp w
// shades half-block w of the row (raster.cpp:201-321), so the 8 warps touch
// the same triangles (L1 reuse). Each warp first stages its tri-half-block
// list from the pool into shared memory (coalesced), keeping the segment
// mapping's dependent lookups on-chip. Empty bins and half-blocks without
// samples composite the background.

// Bulk asynchronous copies (the TMA engine's 1-D cp.async.bulk) completing
// on a per-warp mbarrier, for k_shade's THB-list staging.
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_to_smem(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(phase)
        : "memory");
  } while (!done);
}

// kMode: 0 = broadcast walk for half-blocks with big THBs (also writes every
// half-block without samples), 1 = segment routing for the rest, 2 = alpha
// threshold walk for all. Separate instantiations keep each path's register
// allocation small.
template <int KM, int kMode, bool kTex>
__global__ void __launch_bounds__(256, kMode == 1 ? 4 : 2) k_shade(Buffers B) {
  const FrameConst& fc = c_fc;
  // (an empty segment queue: nothing to shade, skip the table set-up)
  if (kMode == 1) grid_dep_wait();  // (reads the segment count right away)
  if (kMode == 1 && (B.ctr->error || B.ctr->seg_count == 0)) return;
  load_shared_luts();  // (scene-static tables and the frame constants: ahead of the wait)
  fill_axis_light(fc);
  __syncthreads();
  grid_dep_wait();
  // (+8 entries: bulk copies move 16-byte aligned runs around the list)
  __shared__ __align__(16) uint32_t stage_tri[8][kShadeStage + 8];
  __shared__ __align__(16) uint32_t stage_mask[8][kShadeStage + 8];
  __shared__ __align__(16) uint32_t stage_pre[8][kShadeStage + 8];
  __shared__ __align__(16) uint16_t stage_slot[8][kShadeStage + 8];
  __shared__ __align__(8) uint64_t stage_bar[8];
  extern __shared__ __align__(16) uint8_t shade_dyn[];  // staged bin triangles, filter slots
  StagedTri* row_tris = reinterpret_cast<StagedTri*>(shade_dyn);
  __shared__ uint32_t route_s[8][32];
  __shared__ uint32_t item_s;
  if (B.ctr->error) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t bar_phase = 0;
  if (fc.bulk_stage && lane == 0) mbar_init(&stage_bar[warp]);
  __syncwarp();
  __shared__ int hb_next, hb_count;
  __shared__ uint8_t hb_order[32];  // the item's half-blocks, most samples first
  // modes 0/2: CTA items = (bin, part) from k_order_bins, warps pull the
  // part's half-blocks (every parts-th of the bin's longest-first order);
  // mode 1: warp items from the queue mode 0 filled
  const uint32_t nitems = kMode == 1 ? B.ctr->seg_count : B.ctr->order_count;
  uint32_t cta_bin = 0xffffffffu;
  bool staged_ok = false;
  uint32_t seg_ticket = 0;
  HbDesc seg_desc = {0, 0, 0, 0};
  if (kMode == 1 && lane == 0) seg_ticket = atomicAdd(&B.ctr->shade_next[1], 1u);
  for (;;) {
    uint32_t item;
    if (kMode == 1) {
      // the ticket for the next entry is taken one iteration ahead (lane 0)
      const uint32_t t = __shfl_sync(0xffffffffu, seg_ticket, 0);
      if (t >= nitems) break;
      if (lane == 0) seg_ticket = atomicAdd(&B.ctr->shade_next[1], 1u);
      const uint4 e = B.seg_queue[t];
      item = e.x;
      if (!(item & 0x80000000u) && B.prop[(item & 0x7fffffffu) >> 5]) continue;  // stale low-pass entry
      item &= 0x7fffffffu;
      seg_desc = HbDesc{e.y, e.z, e.w, 1u};
    } else {
      // next half-block of the CTA's bin, or the next bin
      int hbi = 32;
      if (cta_bin != 0xffffffffu) {
        if (lane == 0) hbi = atomicAdd(&hb_next, 1);
        hbi = __shfl_sync(0xffffffffu, hbi, 0);
        if (hbi >= hb_count) hbi = 32;
      }
      if (hbi >= 32) {
        __syncthreads();  // everyone is done with the staged bin
        if (threadIdx.x == 0) {
          item_s = atomicAdd(&B.ctr->shade_next[0], 1u);
          hb_next = 0;
        }
        __syncthreads();
        const uint32_t entry = item_s < nitems ? B.bin_order[item_s] : 0xffffffffu;
        if (entry == 0xffffffffu) break;
        cta_bin = entry & 0xffffffu;
        const int bxi = (int)cta_bin % fc.bins_x, byi = (int)cta_bin / fc.bins_x;
        const bool owned = fc.world <= 1 || ((bxi + 3 * byi) % fc.world) == fc.rank;
        staged_ok = false;
        if (kMode == 0 && owned && fc.decoded && B.cat[cta_bin] != 0) {
          // stage the bin's triangles (bin-list expansion order) once
          const uint32_t nq = B.qcnt[cta_bin], nt = B.tcnt[cta_bin], o = B.off[cta_bin];
          const uint32_t T = 2 * nq + nt;
          staged_ok = T <= (uint32_t)kStageTris;
          if (staged_ok)
            for (uint32_t j = threadIdx.x; j < T; j += blockDim.x) {
              const uint32_t tri = j < 2 * nq ? B.items[o + (j >> 1)] * 2 + (j & 1) : B.items[o + nq + (j - 2 * nq)];
              stage_triangle(fc, B, tri, &row_tris[j]);
            }
        }
        if (warp == 0) {
          // longest-first order of the bin's half-blocks (their sample counts
          // are known), so the warps' last pulls are short ones
          uint32_t cost = 0;
          if (owned && B.cat[cta_bin] != 0) {
            const HbDesc hd = B.hbd[(size_t)cta_bin * 32 + lane];
            cost = (kMode == 0 && hd.pad) ? 0u : min(hd.frags + 4u * hd.cnt, 0x7ffffffu);
          }
          uint32_t key = (cost << 5) | (31u - (uint32_t)lane);  // descending, ties by index
#pragma unroll
          for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) {
              const uint32_t other = __shfl_xor_sync(0xffffffffu, key, j);
              const bool desc = (lane & k) == 0, lower = (lane & j) == 0;
              const uint32_t hi = max(key, other), lo = min(key, other);
              key = (desc == lower) ? hi : lo;
            }
          // this part's share: every parts-th entry of the order (the
          // whole order when the bin is one item)
          const uint32_t lp = entry >> 28, part = (entry >> 24) & 7u;
          if ((lane & ((1 << lp) - 1)) == (int)part) hb_order[lane >> lp] = (uint8_t)(31u - (key & 31u));
          if (lane == 0) hb_count = 32 >> lp;
        }
        __syncthreads();
        if (!owned) {
          cta_bin = 0xffffffffu;
          continue;
        }
        if (lane == 0) hbi = atomicAdd(&hb_next, 1);
        hbi = __shfl_sync(0xffffffffu, hbi, 0);
        if (hbi >= hb_count) continue;
      }
      item = cta_bin * 32u + (uint32_t)hb_order[hbi];
    }
    const int bin = (int)(item >> 5), row = (int)((item >> 3) & 3u);
    const int bxi = bin % fc.bins_x, byi = bin / fc.bins_x;
    if (kMode == 1 && !(fc.world <= 1 || ((bxi + 3 * byi) % fc.world) == fc.rank)) continue;
    const int hb = (int)(item & 31u);  // reference half-block index in the bin
    const int block = hb >> 1;
    const int hpx0 = bxi * kBin + (block & 3) * 8;
    const int hpy0 = byi * kBin + (block >> 2) * 8 + (hb & 1) * 4;
    PixelOut po;
    po.acc = make_float4(0.f, 0.f, 0.f, 0.f);
    po.invalid = false;
    po.hash = kHashSeed;
    po.emitted = 0;
    unsigned long long enumerated = 0;
    bool live;
    HbDesc d = {0, 0, 0, 0};
    if (kMode == 1) {  // queued entries carry their descriptor
      live = true;
      d = seg_desc;
    } else {
      live = B.cat[bin] != 0;
      if (live) d = B.hbd[(size_t)bin * 32 + hb];
    }
    if (kMode == 0 && live && d.pad) continue;  // queued for the segment kernel by k_extract
    if (live) {
      enumerated = d.frags;
      const uint32_t* tri_l = B.pool_tri + d.off;
      const uint32_t* mask_l = B.pool_mask + d.off;
      const uint32_t* pre_l = B.pool_pre + d.off;
      const uint16_t* slot_l = B.pool_slot + d.off;
      uint32_t sh4 = 0, sh8 = 0;  // the staged lists' offsets in stage_* (u32 / u16 lists)
      if (d.cnt <= (uint32_t)kShadeStage && fc.bulk_stage) {
        // four bulk copies (16-byte aligned runs covering the list) onto the
        // warp's mbarrier; the generic-proxy reads of the previous list are
        // ordered before the async-proxy writes by the proxy fence
        const uint32_t a4 = d.off & ~3u, n4 = ((d.off + d.cnt + 3u) & ~3u) - a4;  // u32 lists
        const uint32_t a8 = d.off & ~7u, n8 = ((d.off + d.cnt + 7u) & ~7u) - a8;  // u16 list
        __syncwarp();
        if (lane == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(&stage_bar[warp], 3u * 4u * n4 + 2u * n8);
          bulk_to_smem(stage_tri[warp], B.pool_tri + a4, 4u * n4, &stage_bar[warp]);
          bulk_to_smem(stage_mask[warp], B.pool_mask + a4, 4u * n4, &stage_bar[warp]);
          bulk_to_smem(stage_pre[warp], B.pool_pre + a4, 4u * n4, &stage_bar[warp]);
          bulk_to_smem(stage_slot[warp], B.pool_slot + a8, 2u * n8, &stage_bar[warp]);
        }
        mbar_wait(&stage_bar[warp], bar_phase);
        bar_phase ^= 1u;
        sh4 = d.off - a4;
        sh8 = d.off - a8;
        tri_l = stage_tri[warp] + sh4;
        mask_l = stage_mask[warp] + sh4;
        pre_l = stage_pre[warp] + sh4;
        slot_l = stage_slot[warp] + sh8;
      } else if (d.cnt <= (uint32_t)kShadeStage) {
        for (uint32_t i = lane; i < d.cnt; i += 32) {
          stage_tri[warp][i] = tri_l[i];
          stage_mask[warp][i] = mask_l[i];
          stage_pre[warp][i] = pre_l[i];
          stage_slot[warp][i] = slot_l[i];
        }
        __syncwarp();
        tri_l = stage_tri[warp];
        mask_l = stage_mask[warp];
        pre_l = stage_pre[warp];
        slot_l = stage_slot[warp];
      }
      if (kMode == 2) {
        if constexpr (KM == 0) {
          MemFilter f;
          dfm_reset<kMode>(B, shade_dyn, f);
          shade_walk<KM, true, kTex>(fc, B, hpx0, hpy0, tri_l, mask_l, d.cnt, po, &enumerated, f);
        } else {
          RegFilter<KM, true> f;
          f.reset();
          shade_walk<KM, true, kTex>(fc, B, hpx0, hpy0, tri_l, mask_l, d.cnt, po, &enumerated, f);
        }
      } else if (kMode == 0)  // big THBs: wave walk
      {
        if constexpr (KM != 0) {
          SlotFilter<KM> f;
          f.reset(reinterpret_cast<float4*>(shade_dyn + (size_t)kStageTris * sizeof(StagedTri)) +
                  (size_t)warp * KM * 32 + lane);
          if (staged_ok && d.cnt <= (uint32_t)kShadeStage && !fc.wave1) {  // all operands in shared memory
            // (the lists named through stage_* directly: shared-memory loads
            // instead of generic ones through the merged list pointers)
            if (fc.dump) {
              shade_waves_staged2<KM, 2>(fc, hpx0, hpy0, stage_tri[warp] + sh4, stage_mask[warp] + sh4,
                                         stage_slot[warp] + sh8, row_tris, d.cnt, po, f);
            } else {
              shade_waves_staged2<KM, 1>(fc, hpx0, hpy0, stage_tri[warp] + sh4, stage_mask[warp] + sh4,
                                         stage_slot[warp] + sh8, row_tris, d.cnt, po, f);
              // every sample pushed is blended exactly once (no threshold), so the
              // warp's emitted total is the half-block's sample count (stats only;
              // per-pixel counts exist only in dump frames)
              po.emitted = lane == 0 ? d.frags : 0u;
            }
          }
          else if (staged_ok && d.cnt <= (uint32_t)kShadeStage)
            shade_waves<KM, kTex>(fc, B, hpx0, hpy0, tri_l, mask_l, slot_l, row_tris, d.cnt, po, f);
          else
            shade_waves<KM, kTex>(fc, B, hpx0, hpy0, tri_l, mask_l, slot_l, staged_ok ? row_tris : nullptr,
                            d.cnt, po, f);
        } else {
          MemFilter f;
          dfm_reset<kMode>(B, shade_dyn, f);
          shade_waves<KM, kTex>(fc, B, hpx0, hpy0, tri_l, mask_l, slot_l, staged_ok ? row_tris : nullptr,
                          d.cnt, po, f);
        }
      }
      else if (d.frags) {  // small THBs: dense segments + routing
        if constexpr (KM != 0) {
          SlotFilter<KM> f;
          f.reset(reinterpret_cast<float4*>(shade_dyn) + (size_t)warp * KM * 32 + lane);
          // segment lists are staged (k_extract queues only lists that fit):
          // named through the stage arrays, the loads are LDS, not generic
          VEIL_CHECK(d.cnt <= (uint32_t)kShadeStage);
          shade_segments<KM, kTex>(fc, B, hpx0, hpy0, stage_tri[warp] + sh4, stage_mask[warp] + sh4,
                                   stage_pre[warp] + sh4, d.cnt, d.frags, route_s[warp], po, f);
        } else {
          MemFilter f;
          dfm_reset<kMode>(B, shade_dyn, f);
          VEIL_CHECK(d.cnt <= (uint32_t)kShadeStage);
          shade_segments<KM, kTex>(fc, B, hpx0, hpy0, stage_tri[warp] + sh4, stage_mask[warp] + sh4,
                                   stage_pre[warp] + sh4, d.cnt, d.frags, route_s[warp], po, f);
        }
      }
    }
    finish_half_block(fc, B, bin, row, hpx0, hpy0, po, live, enumerated);
  }
}

// Deterministic stat merge (renderer.cpp:170-212): integer sums over the
// owned bins' (bin, block-row) slots; warp shuffles, then one atomic per
// warp and counter.
// Longest-first bin order for k_shade (bins with the most wave-walk work
// first, so the kernel's tail is made of short bins): a 256-bucket
// log-scale counting sort of the per-bin costs k_extract accumulated.
__global__ void __launch_bounds__(1024) k_order_bins(Buffers B, uint32_t shade_ctas) {
  grid_dep_wait();
  grid_dep_launch();  // k_shade's CTAs fill their lookup tables meanwhile
  const FrameConst& fc = c_fc;
  __shared__ uint32_t hist[256];
  __shared__ uint32_t base[256];
  if (B.ctr->error) return;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  auto bucket = [](uint32_t c) -> uint32_t {  // 8 sub-buckets per octave, descending
    if (c == 0) return 255u;
    const uint32_t e = 31u - (uint32_t)__clz(c);
    const uint32_t m = e >= 3 ? (c >> (e - 3)) & 7u : (c << (3 - e)) & 7u;
    return 255u - min(254u, e * 8u + m);
  };
  // bins with no wave-walk work (every half-block queued for the segment
  // kernel) and bins another rank owns are left out; empty bins stay (their
  // half-blocks get the background) unless k_fill_empty paints them
  auto wanted = [&](int b) {
    const int bxi = b % fc.bins_x, byi = b / fc.bins_x;
    if (fc.world > 1 && ((bxi + 3 * byi) % fc.world) != fc.rank) return false;
    return (B.cat[b] == 0 && !fc.fill_split) || (B.bin_cost[b] & 0x80000000u) != 0u;
  };
  // A bin costing more than the frame's fair share per shading CTA (a
  // sharded rank has few bins: its heaviest ones would bound k_shade) is
  // split into 2..8 parts, each a CTA item taking every parts-th half-block.
  // (The frame's total is the sum k_extract accumulated next to the bin costs.)
  const unsigned long long share = max(1ull, B.ctr->walk_cost / max(1u, shade_ctas));
  auto log_parts = [&](uint32_t c) -> uint32_t {
    uint32_t lp = 0;
    while (lp < 3u && (unsigned long long)c > (share << lp)) ++lp;
    return lp;
  };
  for (int b = threadIdx.x; b < fc.nbins; b += blockDim.x)
    if (wanted(b)) {
      const uint32_t c = B.bin_cost[b] & 0x7fffffffu, lp = log_parts(c);
      atomicAdd(&hist[bucket(c >> lp)], 1u << lp);
    }
  __syncthreads();
  if (threadIdx.x < 32) {  // exclusive scan of 256 buckets by one warp
    uint32_t run = 0;
    for (int k = 0; k < 8; ++k) {
      const uint32_t v = hist[k * 32 + threadIdx.x];
      uint32_t x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if ((int)threadIdx.x >= o) x += y;
      }
      base[k * 32 + threadIdx.x] = run + x - v;
      run += __shfl_sync(0xffffffffu, x, 31);
    }
    if (threadIdx.x == 0) B.ctr->order_count = run;
  }
  __syncthreads();
  for (int b = threadIdx.x; b < fc.nbins; b += blockDim.x)
    if (wanted(b)) {
      const uint32_t c = B.bin_cost[b] & 0x7fffffffu, lp = log_parts(c);
      const uint32_t at = atomicAdd(&base[bucket(c >> lp)], 1u << lp);
      for (uint32_t p = 0; p < (1u << lp); ++p) B.bin_order[at + p] = (uint32_t)b | (p << 24) | (lp << 28);
    }
}

__device__ __forceinline__ void finalize_sums(const FrameConst& fc, const Buffers& B);

// host_ctr: the scene's pinned counter block (device-mapped); the last CTA
// copies the frame's final counters there, so no read-back copy follows.
__global__ void __launch_bounds__(256) k_finalize(Buffers B, Counters* host_ctr) {
  grid_dep_wait();
  const FrameConst& fc = c_fc;
  __shared__ bool last;
  if (!B.ctr->error) finalize_sums(fc, B);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&B.ctr->finalize_done, 1u) == gridDim.x - 1u;
  }
  __syncthreads();
  if (last) {
    __threadfence();
    const volatile uint32_t* src = reinterpret_cast<const volatile uint32_t*>(B.ctr);
    uint32_t* dst = reinterpret_cast<uint32_t*>(host_ctr);
    for (uint32_t i = threadIdx.x; i < sizeof(Counters) / 4; i += blockDim.x) dst[i] = src[i];
  }
}

__device__ __forceinline__ void finalize_sums(const FrameConst& fc, const Buffers& B) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long v[6] = {0, 0, 0, 0, 0, 0};
  if (b < fc.nbins) {
    const int bxi = b % fc.bins_x, byi = b / fc.bins_x;
    const bool owned = fc.world <= 1 || ((bxi + 3 * byi) % fc.world) == fc.rank;
    if (owned && B.cat[b]) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int k = 0; k < 5; ++k) v[k] += B.slots[((size_t)b * 4 + r) * 5 + k];
      v[5] = B.prop[b];
    }
  }
#pragma unroll
  for (int k = 0; k < 6; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  if ((threadIdx.x & 31) == 0) {
    unsigned long long* dst[6] = {&B.ctr->samples, &B.ctr->fragments, &B.ctr->thb,
                                  &B.ctr->segments, &B.ctr->invalid, &B.ctr->bins_propagated};
#pragma unroll
    for (int k = 0; k < 6; ++k)
      if (v[k]) atomicAdd(dst[k], v[k]);
  }
}

// The background of the empty bins this rank owns (a CTA per bin): for fused
// raster frames (no k_shade) and, by default, for all frames -- eight 256-thread
// CTAs per SM paint them faster than k_shade's bin loop (two CTAs per SM,
// three block barriers per bin).
__global__ void __launch_bounds__(256) k_fill_empty(Buffers B) {
  grid_dep_wait();
  const FrameConst& fc = c_fc;
  if (B.ctr->error) return;
  for (int b = blockIdx.x; b < fc.nbins; b += gridDim.x) {
    const int bxi = b % fc.bins_x, byi = b / fc.bins_x;
    if (B.cat[b] != 0 || !(fc.world <= 1 || ((bxi + 3 * byi) % fc.world) == fc.rank)) continue;
    const int warp = threadIdx.x >> 5;
    PixelOut po;
    po.acc = make_float4(0.f, 0.f, 0.f, 0.f);
    po.invalid = false;
    po.hash = kHashSeed;
    po.emitted = 0;
    for (int hb = warp; hb < 32; hb += 8) {
      const int block = hb >> 1;
      finish_half_block(fc, B, b, block >> 2, bxi * kBin + (block & 3) * 8,
                        byi * kBin + (block >> 2) * 8 + (hb & 1) * 4, po, false, 0);
    }
  }
}

// RenderConfig::measure_disorder (raster.cpp:286-297) on the frame just
// rendered: a warp per (bin, half-block), lane = pixel. The pixel's samples
// arrive in the canonical enumeration order (THBs in sorted order); sample i's
// disorder is i minus the number of the pixel's samples with a smaller key
// (its position in the sorted sequence; keys are unique). The frame's maximum
// goes to *out. O(n^2) per pixel over the THB list: a measurement, not a
// frame path.
__global__ void __launch_bounds__(256) k_disorder(Buffers B, int* out) {
  grid_dep_wait();
  const FrameConst& fc = c_fc;
  if (B.ctr->error) return;
  const int lane = threadIdx.x & 31;
  const uint32_t nhb = (uint32_t)fc.nbins * 32u;
  const uint32_t gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  int best = 0;
  for (uint32_t item = gwarp; item < nhb; item += nwarps) {
    const int bin = (int)(item >> 5), hb = (int)(item & 31u);
    const int bxi = bin % fc.bins_x, byi = bin / fc.bins_x;
    if (B.cat[bin] == 0 || !(fc.world <= 1 || ((bxi + 3 * byi) % fc.world) == fc.rank)) continue;
    const HbDesc d = B.hbd[item];
    const int block = hb >> 1;
    const int px = bxi * kBin + (block & 3) * 8 + (lane & 7);
    const int py = byi * kBin + (block >> 2) * 8 + (hb & 1) * 4 + (lane >> 3);
    const double x = (double)px + 0.5, y = (double)py + 0.5;
    const uint32_t* tri_l = B.pool_tri + d.off;
    const uint32_t* mask_l = B.pool_mask + d.off;
    auto key_of = [&](uint32_t r) {
      const uint32_t tri = tri_l[r];
      return sample_key(fc, quantize_depth(eval(B.tri[tri].dz, x, y)), tri);
    };
    int i = 0;
    for (uint32_t r = 0; r < d.cnt; ++r) {
      if (!((mask_l[r] >> lane) & 1u)) continue;
      const uint64_t k = key_of(r);
      int smaller = 0;
      for (uint32_t s = 0; s < d.cnt; ++s)
        if (((mask_l[s] >> lane) & 1u) && key_of(s) < k) ++smaller;
      best = max(best, i - smaller);
      ++i;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if (lane == 0 && best > 0) atomicMax(out, best);
}

// a-buffer reference renderer (oracle.cpp:28-117) on the bin lists: every
// triangle covering a pixel is in that pixel's bin list. Fragments are
// blended in exact key order by repeated selection of the next key, so no
// per-pixel list storage is needed (an oracle mode, not a fast path).
__global__ void __launch_bounds__(128) k_abuffer(Buffers B) {
  grid_dep_wait();
  const FrameConst& fc = c_fc;
  load_shared_luts();
  fill_axis_light(fc);
  __syncthreads();
  if (B.ctr->error) return;
  const int px = blockIdx.x * 16 + (threadIdx.x & 15);
  const int py = blockIdx.y * 8 + (threadIdx.x >> 4);
  if (px >= fc.width || py >= fc.height) return;
  const size_t pix = (size_t)py * fc.width + px;
  const int bin = (py / kBin) * fc.bins_x + px / kBin;
  const uint32_t nq = B.qcnt[bin], nt = B.tcnt[bin], o = B.off[bin];
  const uint32_t T = 2 * nq + nt;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  uint64_t hash = kHashSeed;
  uint32_t n = 0;
  uint64_t last = 0;
  bool first = true;
  for (;;) {
    uint64_t best = ~0ull;
    uint32_t best_t = 0;
    bool found = false;
    for (uint32_t i = 0; i < T; ++i) {
      uint32_t ti = i < 2 * nq ? B.items[o + (i >> 1)] * 2 + (i & 1) : B.items[o + nq + (i - 2 * nq)];
      if (!(B.tri_meta[ti].w & 0x100u)) continue;
      const TriRec& t = B.tri[ti];
      if (py < t.y_min || py > t.y_max || !covers(t, px, py)) continue;
      uint32_t qd = quantize_depth(eval(t.dz, (double)px + 0.5, (double)py + 0.5));
      uint64_t k = fc.extended ? (((uint64_t)qd << 32) | ti) : (((uint64_t)qd << 24) | (ti & 0xffffffu));
      if ((first || k > last) && k < best) {
        best = k;
        best_t = ti;
        found = true;
      }
    }
    if (!found) break;
    double depth;
    float4 c = shade_sample<true>(fc, B, best_t, px, py, &depth);
    acc = blend(acc, c);
    hash = (hash ^ best) * kHashPrime;
    ++n;
    last = best;
    first = false;
  }
  float4 out = blend(acc, make_float4(fc.bg[0], fc.bg[1], fc.bg[2], fc.bg[3]));
  B.fb[pix] = quantize_channel(out.x) | (quantize_channel(out.y) << 8) |
              (quantize_channel(out.z) << 16) | (quantize_channel(out.w) << 24);
  B.mask[pix] = 0;
  if (fc.dump) {
    B.hash[pix] = hash;
    B.emit[pix] = n;
  }
  atomicAdd(&B.ctr->samples, (unsigned long long)n);
}

// Owned 32x32 tiles <-> dense tile buffer (RGBA8 4096 B, then mask 1024 B per
// tile), tile i of a rank = its i-th owned bin in row-major bin order. One
// CTA per tile; a thread per pixel (4-byte RGBA word and 1-byte mask).
__global__ void __launch_bounds__(256) k_tile_copy(FrameConst fc, uint32_t* fb, uint8_t* mask,
                                                   uint8_t* tiles, const uint32_t* bins,
                                                   uint32_t ntiles, int unpack) {
  grid_dep_wait();
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int bin = (int)bins[t];
    const int bx = bin % fc.bins_x, by = bin / fc.bins_x;
    uint8_t* tile = tiles + (size_t)t * 5120;
    for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) {
      const int lx = i & 31, ly = i >> 5;
      const int px = bx * kBin + lx, py = by * kBin + ly;
      if (px >= fc.width || py >= fc.height) continue;
      const size_t pix = (size_t)py * fc.width + px;
      uint32_t* tw = reinterpret_cast<uint32_t*>(tile) + i;
      if (unpack) {
        fb[pix] = *tw;
        mask[pix] = tile[4096 + i];
      } else {
        *tw = fb[pix];
        tile[4096 + i] = mask[pix];
      }
    }
  }
}

}  // namespace dev

// ============================================================ host side

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(VEIL_ERR_INTERNAL, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

thread_local int t_device = 0;

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t n) {
    if (n <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    size_t alloc = std::max<size_t>(n, 256);
    ck(cudaMalloc(&p, alloc), "cudaMalloc");
    bytes = alloc;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <typename T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

}  // namespace

struct DeviceScene {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint64_t uploaded_version = 0;
  uint32_t nverts = 0, nquads = 0;
  DevBuf pos, vcol, vnrm, quads, qmat, mats, vuv, texels, texlev, texdesc;
  bool textured = false;  // some material samples a texture (generic shading path)
  DevBuf zero, vq_uv, vq_src, vq_idx, vq_box, vq_flags, vq_mat, vq_col, vq_nrm, tri, tri_meta, shade,
      tri_y;
  DevBuf off, qcur, tcur, cat, bin_list0, bin_list1, prop_q, bin_cost, bin_order, prop, items, item_rows, slots, spill0, spill1, scratch, fb, mask,
      hash, emit, tile_ids, hbd, pool_tri, pool_mask, pool_pre, seg_queue, pool_slot, lpairs, lpair_cols,
      dfm_g, cscratch, tplanes, shard_tris, disorder;
  uint32_t items_cap = 0;
  uint32_t pool_cap = 0;
  uint32_t lpairs_cap = 0;
  dev::FrameConst* fc_host = nullptr;  // pinned staging of c_fc (graph memcpy source)
  void* peer_fb = nullptr;    // imported root framebuffer (cudaIpcOpenMemHandle)
  void* peer_mask = nullptr;
  int peer_w = 0, peer_h = 0;  // the imported framebuffer's viewport
  dev::Counters* ctr_host = nullptr;   // pinned counters readback (written by k_finalize)
  dev::Counters* ctr_dev = nullptr;    // ctr_host's device-mapped address
  // Cached CUDA graph of one whole frame (c_fc upload .. counters readback),
  // valid while the launch-shaping inputs in graph_key are unchanged.
  cudaGraphExec_t graph_exec = nullptr;
  std::vector<uint8_t> graph_key;
  int graph_launches = 0;
  bool extract_configured = false;
  int extract_ctas = 0;
  cudaEvent_t ev[6] = {};  // frame start, setup, binning, low extract, end, high extract
  veil_frame_stats last{};
  int fb_w = 0, fb_h = 0;
  int sm_count = 148;
  int raster_ctas_smem = 0;
  int raster_ctas_global = 0;

  ~DeviceScene() {
    if (peer_fb) cudaIpcCloseMemHandle(peer_fb);
    if (peer_mask) cudaIpcCloseMemHandle(peer_mask);
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    if (fc_host) cudaFreeHost(fc_host);
    if (ctr_host) cudaFreeHost(ctr_host);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {
std::mutex g_pinned_mu;
std::multimap<size_t, uint8_t*> g_pinned_free;  // pooled pinned frames by size
}  // namespace

std::shared_ptr<uint8_t> acquire_host_frame(size_t bytes) {
  uint8_t* p = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    auto it = g_pinned_free.lower_bound(bytes);
    if (it != g_pinned_free.end() && it->first <= bytes * 2) {
      p = it->second;
      bytes = it->first;
      g_pinned_free.erase(it);
    }
  }
  if (!p) ck(cudaMallocHost(reinterpret_cast<void**>(&p), std::max<size_t>(bytes, 64)), "cudaMallocHost");
  return std::shared_ptr<uint8_t>(p, [bytes](uint8_t* q) {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    if (g_pinned_free.size() < 8) {
      g_pinned_free.emplace(bytes, q);
    } else {
      cudaFreeHost(q);
    }
  });
}

void release_device_scene(DeviceScene* d) {
  if (!d) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(d->device);
  delete d;
  cudaSetDevice(prev);
}

void set_current_device(int device) {
  int n = 0;
  ck(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
  if (device < 0 || device >= n) throw Error(VEIL_ERR_INVALID_ARG, "no such CUDA device");
  t_device = device;
  ck(cudaSetDevice(device), "cudaSetDevice");
}

bool bin_owned(int bx, int by, int rank, int world) {
  return world <= 1 || ((bx + 3 * by) % world) == rank;
}

uint64_t shard_tile_count(int bins_x, int bins_y, int rank, int world) {
  uint64_t n = 0;
  for (int y = 0; y < bins_y; ++y)
    for (int x = 0; x < bins_x; ++x)
      if (bin_owned(x, y, rank, world)) ++n;
  return n;
}

namespace {

// The device workspace in `slot` (the scene's own, or one of its multi-device
// shards) on CUDA device `device`, created or moved on first use, with the
// scene's geometry uploaded.
DeviceScene* device_scene_on(const Scene& s, DeviceScene** slot, int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    throw Error(VEIL_ERR_INTERNAL, "no CUDA device available (libveil has no CPU fallback)");
  ck(cudaSetDevice(device), "cudaSetDevice");
  if (*slot && (*slot)->device != device) {
    release_device_scene(*slot);
    *slot = nullptr;
  }
  if (!*slot) {
    DeviceScene* d = new DeviceScene();
    d->device = device;
    ck(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    for (auto& e : d->ev) ck(cudaEventCreate(&e), "cudaEventCreate");
    ck(cudaMallocHost(reinterpret_cast<void**>(&d->fc_host), sizeof(dev::FrameConst)), "cudaMallocHost");
    ck(cudaMallocHost(reinterpret_cast<void**>(&d->ctr_host), sizeof(dev::Counters)), "cudaMallocHost");
    ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d->ctr_dev), d->ctr_host, 0), "cudaHostGetDevicePointer");
    cudaDeviceGetAttribute(&d->sm_count, cudaDevAttrMultiProcessorCount, device);
    {  // exact unpack tables (IEEE float division on the host)
      float lc[256], ln[1024];
      for (int q = 0; q < 256; ++q) lc[q] = float(q) / 255.0f;
      for (int q = -512; q < 512; ++q) ln[q + 512] = float(q) / 511.0f;
      ck(cudaMemcpyToSymbol(dev::g_lut_c, lc, sizeof lc), "lut");
      ck(cudaMemcpyToSymbol(dev::g_lut_n, ln, sizeof ln), "lut");
    }
    *slot = d;
  }
  DeviceScene* d = *slot;
  if (d->uploaded_version != s.geometry_version) {
    const size_t V = s.vertices.size(), Q = s.quads.size();
    std::vector<float4> pos(V);
    std::vector<uint32_t> vcol(V), vnrm(V), qmat(Q);
    std::vector<uint4> quads(Q);
    for (size_t i = 0; i < V; ++i) {
      const veil_vertex& v = s.vertices[i];
      pos[i] = make_float4(v.position[0], v.position[1], v.position[2], 0.0f);
      // pack_color / encode_normal of the vertex (packing.hpp:33-61); the
      // setup kernel gathers these per visible quad (setup.cpp:329-333).
      auto enc = [](float c, double s, long lo, long hi) {
        long q = std::lround(double(c) * s);
        return q < lo ? lo : (q > hi ? hi : q);
      };
      vcol[i] = uint32_t(enc(v.color[0], 255.0, 0, 255)) |
                (uint32_t(enc(v.color[1], 255.0, 0, 255)) << 8) |
                (uint32_t(enc(v.color[2], 255.0, 0, 255)) << 16) |
                (uint32_t(enc(v.color[3], 255.0, 0, 255)) << 24);
      vnrm[i] = (uint32_t(enc(v.normal[0], 511.0, -511, 511)) & 0x3ffu) |
                ((uint32_t(enc(v.normal[1], 511.0, -511, 511)) & 0x3ffu) << 10) |
                ((uint32_t(enc(v.normal[2], 511.0, -511, 511)) & 0x3ffu) << 20);
    }
    for (size_t i = 0; i < Q; ++i) {
      const veil_quad& q = s.quads[i];
      quads[i] = make_uint4(q.v[0], q.v[1], q.v[2], q.v[3]);
      qmat[i] = q.material;
    }
    std::vector<dev::MatDev> mats(s.materials.size());
    for (size_t i = 0; i < mats.size(); ++i) {
      const veil_material& m = s.materials[i];
      dev::MatDev md{};
      for (int k = 0; k < 4; ++k) md.base[k] = m.base_color[k];
      md.opacity = m.opacity;
      bool hc = (m.flags & VEIL_MATERIAL_VERTEX_COLORS) && (s.flags & VEIL_SCENE_HAS_COLORS);
      bool hn = (m.flags & VEIL_MATERIAL_VERTEX_NORMALS) && (s.flags & VEIL_SCENE_HAS_NORMALS);
      // record.has_uvs (setup.cpp:326-328): the material samples a texture
      // with UVs and the scene has them
      bool hu = (m.flags & VEIL_MATERIAL_UVS) && (s.flags & VEIL_SCENE_HAS_UVS) && m.texture >= 0;
      md.flags = (hc ? 1u : 0u) | (hn ? 2u : 0u) | (hu ? 4u : 0u);
      md.texture = m.texture;
      mats[i] = md;
    }
    d->textured = false;
    for (const veil_material& m : s.materials) d->textured |= m.texture >= 0;
    {  // vertex UVs and textures (mip levels as float4 texels)
      std::vector<float2> vuv((s.flags & VEIL_SCENE_HAS_UVS) ? V : 0);
      for (size_t i = 0; i < vuv.size(); ++i) vuv[i] = make_float2(s.vertices[i].uv[0], s.vertices[i].uv[1]);
      std::vector<float4> texels;
      std::vector<uint4> levels;
      std::vector<uint2> descs;
      for (const Texture& t : s.textures) {
        descs.push_back(make_uint2(uint32_t(levels.size()), uint32_t(t.levels.size())));
        for (const TextureLevel& l : t.levels) {
          levels.push_back(make_uint4(uint32_t(texels.size()), uint32_t(l.width), uint32_t(l.height), 0));
          for (size_t k = 0; k + 3 < l.texels.size(); k += 4)
            texels.push_back(make_float4(l.texels[k], l.texels[k + 1], l.texels[k + 2], l.texels[k + 3]));
        }
      }
      d->vuv.ensure(std::max<size_t>(1, vuv.size()) * sizeof(float2));
      d->texels.ensure(std::max<size_t>(1, texels.size()) * sizeof(float4));
      d->texlev.ensure(std::max<size_t>(1, levels.size()) * sizeof(uint4));
      d->texdesc.ensure(std::max<size_t>(1, descs.size()) * sizeof(uint2));
      if (!vuv.empty())
        ck(cudaMemcpy(d->vuv.p, vuv.data(), vuv.size() * sizeof(float2), cudaMemcpyHostToDevice), "upload");
      if (!texels.empty())
        ck(cudaMemcpy(d->texels.p, texels.data(), texels.size() * sizeof(float4), cudaMemcpyHostToDevice), "upload");
      if (!levels.empty())
        ck(cudaMemcpy(d->texlev.p, levels.data(), levels.size() * sizeof(uint4), cudaMemcpyHostToDevice), "upload");
      if (!descs.empty())
        ck(cudaMemcpy(d->texdesc.p, descs.data(), descs.size() * sizeof(uint2), cudaMemcpyHostToDevice), "upload");
    }
    d->pos.ensure(V * sizeof(float4));
    d->vcol.ensure(V * 4);
    d->vnrm.ensure(V * 4);
    d->quads.ensure(Q * sizeof(uint4));
    d->qmat.ensure(Q * 4);
    d->mats.ensure(mats.size() * sizeof(dev::MatDev));
    if (V) {
      ck(cudaMemcpy(d->pos.p, pos.data(), V * sizeof(float4), cudaMemcpyHostToDevice), "upload");
      ck(cudaMemcpy(d->vcol.p, vcol.data(), V * 4, cudaMemcpyHostToDevice), "upload");
      ck(cudaMemcpy(d->vnrm.p, vnrm.data(), V * 4, cudaMemcpyHostToDevice), "upload");
    }
    if (Q) {
      ck(cudaMemcpy(d->quads.p, quads.data(), Q * sizeof(uint4), cudaMemcpyHostToDevice), "upload");
      ck(cudaMemcpy(d->qmat.p, qmat.data(), Q * 4, cudaMemcpyHostToDevice), "upload");
    }
    if (!mats.empty())
      ck(cudaMemcpy(d->mats.p, mats.data(), mats.size() * sizeof(dev::MatDev),
                    cudaMemcpyHostToDevice),
         "upload");
    d->nverts = uint32_t(V);
    d->nquads = uint32_t(Q);
    d->uploaded_version = s.geometry_version;
    d->items_cap = 0;
  }
  return d;
}

DeviceScene* device_scene(const Scene& s) { return device_scene_on(s, &s.device, t_device); }

void camera_vectors(const Camera& c, dev::FrameConst* fc) {
  // camera_eye / camera_forward, scene.cpp:67-84
  fc->has_eye = 0;
  if (c.has_eye) {
    fc->has_eye = 1;
    for (int i = 0; i < 3; ++i) fc->eye[i] = c.eye[i];
  } else {
    double inv[16];
    if (mat4_inverse(c.m, inv)) {
      double v[4] = {0.0, 0.0, 1.0, 0.0}, h[4];
      for (int r = 0; r < 4; ++r)
        h[r] = inv[r * 4] * v[0] + inv[r * 4 + 1] * v[1] + inv[r * 4 + 2] * v[2] + inv[r * 4 + 3] * v[3];
      if (!(std::abs(h[3]) < 1e-12)) {
        double s = 1.0 / h[3];
        fc->eye[0] = h[0] * s;
        fc->eye[1] = h[1] * s;
        fc->eye[2] = h[2] * s;
        fc->has_eye = 1;
      }
    }
  }
  double g[3] = {c.m[8], c.m[9], c.m[10]};
  double len = std::sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
  if (len <= 0.0) {
    fc->fwd[0] = 0.0, fc->fwd[1] = 0.0, fc->fwd[2] = 1.0;
  } else {
    double inv = 1.0 / len;
    for (int i = 0; i < 3; ++i) fc->fwd[i] = g[i] * inv;
  }
}

// Upper bound of resident k_extract<false> CTAs per SM (launch bounds), which
// sizes the fused raster's per-CTA scratch.
constexpr int kExtractCtasPerSmMax = 7;

// Frame kernels are launched with programmatic stream serialization (see
// dev::grid_dep_wait): a kernel's launch and CTA scheduling overlap its
// predecessor's tail instead of following its completion.
template <typename... KArgs, typename... Args>
void pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  static const bool enabled = [] {  // VEIL_NO_PDL=1: plain stream-ordered launches
    const char* e = std::getenv("VEIL_NO_PDL");
    return !(e && *e && *e != '0');
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = enabled ? 1 : 0;
  ck(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "kernel launch");
}

template <int kFuse>
void launch_extract_k(DeviceScene* d, const dev::FrameConst& fc, const dev::Buffers& B, int pass,
                      uint32_t gcap_tbr, uint32_t gcap_tb, int* launches) {
  const size_t smem = sizeof(dev::RasterShared);
  static int per_sm_dev[64];  // per instantiation and device (attributes are per device)
  int& per_sm = per_sm_dev[d->device & 63];
  if (per_sm <= 0) {
    ck(cudaFuncSetAttribute(dev::k_extract<false, kFuse>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            int(smem)),
       "cudaFuncSetAttribute");
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dev::k_extract<false, kFuse>, 128, smem);
    per_sm = std::min(std::max(1, per_sm), kExtractCtasPerSmMax);
  }
  const int grid = int(std::min<long long>((long long)per_sm * d->sm_count, (long long)fc.nbins * 4));
  pdl_launch(dev::k_extract<false, kFuse>, grid, 128, smem, d->stream, B, pass,
             uint32_t(dev::RasterShared::kTbr), uint32_t(dev::RasterShared::kTb));
  ck(cudaGetLastError(), "k_extract launch");
  pdl_launch(dev::k_extract<true, kFuse>, d->raster_ctas_global, 128, 0, d->stream, B, pass, gcap_tbr, gcap_tb);
  *launches += 2;
}

void launch_extract(DeviceScene* d, const dev::FrameConst& fc, const dev::Buffers& B, int pass,
                    uint32_t gcap_tbr, uint32_t gcap_tb, int* launches) {
  if (!fc.fused)
    launch_extract_k<0>(d, fc, B, pass, gcap_tbr, gcap_tb, launches);
  else if (fc.df == 3)
    launch_extract_k<1>(d, fc, B, pass, gcap_tbr, gcap_tb, launches);
  else
    launch_extract_k<2>(d, fc, B, pass, gcap_tbr, gcap_tb, launches);
}

// Ring filters (KM == 0, depth_filter_size > 8) live in dynamic shared memory
// when a block's eight warps' rings fit next to the staged triangles, else in
// a global scratch (VEIL_DFM_GLOBAL=1 forces the latter for A/B tests).
constexpr size_t kDfmBytesPerEntry = 32 * (8 + 16);  // one node per lane: key + colour slot
constexpr size_t kDfmSmemBudget = 190 * 1024;

template <int KM, int kMode, bool kTex>
void launch_shade_mode(DeviceScene* d, const dev::FrameConst& fc, const dev::Buffers& B,
                       int* launches) {
  size_t dyn = (kMode == 0 ? size_t(dev::kStageTris) * sizeof(dev::StagedTri) : 0);
  if (KM != 0)
    dyn += (kMode != 2 ? size_t(8) * KM * 32 * sizeof(float4) : 0);
  else if (!B.dfm_g)
    dyn += size_t(8) * B.dfm_cap * kDfmBytesPerEntry;
  static size_t configured_dev[64];  // per instantiation and device: the largest size set so far
  size_t& configured = configured_dev[d->device & 63];
  if (dyn > configured) {
    ck(cudaFuncSetAttribute(dev::k_shade<KM, kMode, kTex>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            int(dyn)),
       "cudaFuncSetAttribute");
    configured = dyn;
  }
  static std::map<size_t, int> per_sm_by_dyn_dev[64];  // per instantiation and device
  std::map<size_t, int>& per_sm_by_dyn = per_sm_by_dyn_dev[d->device & 63];
  auto it = per_sm_by_dyn.find(dyn);
  if (it == per_sm_by_dyn.end()) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dev::k_shade<KM, kMode, kTex>, 256, dyn);
    it = per_sm_by_dyn.emplace(dyn, per_sm).first;
  }
  const int per_sm = it->second;
  const long long items = kMode == 1 ? ((long long)fc.nbins * 32 + 7) / 8 : (long long)fc.nbins;
  long long cap = (long long)std::max(1, per_sm) * d->sm_count;
  if (KM == 0 && B.dfm_g) cap = std::min<long long>(cap, B.dfm_ctas);  // scratch slices
  const int grid = int(std::max<long long>(1, std::min<long long>(cap, items)));
  pdl_launch(dev::k_shade<KM, kMode, kTex>, grid, 256, dyn, d->stream, B);
  ck(cudaGetLastError(), "k_shade launch");
  ++*launches;
}

template <int KM, bool kTex>
void launch_shade_km(DeviceScene* d, const dev::FrameConst& fc, const dev::Buffers& B,
                     int* launches) {
  if (fc.threshold) {
    launch_shade_mode<KM, 2, kTex>(d, fc, B, launches);
  } else {
    launch_shade_mode<KM, 0, kTex>(d, fc, B, launches);
    launch_shade_mode<KM, 1, kTex>(d, fc, B, launches);
  }
}

template <bool kTex>
void launch_shade_tex(DeviceScene* d, const dev::FrameConst& fc, const dev::Buffers& B, int* launches) {
  const int df = fc.df;
  // KM == df exactly up to 8 (register filters, the capacity a compile-time
  // constant); above 8 the sorted ring filter in memory (KM == 0), any capacity
  if (df == 1) launch_shade_km<1, kTex>(d, fc, B, launches);
  else if (df == 2) launch_shade_km<2, kTex>(d, fc, B, launches);
  else if (df == 3) launch_shade_km<3, kTex>(d, fc, B, launches);
  else if (df == 4) launch_shade_km<4, kTex>(d, fc, B, launches);
  else if (df == 5) launch_shade_km<5, kTex>(d, fc, B, launches);
  else if (df == 6) launch_shade_km<6, kTex>(d, fc, B, launches);
  else if (df == 7) launch_shade_km<7, kTex>(d, fc, B, launches);
  else if (df == 8) launch_shade_km<8, kTex>(d, fc, B, launches);
  else launch_shade_km<0, kTex>(d, fc, B, launches);
}

// Scenes with textured materials get the shading kernels compiled with the
// texture path; the others keep it out of their register allocation.
void launch_shade(DeviceScene* d, const dev::FrameConst& fc, const dev::Buffers& B, int* launches) {
  if (d->textured)
    launch_shade_tex<true>(d, fc, B, launches);
  else
    launch_shade_tex<false>(d, fc, B, launches);
}

template <typename T>
void dump_put(RenderOutput* out, const char* name, const T* dptr, size_t count,
              cudaStream_t stream) {
  DumpArray a;
  a.count = count;
  a.bytes.resize(count * sizeof(T));
  if (count)
    ck(cudaMemcpyAsync(a.bytes.data(), dptr, count * sizeof(T), cudaMemcpyDeviceToHost, stream),
       "dump copy");
  out->dumps[name] = std::move(a);
}

template <typename T>
void dump_put_host(RenderOutput* out, const char* name, const std::vector<T>& v) {
  DumpArray a;
  a.count = v.size();
  a.bytes.resize(v.size() * sizeof(T));
  if (!v.empty()) std::memcpy(a.bytes.data(), v.data(), a.bytes.size());
  out->dumps[name] = std::move(a);
}

struct Prepared {
  dev::FrameConst fc;
  dev::Buffers B;
  size_t zero_bytes;
  uint32_t nblocks;
  uint32_t lpair_cols_cap;
  uint32_t gcap_tbr, gcap_tb;
};

Prepared prepare(DeviceScene* d, const Scene& s, const RenderOptions& opt) {
  const veil_render_params& p = opt.params;
  const Camera& cam = s.camera;
  Prepared P;
  dev::FrameConst& fc = P.fc;
  std::memset(&fc, 0, sizeof fc);
  for (int i = 0; i < 16; ++i) fc.m[i] = cam.m[i];
  camera_vectors(cam, &fc);
  fc.width = cam.width;
  fc.height = cam.height;
  fc.bins_x = (cam.width + kBinSize - 1) / kBinSize;
  fc.bins_y = (cam.height + kBinSize - 1) / kBinSize;
  fc.nbins = fc.bins_x * fc.bins_y;
  fc.backface = (p.flags & VEIL_RENDER_BACKFACE_CULLING) ? 1 : 0;
  fc.extended = s.extended ? 1 : 0;
  fc.nquads = d->nquads;
  {
    // normalize(light_dir) in float, math.hpp:80-85
    float l[3] = {p.light_dir[0], p.light_dir[1], p.light_dir[2]};
    float l2 = l[0] * l[0] + l[1] * l[1] + l[2] * l[2];
    if (l2 <= 0.0f) {
      fc.light[0] = fc.light[1] = fc.light[2] = 0.0f;
    } else {
      float inv = 1.0f / std::sqrt(l2);
      for (int i = 0; i < 3; ++i) fc.light[i] = l[i] * inv;
    }
  }
  fc.ambient = p.ambient;
  float a = p.background[3];
  fc.bg[0] = p.background[0] * a;
  fc.bg[1] = p.background[1] * a;
  fc.bg[2] = p.background[2] * a;
  fc.bg[3] = a;
  fc.df = std::max(1, p.depth_filter_size);
  fc.threshold = (p.flags & VEIL_RENDER_ALPHA_THRESHOLD) ? 1 : 0;
  fc.visualize = (p.flags & VEIL_RENDER_VISUALIZE_ERRORS) ? 1 : 0;
  fc.force_high = (p.flags & VEIL_RENDER_FORCE_HIGH_PATH) ? 1 : 0;
  // limits, renderer.cpp:130-142
  fc.low = {1024, 256, 256, 4095};
  fc.high = {16384, 4096, 4096, 0xffffffffu};
  if (p.limit_low_tbr) fc.low.tbr = p.limit_low_tbr;
  if (p.limit_low_tri_blocks) fc.low.tb = fc.low.thb = p.limit_low_tri_blocks;
  if (p.limit_low_frags) fc.low.frags = p.limit_low_frags;
  if (p.limit_high_tbr) fc.high.tbr = p.limit_high_tbr;
  if (p.limit_high_thb) fc.high.thb = p.limit_high_thb;
  // visible-triangle index space: 24 bits like the reference (setup.hpp:32),
  // 27 bits with extended limits (sort keys pack 22 depth + 1 + 27 + 14 bits)
  fc.tri_cap = s.extended ? (1u << 27) : (1u << 24);
  fc.rank = opt.rank;
  fc.world = opt.world_size;
  if (opt.world_size > 1 && opt.rank != 0 && d->peer_fb) {
    // the root's framebuffer has the stride and size of the viewport it was
    // exported with: a later viewport change must not write through it
    if (d->peer_w != cam.width || d->peer_h != cam.height)
      throw Error(VEIL_ERR_INVALID_ARG,
                  "the imported peer framebuffer has another viewport (re-import it after "
                  "veil_scene_set_viewport)");
    fc.peer_fb = static_cast<uint32_t*>(d->peer_fb);
    fc.peer_mask = static_cast<uint8_t*>(d->peer_mask);
  }
  fc.dump = opt.dump ? 1 : 0;
  // Only the parity dumps need each bin's list in the reference's canonical
  // order: the rasterizer orders tri-blocks by (depth, large, triangle) keys
  // and counts limits, so it is independent of the order of a bin's items.
  // VEIL_BIN_SORT=0/1 forces the choice (tests check dumps of unsorted lists).
  fc.sort_bins = opt.dump ? 1 : 0;
  if (const char* bs = std::getenv("VEIL_BIN_SORT")) fc.sort_bins = std::atoi(bs) ? 1 : 0;
  if (const char* wm = std::getenv("VEIL_WALK_MIN")) fc.walk_min = std::atoi(wm);
  if (const char* wm = std::getenv("VEIL_WALK_MIN_U")) fc.walk_min_u = std::atoi(wm);
  if (const char* w1 = std::getenv("VEIL_WAVE1")) fc.wave1 = std::atoi(w1);
  fc.bulk_stage = 1;  // measured: C2 shade -0.3%, C4 shade -1.1% against the lane loop
  if (const char* bs = std::getenv("VEIL_BULK_STAGE")) fc.bulk_stage = std::atoi(bs);
  fc.fill_split = 1;
  if (const char* fs = std::getenv("VEIL_FILL_SPLIT")) fc.fill_split = std::atoi(fs);

  const uint32_t Q = d->nquads;
  const size_t nb = size_t(fc.nbins);
  P.nblocks = (Q + dev::kSetupBlock - 1) / dev::kSetupBlock;
  // counters, per-bin counts and the setup look-back states share one
  // region, zeroed by a single memset per frame
  const size_t zero_ctr = (sizeof(dev::Counters) + 255) & ~size_t(255);
  const size_t zero_cnt = ((size_t(fc.nbins) * 8 + 255) & ~size_t(255));
  P.zero_bytes = zero_ctr + zero_cnt + std::max<size_t>(1, P.nblocks) * 8;
  d->zero.ensure(P.zero_bytes);
  d->vq_src.ensure(size_t(Q) * 4);
  d->vq_idx.ensure(size_t(Q) * 16);
  d->vq_box.ensure(size_t(Q) * 8);
  d->vq_flags.ensure(size_t(Q) * 4);
  d->vq_mat.ensure(size_t(Q) * 4);
  d->vq_col.ensure(size_t(Q) * 16);
  d->vq_nrm.ensure(size_t(Q) * 16);
  d->vq_uv.ensure(d->textured ? size_t(Q) * 32 : 32);
  d->tri.ensure(size_t(Q) * 2 * sizeof(dev::TriRec));
  d->tri_meta.ensure(size_t(Q) * 2 * 16);
  d->tri_y.ensure(size_t(Q) * 2 * 4);
  // Decoded shading records pay off when triangles cover many pixels (each
  // record is read by every sample of its triangle): >= 8 px per quad at
  // depth complexity 1.
  // Decoded shading records (and the shared-memory staging built on them)
  // carry no UVs: scenes with textured materials shade on the generic path.
  fc.decoded = !d->textured && (double)cam.width * cam.height >= 8.0 * std::max<double>(1.0, Q) ? 1 : 0;
  // Fused raster (tiny triangles: the frames without decoded records): the
  // extraction recomputes small quads' setups and shades as it goes, so the
  // 128-byte records of small quads are not stored (parity dumps still store
  // them for the tri_fn arrays). VEIL_FUSED=0/1 overrides (tests, A/B);
  // textured scenes and the a-buffer reference mode keep the separate path.
  {
    int fused = 0;  // measured slower than the separate kernels
    if (const char* fe = std::getenv("VEIL_FUSED"); fe && *fe) fused = std::atoi(fe) ? 1 : 0;
    if (d->textured || (p.flags & VEIL_RENDER_REFERENCE)) fused = 0;
    fc.fused = fused;
    if (fused) fc.decoded = 0;
    if (const char* fr = std::getenv("VEIL_FUSED_READ"); fr && *fr) fc.fused_read = std::atoi(fr) ? 1 : 0;
    fc.write_tri = (!fused || opt.dump || opt.keep_records || fc.fused_read) ? 1 : 0;
  }
  if (fc.decoded) d->shade.ensure(size_t(Q) * 2 * sizeof(dev::ShadeRec));
  d->off.ensure(nb * 4);
  d->qcur.ensure(nb * 4);
  d->tcur.ensure(nb * 4);
  d->cat.ensure(nb);
  d->bin_list0.ensure(nb * 4);
  d->bin_list1.ensure(nb * 4);
  d->prop_q.ensure(nb * 4);
  d->bin_cost.ensure(nb * 4);
  d->bin_order.ensure(nb * 4 * 8);  // up to 8 parts per bin
  d->prop.ensure(nb);
  d->slots.ensure(nb * 4 * 5 * 8);
  d->spill0.ensure(nb * 4 * 4);
  d->spill1.ensure(nb * 4 * 4);
  // VEIL_INITIAL_CAPACITY (tests): start every grow-on-demand buffer at this
  // many entries so the capacity-retry paths run on small scenes
  uint32_t init_cap = 0;
  if (const char* ic = std::getenv("VEIL_INITIAL_CAPACITY")) init_cap = uint32_t(std::strtoul(ic, nullptr, 10));
  if (d->items_cap == 0) d->items_cap = init_cap ? init_cap : std::max<uint32_t>(1u << 20, Q * 6u);
  d->items.ensure(size_t(d->items_cap) * 4);
  d->item_rows.ensure(size_t(d->items_cap));
  fc.items_cap = d->items_cap;
  const size_t npx = size_t(cam.width) * cam.height;
  d->fb.ensure(npx * 4);
  d->mask.ensure(npx);
  if (opt.dump) {
    d->hash.ensure(npx * 8);
    d->emit.ensure(npx * 4);
  }
  d->hbd.ensure(nb * 32 * sizeof(dev::HbDesc));
  d->seg_queue.ensure(nb * 32 * 16);
  if (d->lpairs_cap == 0)
    d->lpairs_cap = init_cap ? init_cap : std::max<uint32_t>(1u << 16, std::min<uint32_t>(Q * 2u, 1u << 26));
  d->lpairs.ensure(size_t(d->lpairs_cap) * sizeof(uint2));
  if (opt.world_size > 1) d->shard_tris.ensure(size_t(Q) * 2 * 4);
  {  // column-word cache of the large pairs: sized to the pair capacity, at most 64 MB
    const size_t words = std::min<size_t>(size_t(d->lpairs_cap) * size_t((fc.bins_x + 31) / 32), size_t(16) << 20);
    d->lpair_cols.ensure(words * 4);
    P.lpair_cols_cap = uint32_t(words);
  }
  fc.lpairs_cap = d->lpairs_cap;
  if (d->pool_cap == 0)
    d->pool_cap = init_cap ? init_cap : std::max<uint32_t>(1u << 22, uint32_t(std::min<size_t>(nb * 2048, 1u << 26)));
  // (+16 entries of slack: k_shade's bulk copies round list ends up to 16 bytes)
  d->pool_tri.ensure((size_t(d->pool_cap) + 16) * 4);
  d->pool_mask.ensure((size_t(d->pool_cap) + 16) * 4);
  d->pool_pre.ensure((size_t(d->pool_cap) + 16) * 4);
  d->pool_slot.ensure((size_t(d->pool_cap) + 16) * 2);
  fc.pool_cap = d->pool_cap;
  // global scratch for spilled items: capacities follow the active limits
  P.gcap_tbr = std::min<uint32_t>(std::max(fc.low.tbr, fc.high.tbr), 1u << 16);
  P.gcap_tb = std::min<uint32_t>(std::max(std::max(fc.low.tb, fc.high.tb), fc.high.thb), P.gcap_tbr);
  {  // the per-warp bitonic sort pads to a power of two
    uint32_t p2 = 1;
    while (p2 < P.gcap_tb) p2 <<= 1;
    P.gcap_tb = p2;
  }
  size_t per_cta = dev::global_scratch_bytes(P.gcap_tbr, P.gcap_tb);
  per_cta = (per_cta + 255) & ~size_t(255);
  d->raster_ctas_global = d->sm_count * 2;
  d->scratch.ensure(per_cta * d->raster_ctas_global);
  d->fb_w = cam.width;
  d->fb_h = cam.height;
  // Ring depth filters (depth_filter_size > 8): a pixel receives at most one
  // sample per THB of its half-block, and a half-block holds at most
  // max(low, high) THB-limit THBs, so min(k, that) nodes per lane suffice.
  uint32_t dfm_cap = 0, dfm_ctas = 0;
  bool dfm_global = false;
  if (fc.fused && fc.df != 3) {
    // the fused raster's filters (four warps per k_extract CTA) in global memory
    dfm_cap = std::min<uint32_t>(uint32_t(fc.df), std::max(fc.low.thb, fc.high.thb));
    if (dfm_cap > (1u << dev::MemFilter::kSlotBits))
      throw Error(VEIL_ERR_INVALID_ARG,
                  "depth_filter_size above 32768 with a THB limit above 32768 is not supported");
    const size_t ctas = std::max<size_t>(size_t(kExtractCtasPerSmMax) * d->sm_count, d->raster_ctas_global);
    d->dfm_g.ensure(ctas * 4 * dfm_cap * kDfmBytesPerEntry);
    dfm_global = true;
  } else if (fc.df > 8 && !fc.fused) {
    dfm_cap = std::min<uint32_t>(uint32_t(fc.df), std::max(fc.low.thb, fc.high.thb));
    if (dfm_cap > (1u << dev::MemFilter::kSlotBits))
      throw Error(VEIL_ERR_INVALID_ARG,
                  "depth_filter_size above 32768 with a THB limit above 32768 is not supported");
    const size_t per_cta = size_t(8) * dfm_cap * kDfmBytesPerEntry;
    const char* hg = std::getenv("VEIL_DFM_GLOBAL");
    dfm_global = (hg && *hg && *hg != '0') ||
                  size_t(dev::kStageTris) * sizeof(dev::StagedTri) + per_cta > kDfmSmemBudget;
    if (dfm_global) {
      // up to 4 CTAs per SM (the shading kernels' occupancy), fewer when the
      // scratch would pass 4 GiB
      dfm_ctas = uint32_t(d->sm_count) * 4u;
      while (dfm_ctas > uint32_t(d->sm_count) && size_t(dfm_ctas) * per_cta > (size_t(4) << 30))
        dfm_ctas -= uint32_t(d->sm_count);
      d->dfm_g.ensure(size_t(dfm_ctas) * per_cta);
    }
  }

  dev::Buffers& B = P.B;
  std::memset(&B, 0, sizeof B);
  if (fc.fused) {  // per-CTA candidate setups and TBR planes of the fused raster
    const size_t na = size_t(kExtractCtasPerSmMax) * d->sm_count, ng = size_t(d->raster_ctas_global);
    B.cs_per_cta = 4u * dev::RasterShared::kTb;
    B.tp_per_cta = dev::RasterShared::kTbr;
    B.cs_per_cta_g = 4ull * P.gcap_tb;
    B.tp_per_cta_g = P.gcap_tbr;
    B.cs_off_g = na * B.cs_per_cta;
    B.tp_off_g = na * B.tp_per_cta;
    d->cscratch.ensure((B.cs_off_g + ng * B.cs_per_cta_g) * sizeof(dev::TriRec));
    d->tplanes.ensure((B.tp_off_g + ng * B.tp_per_cta_g) * sizeof(dev::TriPlanes));
    B.cscratch = d->cscratch.as<dev::TriRec>();
    B.tplanes = d->tplanes.as<dev::TriPlanes>();
  }
  B.dfm_g = dfm_global ? d->dfm_g.as<uint8_t>() : nullptr;
  B.dfm_cap = dfm_cap;
  B.dfm_ctas = dfm_ctas;
  B.pos = d->pos.as<float4>();
  B.vcol = d->vcol.as<uint32_t>();
  B.vnrm = d->vnrm.as<uint32_t>();
  B.quads = d->quads.as<uint4>();
  B.qmat = d->qmat.as<uint32_t>();
  B.mats = d->mats.as<dev::MatDev>();
  B.vuv = d->vuv.as<float2>();
  B.texels = d->texels.as<float4>();
  B.texlev = d->texlev.as<uint4>();
  B.texdesc = d->texdesc.as<uint2>();
  B.vq_uv = d->vq_uv.as<float4>();
  B.ctr = d->zero.as<dev::Counters>();
  B.qcnt = reinterpret_cast<uint32_t*>(d->zero.as<uint8_t>() + zero_ctr);
  B.tcnt = B.qcnt + fc.nbins;
  B.block_state = reinterpret_cast<unsigned long long*>(d->zero.as<uint8_t>() + zero_ctr + zero_cnt);
  B.vq_src = d->vq_src.as<uint32_t>();
  B.vq_idx = d->vq_idx.as<uint4>();
  B.vq_box = d->vq_box.as<uint2>();
  B.vq_flags = d->vq_flags.as<uint32_t>();
  B.vq_mat = d->vq_mat.as<uint32_t>();
  B.vq_col = d->vq_col.as<uint4>();
  B.vq_nrm = d->vq_nrm.as<uint4>();
  B.tri = d->tri.as<dev::TriRec>();
  B.tri_meta = d->tri_meta.as<uint4>();
  B.tri_y = d->tri_y.as<uint32_t>();
  B.shade = fc.decoded ? d->shade.as<dev::ShadeRec>() : nullptr;
  B.off = d->off.as<uint32_t>();
  B.qcur = d->qcur.as<uint32_t>();
  B.tcur = d->tcur.as<uint32_t>();
  B.cat = d->cat.as<uint8_t>();
  B.bin_list[0] = d->bin_list0.as<uint32_t>();
  B.bin_list[1] = d->bin_list1.as<uint32_t>();
  B.prop_q = d->prop_q.as<uint32_t>();
  B.bin_cost = d->bin_cost.as<uint32_t>();
  B.bin_order = d->bin_order.as<uint32_t>();
  B.prop = d->prop.as<uint8_t>();
  B.items = d->items.as<uint32_t>();
  B.item_rows = d->item_rows.as<uint8_t>();
  B.slots = d->slots.as<unsigned long long>();
  B.spill[0] = d->spill0.as<uint32_t>();
  B.spill[1] = d->spill1.as<uint32_t>();
  B.scratch = d->scratch.as<uint8_t>();
  B.scratch_per_cta = per_cta;
  B.fb = d->fb.as<uint32_t>();
  B.mask = d->mask.as<uint8_t>();
  B.hash = opt.dump ? d->hash.as<uint64_t>() : nullptr;
  B.emit = opt.dump ? d->emit.as<uint32_t>() : nullptr;
  B.hbd = d->hbd.as<dev::HbDesc>();
  B.pool_tri = d->pool_tri.as<uint32_t>();
  B.pool_mask = d->pool_mask.as<uint32_t>();
  B.pool_pre = d->pool_pre.as<uint32_t>();
  B.seg_queue = d->seg_queue.as<uint4>();
  B.pool_slot = d->pool_slot.as<uint16_t>();
  B.lpairs = d->lpairs.as<uint2>();
  B.shard_tris = opt.world_size > 1 ? d->shard_tris.as<uint32_t>() : nullptr;
  B.lpair_cols = d->lpair_cols.as<uint32_t>();
  B.lpair_cols_cap = P.lpair_cols_cap;
  return P;
}

// Stage events: inside a graph capture they must be external event-record
// nodes (a plain record only expresses a dependency there).
void record_event(cudaEvent_t e, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive) {
    cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
  } else {
    cudaEventRecord(e, st);
  }
}

// Enqueues setup + binning; returns kernel launches.
int enqueue_front(DeviceScene* d, Prepared& P) {
  const dev::FrameConst& fc = P.fc;
  const dev::Buffers& B = P.B;
  cudaStream_t st = d->stream;
  int launches = 0;
  *d->fc_host = fc;
  ck(cudaMemcpyToSymbolAsync(dev::c_fc, d->fc_host, sizeof(dev::FrameConst), 0,
                             cudaMemcpyHostToDevice, st),
     "c_fc upload");
  ck(cudaMemsetAsync(B.ctr, 0, P.zero_bytes, st), "memset");  // counters, bin counts, look-back
  record_event(d->ev[0], st);
  if (P.nblocks) {
    pdl_launch(dev::k_setup, P.nblocks, dev::kSetupBlock, 0, st, B, P.nblocks);
    const int tgrid = int(std::min<long long>(((long long)fc.nquads * 2 + dev::kTriBlock - 1) / dev::kTriBlock,
                                              (long long)d->sm_count * 32));
    if (fc.world > 1) {
      pdl_launch(dev::k_shard_tris, std::max(1, std::min<int>(d->sm_count * 8, int((fc.nquads + 255) / 256))), 256, 0,
                 st, B);
      pdl_launch(dev::k_setup_tris<true>, std::max(1, tgrid), dev::kTriBlock, 0, st, B);
      ++launches;
    } else {
      if (fc.nquads >= (1u << 19))  // (a million triangles: the 6-CTA register budget)
        pdl_launch(dev::k_setup_tris<false, 6>, std::max(1, tgrid), dev::kTriBlock, 0, st, B);
      else
        pdl_launch(dev::k_setup_tris<false>, std::max(1, tgrid), dev::kTriBlock, 0, st, B);
    }
    launches += 2;
  }
  record_event(d->ev[1], st);
  int grid = std::max(1, std::min<int>(d->sm_count * 8, int((fc.nquads + 255) / 256)));
  if (fc.world > 1)
    pdl_launch(dev::k_bin_pass<false, true>, grid, 256, 0, st, B);
  else
    pdl_launch(dev::k_bin_pass<false, false>, grid, 256, 0, st, B);
  pdl_launch(dev::k_bin_large<false>, d->sm_count * 8, 256, 0, st, B);
  pdl_launch(dev::k_bin_scan, 1, 1024, 0, st, B);
  if (fc.world > 1)
    pdl_launch(dev::k_bin_pass<true, true>, grid, 256, 0, st, B);
  else
    pdl_launch(dev::k_bin_pass<true, false>, grid, 256, 0, st, B);
  pdl_launch(dev::k_bin_large<true>, d->sm_count * 8, 256, 0, st, B);
  launches += 5;
  if (fc.sort_bins) {
    dev::k_bin_sort<<<std::min(fc.nbins, d->sm_count * 8), 256, 0, st>>>(B);
    ++launches;
  }
  record_event(d->ev[2], st);
  return launches;
}

void read_stats(DeviceScene* d, const dev::Counters& c, const Scene& s, veil_frame_stats* st) {
  float ms[4] = {0, 0, 0, 0};
  cudaEventElapsedTime(&ms[0], d->ev[0], d->ev[1]);
  cudaEventElapsedTime(&ms[1], d->ev[1], d->ev[2]);
  float shade_ms = 0;
  cudaEventElapsedTime(&ms[2], d->ev[2], d->ev[3]);
  cudaEventElapsedTime(&ms[3], d->ev[3], d->ev[5]);
  cudaEventElapsedTime(&shade_ms, d->ev[5], d->ev[4]);
  float total = 0;
  cudaEventElapsedTime(&total, d->ev[0], d->ev[4]);
  st->setup_ms = ms[0];
  st->binning_ms = ms[1];
  st->low_raster_ms = ms[2];
  st->shade_ms = shade_ms;
  st->hi_raster_ms = ms[3];
  st->total_ms = total;
  st->samples = c.samples;
  st->fragments = c.fragments;
  st->tri_half_blocks = c.thb;
  st->segments = c.segments;
  st->input_quads = s.quads.size();
  st->visible_quads = c.cull[0];
  st->culled_degenerate = c.cull[1];
  st->culled_backfacing = c.cull[2];
  st->culled_frustum = c.cull[3];
  st->culled_between_samples = c.cull[4];
  st->bins_empty = c.bins_empty;
  st->bins_low = c.bins_low;
  st->bins_high = c.bins_high;
  st->bins_propagated = c.bins_propagated;
  st->invalid_pixels = c.invalid;
  st->bin_pairs = c.pairs;
  st->large_tris = c.large_tris;
  st->small_quads = c.small_quads;
}

const char* limit_name(int code) {
  if (code == 0) return "tri-block-rows per block-row";
  switch ((code - 1) % 3) {
    case 0: return "tri-blocks per block";
    case 1: return "tri-half-blocks per half-block";
    default: return "fragments per half-block";
  }
}

void check_frame_errors(const dev::Counters& c, const dev::FrameConst& fc) {
  if (c.error & 1u)
    throw Error(VEIL_ERR_CAPACITY, "visible primitive count exceeds 24-bit index space");
  if (c.error & 4u) throw Error(VEIL_ERR_CAPACITY, "a-buffer fragment list capacity exceeded");
  if (c.bin_error != 0ull) {
    const unsigned long long be = ~c.bin_error;
    int bin = int(be / 64), code = int(be % 64);
    throw Error(VEIL_ERR_CAPACITY, "bin (" + std::to_string(bin % fc.bins_x) + "," +
                                       std::to_string(bin / fc.bins_x) +
                                       ") exceeds high-rasterizer limit: " + limit_name(code));
  }
}

void validate_frame(const Scene& s, const RenderOptions& opt) {
  if (s.validated_version != s.geometry_version) {  // index checks once per geometry version
    validate_scene(s);
    s.validated_version = s.geometry_version;
  } else {
    validate_camera(s.camera, s.extended);
  }
  const veil_render_params& p = opt.params;
  bool reference = p.flags & VEIL_RENDER_REFERENCE;
  if (!reference && p.depth_filter_size < 1)
    throw Error(VEIL_ERR_INVALID_ARG, "depth_filter_size must be >= 1");
  int bx = (s.camera.width + kBinSize - 1) / kBinSize, by = (s.camera.height + kBinSize - 1) / kBinSize;
  if (!reference && !s.extended && bx * by > kMaxBins)
    throw Error(VEIL_ERR_CAPACITY, "bin grid exceeds 5120 bins");
  if (!reference) {
    uint32_t lt = p.limit_low_tbr ? p.limit_low_tbr : 1024;
    uint32_t ht = p.limit_high_tbr ? p.limit_high_tbr : 16384;
    uint32_t lb = p.limit_low_tri_blocks ? p.limit_low_tri_blocks : 256;
    uint32_t hb = p.limit_high_thb ? p.limit_high_thb : 4096;
    if (lt > ht || lb > hb)
      throw Error(VEIL_ERR_INVALID_ARG, "low rasterizer limits exceed high limits");
  }
}

void collect_dumps(DeviceScene* d, Prepared& P, const dev::Counters& c, RenderOutput* out) {
  cudaStream_t st = d->stream;
  const uint32_t nv = c.nvis;
  const dev::Buffers& B = P.B;
  const dev::FrameConst& fc = P.fc;
  std::vector<uint32_t> src(nv), flags(nv), mat(nv);
  std::vector<uint2> box(nv);
  std::vector<uint4> col(nv), nrm(nv), meta(size_t(nv) * 2);
  std::vector<dev::TriRec> tri(size_t(nv) * 2);
  if (nv) {
    ck(cudaMemcpyAsync(src.data(), B.vq_src, nv * 4, cudaMemcpyDeviceToHost, st), "dump");
    ck(cudaMemcpyAsync(flags.data(), B.vq_flags, nv * 4, cudaMemcpyDeviceToHost, st), "dump");
    ck(cudaMemcpyAsync(mat.data(), B.vq_mat, nv * 4, cudaMemcpyDeviceToHost, st), "dump");
    ck(cudaMemcpyAsync(box.data(), B.vq_box, nv * 8, cudaMemcpyDeviceToHost, st), "dump");
    ck(cudaMemcpyAsync(col.data(), B.vq_col, nv * 16, cudaMemcpyDeviceToHost, st), "dump");
    ck(cudaMemcpyAsync(nrm.data(), B.vq_nrm, nv * 16, cudaMemcpyDeviceToHost, st), "dump");
    ck(cudaMemcpyAsync(meta.data(), B.tri_meta, size_t(nv) * 32, cudaMemcpyDeviceToHost, st), "dump");
    ck(cudaMemcpyAsync(tri.data(), B.tri, size_t(nv) * 2 * sizeof(dev::TriRec),
                       cudaMemcpyDeviceToHost, st),
       "dump");
  }
  ck(cudaStreamSynchronize(st), "dump sync");
  std::vector<uint64_t> aabb(nv);
  std::vector<uint8_t> cls(nv), valid(size_t(nv) * 2);
  std::vector<uint32_t> attr(size_t(nv) * 9), tmeta(size_t(nv) * 8);
  std::vector<int32_t> yr(size_t(nv) * 4);
  std::vector<double> fn(size_t(nv) * 30);
  for (uint32_t i = 0; i < nv; ++i) {
    uint32_t x0 = box[i].x & 0xffff, x1 = box[i].x >> 16, y0 = box[i].y & 0xffff, y1 = box[i].y >> 16;
    uint32_t cf = (flags[i] >> 4) & 3u;
    aabb[i] = fc.extended ? (uint64_t(x0) | (uint64_t(y0) << 16) | (uint64_t(x1) << 32) | (uint64_t(y1) << 48))
                          : uint64_t(x0 | (y0 << 7) | (x1 << 14) | (y1 << 21) | (cf << 28));
    cls[i] = uint8_t((flags[i] & 15u) | (cf << 4));  // large, colours, normals, uvs, cull bits
    const uint32_t cc[4] = {col[i].x, col[i].y, col[i].z, col[i].w};
    const uint32_t nn[4] = {nrm[i].x, nrm[i].y, nrm[i].z, nrm[i].w};
    for (int k = 0; k < 4; ++k) attr[i * 9 + k] = cc[k], attr[i * 9 + 4 + k] = nn[k];
    attr[i * 9 + 8] = mat[i];
  }
  for (size_t t = 0; t < size_t(nv) * 2; ++t) {
    const dev::TriRec& r = tri[t];
    bool v = meta[t].w & 0x100u;
    valid[t] = v;
    yr[t * 2] = v ? r.y_min : 0;
    yr[t * 2 + 1] = v ? r.y_max : -1;
    const dev::Fn3* fs[5] = {&r.e[0], &r.e[1], &r.e[2], &r.iw, &r.dz};
    for (int k = 0; k < 5; ++k) {
      fn[t * 15 + k * 3] = fs[k]->a;
      fn[t * 15 + k * 3 + 1] = fs[k]->b;
      fn[t * 15 + k * 3 + 2] = fs[k]->c;
    }
    tmeta[t * 4] = meta[t].x;
    tmeta[t * 4 + 1] = meta[t].y;
    tmeta[t * 4 + 2] = meta[t].z;
    tmeta[t * 4 + 3] = meta[t].w & 0xffu;
  }
  fn.resize(size_t(nv) * 30);
  yr.resize(size_t(nv) * 4);
  tmeta.resize(size_t(nv) * 8);
  dump_put_host(out, "quad_source", src);
  dump_put_host(out, "quad_aabb", aabb);
  dump_put_host(out, "quad_class", cls);
  dump_put_host(out, "quad_attr", attr);
  dump_put_host(out, "tri_valid", valid);
  dump_put_host(out, "tri_yrange", yr);
  dump_put_host(out, "tri_fn", fn);
  dump_put_host(out, "tri_meta", tmeta);
  dump_put_host(out, "setup_stats",
                std::vector<uint64_t>{uint64_t(d->nquads), c.cull[0], c.cull[1], c.cull[2], c.cull[3], c.cull[4]});
  dump_put_host(out, "bin_dims", std::vector<int32_t>{fc.bins_x, fc.bins_y});
  const size_t nb = size_t(fc.nbins);
  dump_put(out, "bin_quad_counts", B.qcnt, nb, st);
  dump_put(out, "bin_tri_counts", B.tcnt, nb, st);
  dump_put(out, "bin_offsets", B.off, nb, st);
  dump_put(out, "bin_categories", B.cat, nb, st);
  dump_put(out, "bin_items", B.items, size_t(c.pairs), st);
  std::vector<uint8_t> prop(nb), cat(nb);
  ck(cudaMemcpyAsync(prop.data(), B.prop, nb, cudaMemcpyDeviceToHost, st), "dump");
  ck(cudaMemcpyAsync(cat.data(), B.cat, nb, cudaMemcpyDeviceToHost, st), "dump");
  ck(cudaStreamSynchronize(st), "dump sync");
  std::vector<uint8_t> path(nb);
  bool force_high = fc.force_high;
  for (size_t b = 0; b < nb; ++b) {
    if (cat[b] == 0) path[b] = 0;
    else if (cat[b] == 2 || force_high) path[b] = 2;
    else path[b] = prop[b] ? 3 : 1;
  }
  dump_put_host(out, "bin_path", path);
}

}  // namespace

static void enqueue_raster(DeviceScene* d, Prepared& P, int* launches) {
  launch_extract(d, P.fc, P.B, dev::kPassLow, P.gcap_tbr, P.gcap_tb, launches);
  record_event(d->ev[3], d->stream);
  launch_extract(d, P.fc, P.B, dev::kPassHigh, P.gcap_tbr, P.gcap_tb, launches);
  record_event(d->ev[5], d->stream);
  if (P.fc.fused) {  // the extraction shaded every non-empty bin
    pdl_launch(dev::k_fill_empty, std::min(P.fc.nbins, d->sm_count * 8), 256, 0, d->stream, P.B);
    ++*launches;
  } else {
    if (P.fc.fill_split) {
      pdl_launch(dev::k_fill_empty, std::min(P.fc.nbins, d->sm_count * 8), 256, 0, d->stream, P.B);
      ++*launches;
    }
    // (the split threshold uses mode 0's usual 2 CTAs per SM)
    pdl_launch(dev::k_order_bins, 1, 1024, 0, d->stream, P.B, uint32_t(2 * d->sm_count));
    ++*launches;
    launch_shade(d, P.fc, P.B, launches);
  }
  pdl_launch(dev::k_finalize, (P.fc.nbins + 255) / 256, 256, 0, d->stream, P.B, d->ctr_dev);
  ++*launches;
  record_event(d->ev[4], d->stream);
}

namespace {
// Frames on one device share its __constant__ c_fc: one in flight per device
// (frames on different devices run concurrently).
std::mutex& device_mutex(int device) {
  static std::mutex m[64];
  return m[device & 63];
}
}  // namespace

// One frame on workspace d (the caller holds d's device lock and validated
// the frame). peer_fb / peer_mask: the root's device framebuffer, written by
// this (non-root) shard's shading kernels next to its own (multi-device).
static void render_frame_on(DeviceScene* d, const Scene& s, const RenderOptions& opt, RenderOutput* out,
                            void* peer_fb, void* peer_mask);

void render_frame(const Scene& s, const RenderOptions& opt, RenderOutput* out) {
  std::lock_guard<std::mutex> frame_lock(device_mutex(t_device));
  validate_frame(s, opt);
  DeviceScene* d = device_scene(s);
  render_frame_on(d, s, opt, out, nullptr, nullptr);
}

static void render_frame_on(DeviceScene* d, const Scene& s, const RenderOptions& opt, RenderOutput* out,
                            void* peer_fb, void* peer_mask) {
  static const bool graphs_enabled = [] {
    const char* e = std::getenv("VEIL_NO_GRAPH");
    return !(e && *e && *e != '0');
  }();
  static const bool zero_copy_enabled = [] {
    const char* e = std::getenv("VEIL_NO_ZEROCOPY");
    return !(e && *e && *e != '0');
  }();
  // Zero-copy readback: the shading kernels write the final pixels straight
  // into the render's pinned host frame (device-mapped), so the transfer
  // overlaps the frame instead of following it.
  const size_t npx_frame = size_t(s.camera.width) * s.camera.height;
  std::shared_ptr<uint8_t> zc;
  uint8_t* zc_dev = nullptr;
  // Scattered 32-byte writes over the host link reach ~10 GB/s, a bulk copy
  // ~50 GB/s: zero-copy pays when the transfer hides inside the frame, judged
  // by this scene's previous frame time (first frames use the copy).
  const double zc_seconds = double(npx_frame) * 5.0 / 10e9;
  const bool zc_hides = d->last.total_ms * 1e-3 >= zc_seconds;
  if (zero_copy_enabled && zc_hides && opt.host_readback && !opt.dump && opt.world_size <= 1) {
    zc = acquire_host_frame(npx_frame * 5);
    void* dp = nullptr;
    if (cudaHostGetDevicePointer(&dp, zc.get(), 0) == cudaSuccess) {
      zc_dev = static_cast<uint8_t*>(dp);
    } else {
      cudaGetLastError();
      zc.reset();
    }
  }
  for (int attempt = 0; attempt < 8; ++attempt) {
    Prepared P = prepare(d, s, opt);
    if (zc_dev) {
      P.fc.host_fb = reinterpret_cast<uint32_t*>(zc_dev);
      P.fc.host_mask = zc_dev + npx_frame * 4;
    }
    if (peer_fb) {
      P.fc.peer_fb = static_cast<uint32_t*>(peer_fb);
      P.fc.peer_mask = static_cast<uint8_t*>(peer_mask);
    }
    int launches = 0;
    if (graphs_enabled && !opt.dump) {
      // One graph launch per frame. Everything a launch configuration or a
      // kernel pointer depends on is in the key; per-frame values (camera,
      // colours) reach the kernels through the c_fc memcpy node, which reads
      // the pinned staging copy when the graph executes.
      std::vector<uint8_t> key(sizeof(dev::Buffers) + sizeof(dev::FrameConst) + 12);
      dev::FrameConst kf = P.fc;
      std::memset(kf.m, 0, sizeof kf.m);
      std::memset(kf.eye, 0, sizeof kf.eye);
      std::memset(kf.fwd, 0, sizeof kf.fwd);
      std::memset(kf.light, 0, sizeof kf.light);
      std::memset(kf.bg, 0, sizeof kf.bg);
      kf.ambient = 0;
      kf.host_fb = nullptr;  // per-frame host frame: in c_fc, not the graph
      kf.host_mask = nullptr;
      kf.peer_fb = nullptr;
      kf.peer_mask = nullptr;
      std::memcpy(key.data(), &P.B, sizeof(dev::Buffers));
      std::memcpy(key.data() + sizeof(dev::Buffers), &kf, sizeof kf);
      uint32_t extra[3] = {P.nblocks, P.gcap_tbr, P.gcap_tb};
      std::memcpy(key.data() + sizeof(dev::Buffers) + sizeof kf, extra, sizeof extra);
      if (!d->graph_exec || key != d->graph_key) {
        if (d->graph_exec) {
          cudaGraphExecDestroy(d->graph_exec);
          d->graph_exec = nullptr;
        }
        cudaGraph_t g = nullptr;
        ck(cudaStreamBeginCapture(d->stream, cudaStreamCaptureModeRelaxed), "graph capture");
        int n = 0;
        try {
          n = enqueue_front(d, P);
          enqueue_raster(d, P, &n);  // (k_finalize publishes the counters to ctr_host)
        } catch (...) {
          if (cudaStreamEndCapture(d->stream, &g) == cudaSuccess && g) cudaGraphDestroy(g);
          throw;
        }
        ck(cudaStreamEndCapture(d->stream, &g), "graph capture");
        cudaError_t ie = cudaGraphInstantiate(&d->graph_exec, g, 0);
        cudaGraphDestroy(g);
        ck(ie, "cudaGraphInstantiate");
        d->graph_key = std::move(key);
        d->graph_launches = n;
      }
      *d->fc_host = P.fc;
      if (opt.ev_start) ck(cudaEventRecord(static_cast<cudaEvent_t>(opt.ev_start), d->stream), "event");
      ck(cudaGraphLaunch(d->graph_exec, d->stream), "cudaGraphLaunch");
      launches = d->graph_launches;
    } else {
      if (opt.ev_start) ck(cudaEventRecord(static_cast<cudaEvent_t>(opt.ev_start), d->stream), "event");
      launches = enqueue_front(d, P);
      enqueue_raster(d, P, &launches);
    }
    if (opt.ev_end) ck(cudaEventRecord(static_cast<cudaEvent_t>(opt.ev_end), d->stream), "event");
    ck(cudaStreamSynchronize(d->stream), "frame");
    const dev::Counters c = *d->ctr_host;
    // Grow-on-demand buffers (first frames of a scene only): the device
    // counters keep counting past a capacity, so each overflowed buffer is
    // grown to the demand seen (+25%) and the frame re-runs. A stage that
    // could not run because an earlier one overflowed shows its demand on
    // the next attempt.
    bool grow = false;
    auto grown = [](unsigned long long need) {
      return uint32_t(std::min<unsigned long long>(need + need / 4 + 1024, 0xffffffffull));
    };
    if (c.error & 2u) {  // bin items
      d->items_cap = std::max(d->items_cap, grown(c.pairs));
      grow = true;
    }
    if (c.error & 8u) {  // THB pool
      d->pool_cap = std::max(grown(c.pool_pair), uint32_t(std::min<unsigned long long>(2ull * d->pool_cap, 0xffffffffull)));
      grow = true;
    }
    if (c.error & 16u) {  // large-triangle (triangle, bin row) pairs
      d->lpairs_cap = std::max(d->lpairs_cap, grown(c.large_pairs));
      grow = true;
    }
    if (grow) continue;
    check_frame_errors(c, P.fc);
    out->width = s.camera.width;
    out->height = s.camera.height;
    read_stats(d, c, s, &out->stats);
    out->stats.kernel_launches = launches;
    d->last = out->stats;
    if (opt.dump) {
      collect_dumps(d, P, c, out);
      // tri-half-block lists from the pool in (bin, half-block) order
      const size_t nb = size_t(P.fc.nbins);
      std::vector<dev::HbDesc> hbd(nb * 32);
      std::vector<uint8_t> cat(nb);
      ck(cudaMemcpy(hbd.data(), P.B.hbd, nb * 32 * sizeof(dev::HbDesc), cudaMemcpyDeviceToHost), "dump");
      ck(cudaMemcpy(cat.data(), P.B.cat, nb, cudaMemcpyDeviceToHost), "dump");
      const size_t used = std::min<size_t>(uint32_t(c.pool_pair), d->pool_cap);
      std::vector<uint32_t> ptri(used), pmask(used), ppre(used);
      if (used) {
        ck(cudaMemcpy(ptri.data(), P.B.pool_tri, used * 4, cudaMemcpyDeviceToHost), "dump");
        ck(cudaMemcpy(pmask.data(), P.B.pool_mask, used * 4, cudaMemcpyDeviceToHost), "dump");
        ck(cudaMemcpy(ppre.data(), P.B.pool_pre, used * 4, cudaMemcpyDeviceToHost), "dump");
      }
      std::vector<uint64_t> offs(nb * 32 + 1, 0), bits;
      std::vector<uint32_t> tris, pres;
      for (size_t i = 0; i < nb * 32; ++i) {
        const int b = int(i / 32);
        const bool owned = bin_owned(b % P.fc.bins_x, b / P.fc.bins_x, opt.rank, opt.world_size);
        if (cat[b] && owned) {
          const dev::HbDesc& h = hbd[i];
          for (uint32_t k = 0; k < h.cnt; ++k) {
            const uint32_t m = pmask[h.off + k], tri = ptri[h.off + k];
            uint64_t w = 0;  // TriHalfBlock::make, packing.hpp:154-176
            for (int y = 0; y < 4; ++y) {
              const uint32_t rb = (m >> (8 * y)) & 0xffu;
              uint32_t bb = 7, ll = 0;
              if (rb) {
                bb = uint32_t(__builtin_ctz(rb));
                ll = 31u - uint32_t(__builtin_clz(rb));
              }
              w |= uint64_t(bb | (ll << 3)) << (6 * y);
            }
            const uint32_t prefix = ppre[h.off + k] + uint32_t(__builtin_popcount(m));
            bits.push_back(w | (uint64_t(tri & 0xffffffu) << 24) | (uint64_t(prefix & 0xfffu) << 48));
            tris.push_back(tri);
            pres.push_back(prefix);
          }
        }
        offs[i + 1] = bits.size();
      }
      dump_put_host(out, "thb_offsets", offs);
      dump_put_host(out, "thb", bits);
      dump_put_host(out, "thb_tri", tris);
      dump_put_host(out, "thb_prefix", pres);
      const size_t npx = size_t(s.camera.width) * s.camera.height;
      dump_put(out, "emit_hash", P.B.hash, npx, d->stream);
      dump_put(out, "emit_count", P.B.emit, npx, d->stream);
      ck(cudaStreamSynchronize(d->stream), "dump");
    }
    if (zc) {
      out->host = zc;  // already written by the kernels
    } else if (opt.host_readback || opt.dump) {
      const size_t npx = size_t(s.camera.width) * s.camera.height;
      out->host = acquire_host_frame(npx * 5);
      ck(cudaMemcpyAsync(out->rgba(), P.B.fb, npx * 4, cudaMemcpyDeviceToHost, d->stream), "readback");
      ck(cudaMemcpyAsync(out->mask(), P.B.mask, npx, cudaMemcpyDeviceToHost, d->stream), "readback");
      ck(cudaStreamSynchronize(d->stream), "readback");
    }
    if (opt.dump) {
      DumpArray img, msk;
      const size_t npx = size_t(s.camera.width) * s.camera.height;
      img.count = npx * 4;
      img.bytes.assign(out->rgba(), out->rgba() + npx * 4);
      msk.count = npx;
      msk.bytes.assign(out->mask(), out->mask() + npx);
      out->dumps["image"] = std::move(img);
      out->dumps["mask"] = std::move(msk);
      const veil_frame_stats& t = out->stats;
      dump_put_host(out, "counters",
                    std::vector<uint64_t>{t.samples, t.fragments, t.tri_half_blocks, t.segments,
                                          t.bins_empty, t.bins_low, t.bins_high, t.bins_propagated,
                                          t.invalid_pixels});
    }
    return;
  }
  throw Error(VEIL_ERR_INTERNAL, "frame buffers could not be sized after 8 attempts");
}

void render_reference_frame(const Scene& s, const RenderOptions& opt, RenderOutput* out) {
  std::lock_guard<std::mutex> frame_lock(device_mutex(t_device));
  validate_scene(s);
  DeviceScene* d = device_scene(s);
  Prepared P = prepare(d, s, opt);
  for (int attempt = 0; attempt < 8; ++attempt) {
    int launches = enqueue_front(d, P);
    dim3 grid((s.camera.width + 15) / 16, (s.camera.height + 7) / 8);
    dev::k_abuffer<<<grid, 128, 0, d->stream>>>(P.B);
    ++launches;
    record_event(d->ev[3], d->stream);
    record_event(d->ev[5], d->stream);
    record_event(d->ev[4], d->stream);
    dev::Counters c;
    ck(cudaMemcpyAsync(&c, P.B.ctr, sizeof c, cudaMemcpyDeviceToHost, d->stream), "counters");
    ck(cudaStreamSynchronize(d->stream), "frame");
    if (c.error & (2u | 16u)) {  // capacity of the bin items / large-triangle pairs
      if (c.error & 2u)
        d->items_cap = uint32_t(std::min<unsigned long long>(c.pairs + c.pairs / 4 + 1024, 0xffffffffull));
      if (c.error & 16u)
        d->lpairs_cap = uint32_t(std::min<unsigned long long>(c.large_pairs + c.large_pairs / 4 + 1024, 0xffffffffull));
      P = prepare(d, s, opt);
      continue;
    }
    check_frame_errors(c, P.fc);
    out->width = s.camera.width;
    out->height = s.camera.height;
    out->reference = true;
    read_stats(d, c, s, &out->stats);
    out->stats.fragments = c.samples;
    out->stats.tri_half_blocks = 0;
    out->stats.segments = 0;
    out->stats.bins_empty = out->stats.bins_low = out->stats.bins_high = 0;
    out->stats.setup_ms = out->stats.binning_ms = out->stats.low_raster_ms = out->stats.hi_raster_ms = 0;
    out->stats.kernel_launches = launches;
    const size_t npx = size_t(s.camera.width) * s.camera.height;
    out->host = acquire_host_frame(npx * 5);
    std::memset(out->mask(), 0, npx);
    ck(cudaMemcpy(out->rgba(), P.B.fb, npx * 4, cudaMemcpyDeviceToHost), "readback");
    if (opt.dump) {
      dump_put(out, "emit_hash", P.B.hash, npx, d->stream);
      dump_put(out, "emit_count", P.B.emit, npx, d->stream);
      ck(cudaStreamSynchronize(d->stream), "dump");
      dump_put_host(out, "image", std::vector<uint8_t>(out->rgba(), out->rgba() + npx * 4));
      dump_put_host(out, "mask", std::vector<uint8_t>(out->mask(), out->mask() + npx));
    }
    return;
  }
  throw Error(VEIL_ERR_INTERNAL, "frame buffers could not be sized after 8 attempts");
}

// One frame over several devices in this process (veil_render_scene_multi):
// shard i renders the bins owned by rank i of n (the same bin interleave as the
// one-process-per-GPU path) on devices[i], each shard in its own workspace and
// host thread, with its shading kernels writing finished pixels straight into
// shard 0's device framebuffer (peer memory over NVLink, or the same buffer
// when two shards share a device). Shard 0's framebuffer then holds the whole
// frame; it is read back once. Counters of owned bins are summed, replicated
// setup counters taken once, stage times are the maximum over shards.
void render_frame_multi(const Scene& s, const RenderOptions& opt, const int* devices, int n,
                        RenderOutput* out) {
  validate_frame(s, opt);
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    throw Error(VEIL_ERR_INTERNAL, "no CUDA device available (libveil has no CPU fallback)");
  for (int i = 0; i < n; ++i)
    if (devices[i] < 0 || devices[i] >= count) throw Error(VEIL_ERR_INVALID_ARG, "no such CUDA device");
  if (s.shards.size() < size_t(n)) s.shards.resize(size_t(n), nullptr);
  const size_t npx = size_t(s.camera.width) * s.camera.height;
  DeviceScene* root = nullptr;
  {
    std::lock_guard<std::mutex> lk(device_mutex(devices[0]));
    root = device_scene_on(s, &s.shards[0], devices[0]);
    root->fb.ensure(npx * 4);
    root->mask.ensure(npx);
  }
  for (int i = 1; i < n; ++i) {
    if (devices[i] == devices[0]) continue;
    int ok = 0;
    ck(cudaDeviceCanAccessPeer(&ok, devices[i], devices[0]), "cudaDeviceCanAccessPeer");
    if (!ok) throw Error(VEIL_ERR_INTERNAL, "device " + std::to_string(devices[i]) +
                                               " cannot write device " + std::to_string(devices[0]) +
                                               "'s memory (no peer access)");
    ck(cudaSetDevice(devices[i]), "cudaSetDevice");
    const cudaError_t e = cudaDeviceEnablePeerAccess(devices[0], 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled)
      cudaGetLastError();
    else
      ck(e, "cudaDeviceEnablePeerAccess");
  }
  std::vector<RenderOutput> outs(static_cast<size_t>(n));
  std::vector<std::exception_ptr> errs(static_cast<size_t>(n));
  std::vector<std::thread> threads;
  for (int i = 0; i < n; ++i)
    threads.emplace_back([&, i] {
      try {
        std::lock_guard<std::mutex> lk(device_mutex(devices[i]));
        t_device = devices[i];
        DeviceScene* d = i == 0 ? root : device_scene_on(s, &s.shards[size_t(i)], devices[i]);
        RenderOptions o = opt;
        o.rank = i;
        o.world_size = n;
        o.host_readback = false;
        o.dump = false;
        render_frame_on(d, s, o, &outs[size_t(i)], i ? root->fb.p : nullptr, i ? root->mask.p : nullptr);
      } catch (...) {
        errs[size_t(i)] = std::current_exception();
      }
    });
  for (auto& t : threads) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
  ck(cudaSetDevice(devices[0]), "cudaSetDevice");
  out->width = s.camera.width;
  out->height = s.camera.height;
  out->host = acquire_host_frame(npx * 5);
  ck(cudaMemcpy(out->rgba(), root->fb.p, npx * 4, cudaMemcpyDeviceToHost), "readback");
  ck(cudaMemcpy(out->mask(), root->mask.p, npx, cudaMemcpyDeviceToHost), "readback");
  veil_frame_stats& st = out->stats;
  st = outs[0].stats;  // replicated cull counters
  st.samples = st.fragments = st.tri_half_blocks = st.segments = st.invalid_pixels = 0;
  st.bins_propagated = st.bin_pairs = st.kernel_launches = 0;
  st.bins_low = st.bins_high = 0;  // a shard categorises its own bins (the others read as empty)
  const uint64_t nbins = uint64_t((s.camera.width + kBinSize - 1) / kBinSize) *
                         uint64_t((s.camera.height + kBinSize - 1) / kBinSize);
  for (const RenderOutput& o : outs) {
    const veil_frame_stats& x = o.stats;
    st.bins_low += x.bins_low;
    st.bins_high += x.bins_high;
    st.samples += x.samples;
    st.fragments += x.fragments;
    st.tri_half_blocks += x.tri_half_blocks;
    st.segments += x.segments;
    st.invalid_pixels += x.invalid_pixels;
    st.bins_propagated += x.bins_propagated;
    st.bin_pairs += x.bin_pairs;
    st.kernel_launches += x.kernel_launches;
    st.setup_ms = std::max(st.setup_ms, x.setup_ms);
    st.binning_ms = std::max(st.binning_ms, x.binning_ms);
    st.low_raster_ms = std::max(st.low_raster_ms, x.low_raster_ms);
    st.hi_raster_ms = std::max(st.hi_raster_ms, x.hi_raster_ms);
    st.shade_ms = std::max(st.shade_ms, x.shade_ms);
    st.total_ms = std::max(st.total_ms, x.total_ms);
  }
  st.bins_empty = nbins - st.bins_low - st.bins_high;
}

void shard_tiles_device(const Scene& s, int rank, int world, void* tiles, uint64_t bytes,
                        bool unpack) {
  DeviceScene* d = s.device;
  if (!d || d->fb_w != s.camera.width || d->fb_h != s.camera.height)
    throw Error(VEIL_ERR_INVALID_ARG, "scene has no device frame of its current viewport");
  ck(cudaSetDevice(d->device), "cudaSetDevice");
  const int bx = (s.camera.width + kBinSize - 1) / kBinSize, by = (s.camera.height + kBinSize - 1) / kBinSize;
  std::vector<uint32_t> bins;
  for (int y = 0; y < by; ++y)
    for (int x = 0; x < bx; ++x)
      if (bin_owned(x, y, rank, world)) bins.push_back(uint32_t(y * bx + x));
  if (bytes < bins.size() * 5120ull) throw Error(VEIL_ERR_INVALID_ARG, "tile buffer too small");
  if (bins.empty()) return;
  DevBuf& ids = d->tile_ids;
  ids.ensure(bins.size() * 4);
  ck(cudaMemcpyAsync(ids.p, bins.data(), bins.size() * 4, cudaMemcpyHostToDevice, d->stream), "tiles");
  dev::FrameConst fc;
  std::memset(&fc, 0, sizeof fc);
  fc.width = s.camera.width;
  fc.height = s.camera.height;
  fc.bins_x = bx;
  fc.bins_y = by;
  int grid = std::min<int>(int(bins.size()), d->sm_count * 8);
  dev::k_tile_copy<<<grid, 256, 0, d->stream>>>(fc, d->fb.as<uint32_t>(), d->mask.as<uint8_t>(),
                                                 reinterpret_cast<uint8_t*>(tiles), ids.as<uint32_t>(),
                                                 uint32_t(bins.size()), unpack ? 1 : 0);
  ck(cudaGetLastError(), "k_tile_copy");
  ck(cudaStreamSynchronize(d->stream), "tiles");
}

void export_framebuffer(const Scene& s, veil_ipc_framebuffer* out) {
  DeviceScene* d = device_scene(s);
  const size_t npx = size_t(s.camera.width) * s.camera.height;
  d->fb.ensure(npx * 4);
  d->mask.ensure(npx);
  cudaIpcMemHandle_t h;
  ck(cudaIpcGetMemHandle(&h, d->fb.p), "cudaIpcGetMemHandle");
  std::memcpy(out->rgba, &h, sizeof h);
  ck(cudaIpcGetMemHandle(&h, d->mask.p), "cudaIpcGetMemHandle");
  std::memcpy(out->mask, &h, sizeof h);
  out->width = s.camera.width;
  out->height = s.camera.height;
}

void import_peer_framebuffer(const Scene& s, const veil_ipc_framebuffer* fb) {
  DeviceScene* d = device_scene(s);
  if (d->peer_fb) cudaIpcCloseMemHandle(d->peer_fb);
  if (d->peer_mask) cudaIpcCloseMemHandle(d->peer_mask);
  d->peer_fb = d->peer_mask = nullptr;
  d->graph_key.clear();  // re-capture with the new constants layout
  if (!fb) return;
  if (fb->width != s.camera.width || fb->height != s.camera.height)
    throw Error(VEIL_ERR_INVALID_ARG, "peer framebuffer has another viewport");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, fb->rgba, sizeof h);
  ck(cudaIpcOpenMemHandle(&d->peer_fb, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  std::memcpy(&h, fb->mask, sizeof h);
  ck(cudaIpcOpenMemHandle(&d->peer_mask, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  d->peer_w = fb->width;
  d->peer_h = fb->height;
}

// The reference pipeline's maximum per-pixel sort disorder for these
// parameters (RenderConfig::measure_disorder): one device frame, then
// k_disorder over its THB lists.
int measure_disorder(const Scene& s, const RenderOptions& opt) {
  RenderOptions o = opt;
  o.host_readback = false;
  o.keep_records = true;  // k_disorder reads every triangle's depth plane
  std::lock_guard<std::mutex> frame_lock(device_mutex(t_device));
  validate_frame(s, o);
  DeviceScene* d = device_scene(s);
  RenderOutput out;
  render_frame_on(d, s, o, &out, nullptr, nullptr);
  Prepared P = prepare(d, s, o);  // the same buffers (no growth after a completed frame)
  DevBuf& res = d->disorder;
  res.ensure(256);
  ck(cudaMemsetAsync(res.p, 0, 4, d->stream), "memset");
  dev::k_disorder<<<d->sm_count * 8, 256, 0, d->stream>>>(P.B, res.as<int>());
  ck(cudaGetLastError(), "k_disorder");
  int v = 0;
  ck(cudaMemcpyAsync(&v, res.p, 4, cudaMemcpyDeviceToHost, d->stream), "disorder");
  ck(cudaStreamSynchronize(d->stream), "disorder");
  return v;
}

void device_framebuffer(const Scene& s, void** rgba, void** mask) {
  if (!s.device) throw Error(VEIL_ERR_INVALID_ARG, "scene has not been rendered on a device");
  if (rgba) *rgba = s.device->fb.p;
  if (mask) *mask = s.device->mask.p;
}

void* device_stream(const Scene& s) {
  DeviceScene* d = device_scene(s);
  return d->stream;
}

const veil_frame_stats& device_last_stats(const Scene& s) {
  if (!s.device) throw Error(VEIL_ERR_INVALID_ARG, "scene has not been rendered on a device");
  return s.device->last;
}

}  // namespace veil
