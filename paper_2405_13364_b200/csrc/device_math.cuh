// Bit-exact device arithmetic shared by the sm_100a kernels.
//
// The parity contract (BASELINE.json north_star) is bit-exact culling, bin
// lists and per-pixel blend order, which requires the reference's exact
// IEEE operation sequence: separate multiply and add (the build passes
// -fmad=false and never -use_fast_math), left-to-right sums, IEEE div/sqrt,
// round-half-away-from-zero for std::lround, std::min/max tie semantics.
// Each helper cites the reference expression it reproduces.
#pragma once

#include <cstdint>

namespace veil {
namespace dev {

constexpr int kBin = 32;

// std::min / std::max: min(a,b) = (b < a) ? b : a, max(a,b) = (a < b) ? b : a
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ float sminf(float a, float b) { return (b < a) ? b : a; }
__device__ __forceinline__ float smaxf(float a, float b) { return (a < b) ? b : a; }

struct Fn3 {
  double a, b, c;
};

// AffineFn::eval, setup.hpp:38: (a*px + b*py) + c
__device__ __forceinline__ double eval(const Fn3& f, double x, double y) {
  return __dadd_rn(__dadd_rn(__dmul_rn(f.a, x), __dmul_rn(f.b, y)), f.c);
}

// Per-triangle setup, 128 bytes (one L2 line): three oriented edge
// functions, 1/w and depth planes (setup.hpp:46-56) plus the pixel-row range.
struct __align__(16) TriRec {
  Fn3 e[3];
  Fn3 iw;
  Fn3 dz;
  int32_t y_min, y_max;
};
static_assert(sizeof(TriRec) == 128, "TriRec must be one cache line");

// llround for 0 <= v < 2^31: truncate, then round half away from zero on
// the exact fractional part (v - trunc(v) is representable).
__device__ __forceinline__ uint32_t round_half_away_pos(double v) {
  const uint32_t t = __double2uint_rz(v);
  return t + (__dsub_rn(v, (double)t) >= 0.5 ? 1u : 0u);
}

// quantize_depth, packing.hpp:190-195
__device__ __forceinline__ uint32_t quantize_depth(double d) {
  if (!(d > 0.0)) return 0u;
  if (d >= 1.0) return 4194303u;
  return round_half_away_pos(__dmul_rn(d, 4194303.0));
}

// quantize_channel, raster.hpp:86-90
__device__ __forceinline__ uint32_t quantize_channel(float v) {
  if (!(v > 0.0f)) return 0u;
  if (v >= 1.0f) return 255u;
  return (uint32_t)llround(__dmul_rn((double)v, 255.0));
}

// encode_normal / decode_normal, packing.hpp:33-49
__device__ __forceinline__ uint32_t enc_normal_c(float c) {
  long long q = llround(__dmul_rn((double)c, 511.0));
  if (q > 511) q = 511;
  if (q < -511) q = -511;
  return (uint32_t)q & 0x3ffu;
}
__device__ __forceinline__ uint32_t encode_normal(float x, float y, float z) {
  return enc_normal_c(x) | (enc_normal_c(y) << 10) | (enc_normal_c(z) << 20);
}
__device__ __forceinline__ float dec_normal_c(uint32_t field) {
  int32_t q = (int32_t)(field << 22) >> 22;
  return __fdiv_rn((float)q, 511.0f);
}

// pack_color / unpack_color, packing.hpp:53-66
__device__ __forceinline__ uint32_t enc_color_c(float v) {
  long long q = llround(__dmul_rn((double)v, 255.0));
  if (q < 0) q = 0;
  if (q > 255) q = 255;
  return (uint32_t)q;
}
__device__ __forceinline__ float unpack_c(uint32_t w, int shift) {
  return __fdiv_rn((float)((w >> shift) & 0xffu), 255.0f);
}

// homogeneous_pixel, setup.cpp:30-32: ((x + w) * 0.5) * width, ((w - y) * 0.5) * height
__device__ __forceinline__ void hpixel(const double c[4], int w, int h, double out[3]) {
  out[0] = __dmul_rn(__dmul_rn(__dadd_rn(c[0], c[3]), 0.5), (double)w);
  out[1] = __dmul_rn(__dmul_rn(__dsub_rn(c[3], c[1]), 0.5), (double)h);
  out[2] = c[3];
}

// cross / dot, math.hpp:68-72
__device__ __forceinline__ void cross3(const double a[3], const double b[3], double o[3]) {
  o[0] = __dsub_rn(__dmul_rn(a[1], b[2]), __dmul_rn(a[2], b[1]));
  o[1] = __dsub_rn(__dmul_rn(a[2], b[0]), __dmul_rn(a[0], b[2]));
  o[2] = __dsub_rn(__dmul_rn(a[0], b[1]), __dmul_rn(a[1], b[0]));
}
__device__ __forceinline__ double dot3(const double a[3], const double b[3]) {
  return __dadd_rn(__dadd_rn(__dmul_rn(a[0], b[0]), __dmul_rn(a[1], b[1])), __dmul_rn(a[2], b[2]));
}

// Mat4::transform of (x, y, z, 1), math.hpp:101-108 (left-to-right sums)
__device__ __forceinline__ void to_clip(const double* m, float px, float py, float pz,
                                        double out[4]) {
  const double x = px, y = py, z = pz;
#pragma unroll
  for (int r = 0; r < 4; ++r)
    out[r] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(m[r * 4 + 0], x), __dmul_rn(m[r * 4 + 1], y)),
                                 __dmul_rn(m[r * 4 + 2], z)),
                       __dmul_rn(m[r * 4 + 3], 1.0));
}

// extend_axis, setup.cpp:37-71
template <int N, int E>
__device__ __forceinline__ void extend_axis(const double* coord, const double* w,
                                            const int (*edges)[2], double limit, double* lo,
                                            double* hi) {
  bool any = false;
  double l = limit, h = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    if (w[i] > 0.0) {
      double p = __ddiv_rn(coord[i], w[i]);
      l = smin(l, p);
      h = smax(h, p);
      any = true;
    }
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    int i = edges[e][0], j = edges[e][1];
    if ((w[i] > 0.0) == (w[j] > 0.0)) continue;
    double t = __ddiv_rn(w[i], __dsub_rn(w[i], w[j]));
    double c = __dadd_rn(coord[i], __dmul_rn(__dsub_rn(coord[j], coord[i]), t));
    if (c > 0.0) {
      h = limit;
    } else if (c < 0.0) {
      l = 0.0;
    } else {
      l = 0.0;
      h = limit;
    }
    any = true;
  }
  if (!any) {
    *lo = 1.0;
    *hi = 0.0;
    return;
  }
  *lo = smax(l, 0.0);
  *hi = smin(h, limit);
}

// pixel_range, setup.cpp:194-202
__device__ __forceinline__ void pixel_range(double lo, double hi, int limit, int* first,
                                            int* last) {
  *first = 0;
  *last = -1;
  if (!(lo <= hi)) return;
  double f = ceil(__dsub_rn(lo, 0.5));
  double l = floor(__dsub_rn(hi, 0.5));
  int fi = (int)f, li = (int)l;
  *first = fi > 0 ? fi : 0;
  *last = li < limit - 1 ? li : limit - 1;
}

// covers_pixel, scanline.hpp:38-42
__device__ __forceinline__ bool covers(const TriRec& t, int px, int py) {
  double x = (double)px + 0.5, y = (double)py + 0.5;
  return eval(t.e[0], x, y) >= 0.0 && eval(t.e[1], x, y) >= 0.0 && eval(t.e[2], x, y) >= 0.0 &&
         eval(t.iw, x, y) > 0.0;
}

// scanline_row_interval, scanline.hpp:47-86 (caller checks valid / y range).
// Returns false when the row is empty within [x_first, x_last]. The four
// functions' b*y products are formed once per row and reused by every
// covers_pixel test of the refinement, which evaluates ((a*x + b*y) + c) with
// the same roundings as eval().
__device__ __forceinline__ bool row_span(const TriRec& t, int py, int x_first, int x_last,
                                         int* b_out, int* l_out) {
  const double y = (double)py + 0.5;
  double lo = (double)x_first + 0.5;
  double hi = (double)x_last + 0.5;
  double fa[4], fby[4], fc[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const Fn3& f = i < 3 ? t.e[i] : t.iw;
    fa[i] = f.a;
    fby[i] = __dmul_rn(f.b, y);
    fc[i] = f.c;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double k = __dadd_rn(fby[i], fc[i]);
    if (fa[i] == 0.0) {
      const bool ok = i == 3 ? k > 0.0 : k >= 0.0;
      if (!ok) return false;
      continue;
    }
    const double root = __ddiv_rn(-k, fa[i]);
    if (fa[i] > 0.0)
      lo = smax(lo, root);
    else
      hi = smin(hi, root);
  }
  if (!(lo <= __dadd_rn(hi, 1.0))) return false;
  int begin = (int)ceil(__dsub_rn(lo, 0.5));
  int last = (int)floor(__dsub_rn(hi, 0.5));
  if (begin < x_first) begin = x_first;
  if (last > x_last) last = x_last;
  // covers_pixel (scanline.hpp:38-42) at (px + 0.5, y)
  auto cov = [&](int px) {
    const double x = (double)px + 0.5;
    bool in = true;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double v = __dadd_rn(__dadd_rn(__dmul_rn(fa[i], x), fby[i]), fc[i]);
      in = in && (i == 3 ? v > 0.0 : v >= 0.0);
    }
    return in;
  };
  while (begin <= last && !cov(begin)) ++begin;
  while (begin > x_first && cov(begin - 1)) --begin;
  while (last >= begin && !cov(last)) --last;
  while (last < x_last && last >= begin && cov(last + 1)) ++last;
  if (begin > last) return false;
  *b_out = begin;
  *l_out = last;
  return true;
}

}  // namespace dev
}  // namespace veil
