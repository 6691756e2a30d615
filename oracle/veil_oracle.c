/*
 * veil_oracle.c -- single-threaded C restatement of the reference's
 * sort-middle OIT pipeline. TEST INFRASTRUCTURE ONLY (see veil_oracle.h).
 *
 * Every function cites the reference function it restates, as
 * file:line under /root/reference/proj. Arithmetic is written in the same
 * operation order (left-to-right sums, separate multiplies and adds; the
 * Makefile passes -ffp-contract=off) because the parity contract is
 * bit-exact culling, bin lists and per-pixel blend order.
 */
#include "veil_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- utils */

typedef struct {
  char name[32];
  void* data;
  uint64_t count;
} vo_arr;

struct vo_frame {
  vo_arr arrays[48];
  int narrays;
  char message[256];
};

static void* xcalloc(size_t n, size_t sz) {
  void* p = calloc(n ? n : 1, sz ? sz : 1);
  if (!p) {
    fprintf(stderr, "veil_oracle: out of memory\n");
    abort();
  }
  return p;
}

static void* xrealloc(void* p, size_t bytes) {
  void* q = realloc(p, bytes ? bytes : 1);
  if (!q) {
    fprintf(stderr, "veil_oracle: out of memory\n");
    abort();
  }
  return q;
}

static void add_array(vo_frame* f, const char* name, void* data, uint64_t count) {
  vo_arr* a = &f->arrays[f->narrays++];
  snprintf(a->name, sizeof a->name, "%s", name);
  a->data = data;
  a->count = count;
}

/* growable byte vector */
typedef struct {
  uint8_t* p;
  size_t n, cap;
} vec;

static void vec_push(vec* v, const void* x, size_t sz) {
  if (v->n + sz > v->cap) {
    v->cap = (v->n + sz) * 2 + 64;
    v->p = (uint8_t*)xrealloc(v->p, v->cap);
  }
  memcpy(v->p + v->n, x, sz);
  v->n += sz;
}

/* std::min / std::max semantics: min(a,b) = (b < a) ? b : a. */
static double dmin(double a, double b) { return (b < a) ? b : a; }
static double dmax(double a, double b) { return (a < b) ? b : a; }
static float fminf_std(float a, float b) { return (b < a) ? b : a; }
static float fmaxf_std(float a, float b) { return (a < b) ? b : a; }
static int imin(int a, int b) { return b < a ? b : a; }
static int imax(int a, int b) { return a < b ? b : a; }

/* ----------------------------------------------------------- constants */

enum { BIN = 32 };
static const uint32_t kHighThreshold = 1024;        /* binning.hpp:34-35 */
static const float kAlphaThreshold = 1.0f - 1.0f / 128.0f; /* raster.hpp:51 */
static const uint64_t kHashSeed = 0xcbf29ce484222325ull;
static const uint64_t kHashPrime = 0x100000001b3ull;

/* --------------------------------------------------------- packing.hpp */

/* encode_normal, packing.hpp:33-41 */
static uint32_t enc_normal_c(float c) {
  long q = lround((double)c * 511.0);
  if (q > 511) q = 511;
  if (q < -511) q = -511;
  return (uint32_t)q & 0x3ffu;
}
static uint32_t encode_normal(float x, float y, float z) {
  return enc_normal_c(x) | (enc_normal_c(y) << 10) | (enc_normal_c(z) << 20);
}
/* decode_normal, packing.hpp:43-49 */
static float dec_normal_c(uint32_t field) {
  int32_t q = (int32_t)(field << 22) >> 22;
  return (float)q / 511.0f;
}
/* pack_color / unpack_color, packing.hpp:53-66 */
static uint32_t enc_color_c(float v) {
  long q = lround((double)v * 255.0);
  if (q < 0) q = 0;
  if (q > 255) q = 255;
  return (uint32_t)q;
}
static uint32_t pack_color(const float c[4]) {
  return enc_color_c(c[0]) | (enc_color_c(c[1]) << 8) | (enc_color_c(c[2]) << 16) |
         (enc_color_c(c[3]) << 24);
}
static void unpack_color(uint32_t w, float out[4]) {
  out[0] = (float)(w & 0xffu) / 255.0f;
  out[1] = (float)((w >> 8) & 0xffu) / 255.0f;
  out[2] = (float)((w >> 16) & 0xffu) / 255.0f;
  out[3] = (float)((w >> 24) & 0xffu) / 255.0f;
}
/* quantize_depth, packing.hpp:190-195 */
static uint32_t quantize_depth(double d) {
  const double kMax = 4194303.0;
  if (!(d > 0.0)) return 0;
  if (d >= 1.0) return (uint32_t)kMax;
  return (uint32_t)lround(d * kMax);
}
/* quantize_channel, raster.hpp:86-90 */
static uint8_t quantize_channel(float v) {
  if (!(v > 0.0f)) return 0;
  if (v >= 1.0f) return 255;
  return (uint8_t)lround((double)v * 255.0);
}

/* ------------------------------------------------------------ geometry */

typedef struct {
  double a, b, c;
} fn3;

/* AffineFn::eval, setup.hpp:38: (a*px + b*py) + c */
static double fn_eval(fn3 f, double x, double y) { return f.a * x + f.b * y + f.c; }

typedef struct {
  fn3 e[3], inv_w, depth;
  int32_t y_min, y_max;
  uint32_t flat_normal, material, quad_index;
  uint8_t tri, valid;
} tri_setup;

typedef struct {
  uint32_t x0, y0, x1, y1, cull; /* bin AABB + per-triangle cull bits */
  uint32_t colors[4], normals[4];
  uint32_t material, source;
  uint8_t large, has_c, has_n, has_uv;
} vis_quad;

typedef struct {
  double m[16];
  int w, h;
  int has_eye;
  double eye[3];
  double fwd[3];
} camera_t;

/* Mat4::transform, math.hpp:101-108 (position widened, w = 1.0) */
static void to_clip(const double* m, const float p[3], double out[4]) {
  double x = p[0], y = p[1], z = p[2], w = 1.0;
  for (int r = 0; r < 4; ++r)
    out[r] = m[r * 4 + 0] * x + m[r * 4 + 1] * y + m[r * 4 + 2] * z + m[r * 4 + 3] * w;
}

/* homogeneous_pixel, setup.cpp:30-32 */
static void hpixel(const double c[4], int w, int h, double out[3]) {
  out[0] = (c[0] + c[3]) * 0.5 * w;
  out[1] = (c[3] - c[1]) * 0.5 * h;
  out[2] = c[3];
}

/* extend_axis, setup.cpp:37-71 */
static void extend_axis(const double* coord, const double* w, int count, const int (*edges)[2],
                        int nedges, double limit, double* lo, double* hi) {
  int any = 0;
  *lo = limit;
  *hi = 0.0;
  for (int i = 0; i < count; ++i) {
    if (w[i] > 0.0) {
      double p = coord[i] / w[i];
      *lo = dmin(*lo, p);
      *hi = dmax(*hi, p);
      any = 1;
    }
  }
  for (int e = 0; e < nedges; ++e) {
    int i = edges[e][0], j = edges[e][1];
    if ((w[i] > 0.0) == (w[j] > 0.0)) continue;
    double t = w[i] / (w[i] - w[j]);
    double c = coord[i] + (coord[j] - coord[i]) * t;
    if (c > 0.0) {
      *hi = limit;
    } else if (c < 0.0) {
      *lo = 0.0;
    } else {
      *lo = 0.0;
      *hi = limit;
    }
    any = 1;
  }
  if (!any) {
    *lo = 1.0;
    *hi = 0.0;
    return;
  }
  *lo = dmax(*lo, 0.0);
  *hi = dmin(*hi, limit);
}

static const int kQuadEdges[5][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {0, 2}};
static const int kTriEdges[3][2] = {{0, 1}, {1, 2}, {2, 0}};

/* screen_aabb_impl, setup.cpp:73-87 -> box {x0,y0,x1,y1} */
static void screen_aabb(const double (*clip)[4], int count, const int (*edges)[2], int nedges,
                        int w, int h, double box[4]) {
  double px[4], py[4], pw[4];
  for (int i = 0; i < count; ++i) {
    double hp[3];
    hpixel(clip[i], w, h, hp);
    px[i] = hp[0];
    py[i] = hp[1];
    pw[i] = hp[2];
  }
  extend_axis(px, pw, count, edges, nedges, (double)w, &box[0], &box[2]);
  extend_axis(py, pw, count, edges, nedges, (double)h, &box[1], &box[3]);
}

/* pixel_range, setup.cpp:194-202 */
static void pixel_range(double lo, double hi, int limit, int* first, int* last) {
  *first = 0;
  *last = -1;
  if (!(lo <= hi)) return;
  double f = ceil(lo - 0.5);
  double l = floor(hi - 0.5);
  *first = imax(0, (int)f);
  *last = imin(limit - 1, (int)l);
}

/* outside_mask, setup.cpp:93-102 */
static uint32_t outside_mask(const double c[4]) {
  uint32_t m = 0;
  if (c[0] < -c[3]) m |= 1u;
  if (c[0] > c[3]) m |= 2u;
  if (c[1] < -c[3]) m |= 4u;
  if (c[1] > c[3]) m |= 8u;
  if (c[2] < 0.0) m |= 16u;
  if (c[2] > c[3]) m |= 32u;
  return m;
}

static void cross3(const double a[3], const double b[3], double o[3]) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}
static double dot3(const double a[3], const double b[3]) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

/* inverse, scene.cpp:86-126 (Gauss-Jordan, partial pivoting) */
static int mat_inverse(const double* in, double* out) {
  double a[4][8];
  for (int i = 0; i < 4; ++i) {
    for (int j = 0; j < 4; ++j) a[i][j] = in[i * 4 + j];
    for (int j = 0; j < 4; ++j) a[i][4 + j] = (i == j) ? 1.0 : 0.0;
  }
  for (int col = 0; col < 4; ++col) {
    int pivot = col;
    for (int r = col + 1; r < 4; ++r)
      if (fabs(a[r][col]) > fabs(a[pivot][col])) pivot = r;
    if (fabs(a[pivot][col]) < 1e-14) return 0;
    if (pivot != col)
      for (int j = 0; j < 8; ++j) {
        double t = a[pivot][j];
        a[pivot][j] = a[col][j];
        a[col][j] = t;
      }
    double inv_p = 1.0 / a[col][col];
    for (int j = 0; j < 8; ++j) a[col][j] *= inv_p;
    for (int r = 0; r < 4; ++r) {
      if (r == col) continue;
      double f = a[r][col];
      if (f == 0.0) continue;
      for (int j = 0; j < 8; ++j) a[r][j] -= f * a[col][j];
    }
  }
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) out[i * 4 + j] = a[i][4 + j];
  return 1;
}

/* camera_eye / camera_forward, scene.cpp:67-84 */
static void camera_init(camera_t* cam, const veil_scene_desc* d) {
  memcpy(cam->m, d->view_projection, sizeof cam->m);
  cam->w = d->width;
  cam->h = d->height;
  cam->has_eye = 0;
  if (d->has_eye) {
    cam->has_eye = 1;
    memcpy(cam->eye, d->eye, sizeof cam->eye);
  } else {
    double inv[16];
    if (mat_inverse(cam->m, inv)) {
      double v[4] = {0.0, 0.0, 1.0, 0.0}, hv[4];
      for (int r = 0; r < 4; ++r)
        hv[r] = inv[r * 4 + 0] * v[0] + inv[r * 4 + 1] * v[1] + inv[r * 4 + 2] * v[2] +
                inv[r * 4 + 3] * v[3];
      if (!(fabs(hv[3]) < 1e-12)) {
        double s = 1.0 / hv[3];
        cam->eye[0] = hv[0] * s;
        cam->eye[1] = hv[1] * s;
        cam->eye[2] = hv[2] * s;
        cam->has_eye = 1;
      }
    }
  }
  double g[3] = {cam->m[8], cam->m[9], cam->m[10]};
  double len = sqrt(dot3(g, g));
  if (len <= 0.0) {
    cam->fwd[0] = 0.0;
    cam->fwd[1] = 0.0;
    cam->fwd[2] = 1.0;
  } else {
    double inv = 1.0 / len;
    cam->fwd[0] = g[0] * inv;
    cam->fwd[1] = g[1] * inv;
    cam->fwd[2] = g[2] * inv;
  }
}

/* triangle_front_facing, setup.cpp:104-110 */
static int front_facing(const double p[3][3], const camera_t* cam) {
  double e1[3] = {p[1][0] - p[0][0], p[1][1] - p[0][1], p[1][2] - p[0][2]};
  double e2[3] = {p[2][0] - p[0][0], p[2][1] - p[0][1], p[2][2] - p[0][2]};
  double n[3];
  cross3(e1, e2, n);
  if (cam->has_eye) {
    double v[3] = {cam->eye[0] - p[0][0], cam->eye[1] - p[0][1], cam->eye[2] - p[0][2]};
    return dot3(n, v) > 0.0;
  }
  return dot3(n, cam->fwd) < 0.0;
}

/* compute_triangle_setup, setup.cpp:209-239 */
static void triangle_setup(const double (*clip)[4], const camera_t* cam, tri_setup* s) {
  double v0[3], v1[3], v2[3], e0[3], e1[3], e2[3];
  hpixel(clip[0], cam->w, cam->h, v0);
  hpixel(clip[1], cam->w, cam->h, v1);
  hpixel(clip[2], cam->w, cam->h, v2);
  cross3(v1, v2, e0);
  cross3(v2, v0, e1);
  cross3(v0, v1, e2);
  double det = dot3(e0, v0);
  if (det == 0.0 || !isfinite(det)) return; /* stays invalid */
  double sgn = det > 0.0 ? 1.0 : -1.0;
  const double* es[3] = {e0, e1, e2};
  for (int i = 0; i < 3; ++i) {
    s->e[i].a = es[i][0] * sgn;
    s->e[i].b = es[i][1] * sgn;
    s->e[i].c = es[i][2] * sgn;
  }
  double inv_det = 1.0 / det;
  double z0 = clip[0][2], z1 = clip[1][2], z2 = clip[2][2];
  s->depth.a = (e0[0] * z0 + e1[0] * z1 + e2[0] * z2) * inv_det;
  s->depth.b = (e0[1] * z0 + e1[1] * z1 + e2[1] * z2) * inv_det;
  s->depth.c = (e0[2] * z0 + e1[2] * z1 + e2[2] * z2) * inv_det;
  s->inv_w.a = (e0[0] + e1[0] + e2[0]) * inv_det;
  s->inv_w.b = (e0[1] + e1[1] + e2[1]) * inv_det;
  s->inv_w.c = (e0[2] + e1[2] + e2[2]) * inv_det;
  double box[4];
  screen_aabb(clip, 3, kTriEdges, 3, cam->w, cam->h, box);
  int f, l;
  pixel_range(box[1], box[3], cam->h, &f, &l);
  s->y_min = f;
  s->y_max = l;
  s->valid = 1;
}

/* ------------------------------------------------------------ scanline */

/* covers_pixel, scanline.hpp:38-42 */
static int covers(const tri_setup* t, int px, int py) {
  double x = px + 0.5, y = py + 0.5;
  return fn_eval(t->e[0], x, y) >= 0.0 && fn_eval(t->e[1], x, y) >= 0.0 &&
         fn_eval(t->e[2], x, y) >= 0.0 && fn_eval(t->inv_w, x, y) > 0.0;
}

/* scanline_row_interval, scanline.hpp:47-86; returns 0 when empty */
static int row_span(const tri_setup* t, int py, int x_first, int x_last, int* b_out,
                    int* l_out) {
  if (!t->valid || py < t->y_min || py > t->y_max) return 0;
  double y = py + 0.5;
  double lo = x_first + 0.5;
  double hi = x_last + 0.5;
  const fn3* fns[4] = {&t->e[0], &t->e[1], &t->e[2], &t->inv_w};
  for (int i = 0; i < 4; ++i) {
    const fn3* f = fns[i];
    double k = f->b * y + f->c;
    if (f->a == 0.0) {
      int ok = i == 3 ? k > 0.0 : k >= 0.0;
      if (!ok) return 0;
      continue;
    }
    double root = -k / f->a;
    if (f->a > 0.0)
      lo = dmax(lo, root);
    else
      hi = dmin(hi, root);
  }
  if (!(lo <= hi + 1.0)) return 0;
  int begin = imax(x_first, (int)ceil(lo - 0.5));
  int last = imin(x_last, (int)floor(hi - 0.5));
  while (begin <= last && !covers(t, begin, py)) ++begin;
  while (begin > x_first && covers(t, begin - 1, py)) --begin;
  while (last >= begin && !covers(t, last, py)) --last;
  while (last < x_last && last >= begin && covers(t, last + 1, py)) ++last;
  if (begin > last) return 0;
  *b_out = begin;
  *l_out = last;
  return 1;
}

/* -------------------------------------------------------------- frame */

typedef struct {
  const veil_scene_desc* sc;
  const veil_render_params* prm;
  int extended;
  camera_t cam;
  /* setup outputs */
  uint32_t nvis;
  vis_quad* vq;
  tri_setup* ts;
  uint64_t stats[6];
  /* bins */
  int bx, by, nbins;
  uint32_t *qcnt, *tcnt, *off, *items;
  uint8_t* cat;
  uint64_t nitems;
  /* raster */
  float light[3];
  float bg[4];
  uint8_t* image;
  uint8_t* mask;
  uint64_t* hash;
  uint64_t* hash_std;
  uint32_t* emit;
  int df;
  int threshold;
} ctx_t;

static int fail(vo_frame* f, int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(f->message, sizeof f->message, fmt, ap);
  va_end(ap);
  return status;
}

/* validate_camera / validate_scene, scene.cpp:38-61 */
static int validate(vo_frame* f, const veil_scene_desc* d, int extended) {
  int maxw = extended ? 16384 : 2560, maxh = extended ? 16384 : 2048;
  if (d->width <= 0 || d->height <= 0)
    return fail(f, VEIL_ERR_INVALID_ARG, "viewport dimensions must be positive");
  if (d->width > maxw || d->height > maxh)
    return fail(f, VEIL_ERR_INVALID_ARG, "viewport exceeds the 2560x2048 limit");
  for (uint64_t i = 0; i < d->quad_count; ++i) {
    for (int k = 0; k < 4; ++k)
      if (d->quads[i].v[k] >= d->vertex_count)
        return fail(f, VEIL_ERR_INVALID_ARG, "quad %llu references vertex %u out of range",
                    (unsigned long long)i, d->quads[i].v[k]);
    if (d->quads[i].material >= d->material_count)
      return fail(f, VEIL_ERR_INVALID_ARG, "quad %llu references material out of range",
                  (unsigned long long)i);
  }
  return VEIL_OK;
}

typedef struct {
  double clip[4][4];
  double world[4][3];
  int deg[2];
} quad_geo;

/* project_quad, setup.cpp:119-131 */
static void project_quad(const ctx_t* c, const veil_quad* q, quad_geo* g) {
  for (int i = 0; i < 4; ++i) {
    const float* p = c->sc->vertices[q->v[i]].position;
    g->world[i][0] = p[0];
    g->world[i][1] = p[1];
    g->world[i][2] = p[2];
    to_clip(c->cam.m, p, g->clip[i]);
  }
  /* triangle_degenerate on (v0,v1,v2) and (v0,v2,v3), scene.hpp:54-68 */
  g->deg[0] = q->v[0] == q->v[1] || q->v[1] == q->v[2] || q->v[0] == q->v[2];
  g->deg[1] = q->v[0] == q->v[2] || q->v[2] == q->v[3] || q->v[0] == q->v[3];
}

enum { CULL_NONE = 0, CULL_DEGENERATE, CULL_BACKFACE, CULL_FRUSTUM, CULL_BETWEEN };

/* cull_projected, setup.cpp:133-186; returns the reason, fills q on visible */
static int cull(const ctx_t* c, const quad_geo* g, vis_quad* q) {
  uint32_t flags = 0;
  if (g->deg[0]) flags |= 1u;
  if (g->deg[1]) flags |= 2u;
  if (g->deg[0] && g->deg[1]) return CULL_DEGENERATE;
  if (c->prm->flags & VEIL_RENDER_BACKFACE_CULLING) {
    int back[2];
    static const int corners[2][3] = {{0, 1, 2}, {0, 2, 3}};
    for (int t = 0; t < 2; ++t) {
      if (g->deg[t]) {
        back[t] = 1;
        continue;
      }
      double p[3][3];
      for (int i = 0; i < 3; ++i) memcpy(p[i], g->world[corners[t][i]], sizeof p[i]);
      back[t] = !front_facing(p, &c->cam);
      if (back[t]) flags |= 1u << t;
    }
    if (back[0] && back[1]) return CULL_BACKFACE;
  }
  uint32_t out = outside_mask(g->clip[0]) & outside_mask(g->clip[1]) &
                 outside_mask(g->clip[2]) & outside_mask(g->clip[3]);
  if (out != 0) return CULL_FRUSTUM;
  double box[4];
  screen_aabb(g->clip, 4, kQuadEdges, 5, c->cam.w, c->cam.h, box);
  int xf, xl, yf, yl;
  pixel_range(box[0], box[2], c->cam.w, &xf, &xl);
  pixel_range(box[1], box[3], c->cam.h, &yf, &yl);
  if (box[0] > box[2] || box[1] > box[3] || xf > xl || yf > yl) return CULL_BETWEEN;
  q->x0 = (uint32_t)(xf / BIN);
  q->y0 = (uint32_t)(yf / BIN);
  q->x1 = (uint32_t)(xl / BIN);
  q->y1 = (uint32_t)(yl / BIN);
  q->cull = flags;
  q->large = (q->x1 - q->x0 + 1) * (q->y1 - q->y0 + 1) > 4;
  return CULL_NONE;
}

/* run_setup, setup.cpp:241-351 (chunking has no semantic effect) */
static int run_setup(vo_frame* f, ctx_t* c) {
  const veil_scene_desc* d = c->sc;
  uint32_t* vis_idx = (uint32_t*)xcalloc(d->quad_count, sizeof(uint32_t));
  vis_quad* tmp = (vis_quad*)xcalloc(d->quad_count, sizeof(vis_quad));
  uint64_t nvis = 0;
  memset(c->stats, 0, sizeof c->stats);
  for (uint64_t i = 0; i < d->quad_count; ++i) {
    quad_geo g;
    project_quad(c, &d->quads[i], &g);
    vis_quad q;
    memset(&q, 0, sizeof q);
    int reason = cull(c, &g, &q);
    ++c->stats[0];
    if (reason == CULL_NONE) {
      ++c->stats[1];
      tmp[nvis] = q;
      vis_idx[nvis++] = (uint32_t)i;
    } else {
      ++c->stats[1 + reason];
    }
  }
  uint64_t tri_cap = c->extended ? (1ull << 31) : (1ull << 24);
  if (nvis * 2 > tri_cap) {
    free(vis_idx);
    free(tmp);
    return fail(f, VEIL_ERR_CAPACITY, "visible primitive count exceeds 24-bit index space");
  }
  if (!c->extended) {
    for (uint64_t s = 0; s < nvis; ++s)
      if (tmp[s].x0 > 127 || tmp[s].y0 > 127 || tmp[s].x1 > 127 || tmp[s].y1 > 127) {
        free(vis_idx);
        free(tmp);
        return fail(f, VEIL_ERR_CAPACITY, "bin AABB coordinate exceeds 7 bits");
      }
  }
  c->nvis = (uint32_t)nvis;
  c->vq = tmp;
  c->ts = (tri_setup*)xcalloc(nvis * 2, sizeof(tri_setup));
  for (uint64_t s = 0; s < nvis; ++s) {
    uint32_t qi = vis_idx[s];
    const veil_quad* quad = &d->quads[qi];
    const veil_material* mat = &d->materials[quad->material];
    vis_quad* rec = &c->vq[s];
    quad_geo g;
    project_quad(c, quad, &g);
    rec->material = quad->material;
    rec->source = qi;
    rec->has_c = (mat->flags & VEIL_MATERIAL_VERTEX_COLORS) && (d->flags & VEIL_SCENE_HAS_COLORS);
    rec->has_n =
        (mat->flags & VEIL_MATERIAL_VERTEX_NORMALS) && (d->flags & VEIL_SCENE_HAS_NORMALS);
    rec->has_uv = (mat->flags & VEIL_MATERIAL_UVS) && (d->flags & VEIL_SCENE_HAS_UVS) &&
                  mat->texture >= 0;
    for (int v = 0; v < 4; ++v) {
      const veil_vertex* vx = &d->vertices[quad->v[v]];
      if (rec->has_c) rec->colors[v] = pack_color(vx->color);
      if (rec->has_n) rec->normals[v] = encode_normal(vx->normal[0], vx->normal[1], vx->normal[2]);
    }
    static const int corners[2][3] = {{0, 1, 2}, {0, 2, 3}};
    for (int t = 0; t < 2; ++t) {
      tri_setup* ts = &c->ts[s * 2 + t];
      if (rec->cull & (1u << t)) continue;
      double clip[3][4], w[3][3];
      for (int k = 0; k < 3; ++k) {
        memcpy(clip[k], g.clip[corners[t][k]], sizeof clip[k]);
        memcpy(w[k], g.world[corners[t][k]], sizeof w[k]);
      }
      triangle_setup(clip, &c->cam, ts);
      /* flat normal: normalize(cross(w1-w0, w2-w0)), math.hpp:80-85 */
      double a[3] = {w[1][0] - w[0][0], w[1][1] - w[0][1], w[1][2] - w[0][2]};
      double b[3] = {w[2][0] - w[0][0], w[2][1] - w[0][1], w[2][2] - w[0][2]};
      double n[3];
      cross3(a, b, n);
      double len2 = dot3(n, n);
      if (len2 <= 0.0) {
        n[0] = n[1] = n[2] = 0.0;
      } else {
        double inv = 1.0 / sqrt(len2);
        n[0] = n[0] * inv;
        n[1] = n[1] * inv;
        n[2] = n[2] * inv;
      }
      ts->flat_normal = encode_normal((float)n[0], (float)n[1], (float)n[2]);
      ts->material = quad->material;
      ts->quad_index = (uint32_t)s;
      ts->tri = (uint8_t)t;
    }
  }
  free(vis_idx);
  return VEIL_OK;
}

/* rasterize_triangle_bins, binning.hpp:89-117: calls sink per covered bin */
typedef void (*bin_sink)(ctx_t* c, int bin, uint32_t prim, int pass);
static void tri_bins(ctx_t* c, const tri_setup* t, uint32_t prim, int pass, bin_sink sink) {
  if (!t->valid) return;
  int w = c->cam.w;
  int words = (c->bx + 63) / 64;
  uint64_t mask[8];
  int y = t->y_min;
  while (y <= t->y_max) {
    int bin_row = y / BIN;
    int row_end = imin(t->y_max, (bin_row + 1) * BIN - 1);
    memset(mask, 0, sizeof mask);
    for (; y <= row_end; ++y) {
      int b, l;
      if (!row_span(t, y, 0, w - 1, &b, &l)) continue;
      for (int k = b / BIN; k <= l / BIN; ++k) mask[k >> 6] |= 1ull << (k & 63);
    }
    for (int wd = 0; wd < words; ++wd)
      for (int k = 0; k < 64; ++k)
        if ((mask[wd] >> k) & 1) {
          int bcol = wd * 64 + k;
          if (bcol < c->bx) sink(c, bin_row * c->bx + bcol, prim, pass);
        }
  }
}

static uint32_t* g_cursor; /* write cursors for the current frame (single-threaded) */

static void sink_count(ctx_t* c, int bin, uint32_t prim, int pass) {
  (void)prim;
  if (pass == 0)
    c->qcnt[bin]++;
  else
    c->tcnt[bin]++;
}
static void sink_write(ctx_t* c, int bin, uint32_t prim, int pass) {
  (void)pass;
  c->items[g_cursor[bin]++] = prim;
}

/* run_binning, binning.cpp:75-189; ordering per SPEC.md:292 */
static int run_binning(vo_frame* f, ctx_t* c) {
  c->bx = (c->cam.w + BIN - 1) / BIN;
  c->by = (c->cam.h + BIN - 1) / BIN;
  c->nbins = c->bx * c->by;
  if (!c->extended && c->nbins > 5120)
    return fail(f, VEIL_ERR_CAPACITY, "bin grid exceeds 5120 bins");
  int nb = c->nbins;
  c->qcnt = (uint32_t*)xcalloc(nb, 4);
  c->tcnt = (uint32_t*)xcalloc(nb, 4);
  c->off = (uint32_t*)xcalloc(nb, 4);
  c->cat = (uint8_t*)xcalloc(nb, 1);
  for (int pass = 0; pass < 2; ++pass) {
    bin_sink sink = pass == 0 ? sink_count : sink_write;
    if (pass == 1) {
      uint64_t sum = 0;
      for (int b = 0; b < nb; ++b) {
        c->off[b] = (uint32_t)sum;
        sum += (uint64_t)c->qcnt[b] + c->tcnt[b];
        uint32_t eq = 2 * c->qcnt[b] + c->tcnt[b];
        c->cat[b] = eq == 0 ? 0 : (eq < kHighThreshold ? 1 : 2);
      }
      c->nitems = sum;
      c->items = (uint32_t*)xcalloc(sum, 4);
      g_cursor = (uint32_t*)xcalloc(nb, 4);
      for (int b = 0; b < nb; ++b) g_cursor[b] = c->off[b];
    }
    /* small quads ascending: every bin of the AABB (binning.hpp:76-81) */
    for (uint32_t q = 0; q < c->nvis; ++q) {
      const vis_quad* v = &c->vq[q];
      if (v->large) continue;
      for (uint32_t yy = v->y0; yy <= v->y1; ++yy)
        for (uint32_t xx = v->x0; xx <= v->x1; ++xx)
          if (pass == 0)
            c->qcnt[yy * c->bx + xx]++;
          else
            sink(c, (int)(yy * c->bx + xx), q, 0);
    }
    if (pass == 1)
      for (int b = 0; b < nb; ++b) g_cursor[b] = c->off[b] + c->qcnt[b];
    /* valid triangles of large quads ascending */
    for (uint32_t q = 0; q < c->nvis; ++q) {
      if (!c->vq[q].large) continue;
      for (uint32_t t = 0; t < 2; ++t) tri_bins(c, &c->ts[q * 2 + t], q * 2 + t, 1, sink);
    }
  }
  free(g_cursor);
  g_cursor = NULL;
  return VEIL_OK;
}

/* ---------------------------------------------------------- raster */

typedef struct {
  uint8_t b[8], l[8]; /* per row, empty = (31,0) */
  uint32_t cols;
  uint32_t tri;
} tbr_t;

typedef struct {
  uint8_t b[4], l[4]; /* empty = (7,0) */
  uint32_t tri;
  uint32_t prefix;
} thb_t;

typedef struct {
  uint32_t max_tbr, max_tb, max_thb, max_frags;
} limits_t;

typedef struct {
  uint64_t key;
  uint32_t ref;
} sortrec;

static int cmp_sortrec(const void* a, const void* b) {
  uint64_t x = ((const sortrec*)a)->key, y = ((const sortrec*)b)->key;
  return x < y ? -1 : (x > y ? 1 : 0);
}

typedef struct {
  tbr_t* tbr[4];
  uint32_t ntbr[4], cap_tbr[4];
  thb_t* thb[32];
  uint32_t nthb[32], cap_thb[32];
  sortrec* sr;
  uint32_t cap_sr;
  char err[96];
} bin_scratch;

static void push_tbr(bin_scratch* s, int r, const tbr_t* t) {
  if (s->ntbr[r] == s->cap_tbr[r]) {
    s->cap_tbr[r] = s->cap_tbr[r] * 2 + 16;
    s->tbr[r] = (tbr_t*)xrealloc(s->tbr[r], s->cap_tbr[r] * sizeof(tbr_t));
  }
  s->tbr[r][s->ntbr[r]++] = *t;
}

static void push_thb(bin_scratch* s, int h, const thb_t* t) {
  if (s->nthb[h] == s->cap_thb[h]) {
    s->cap_thb[h] = s->cap_thb[h] * 2 + 16;
    s->thb[h] = (thb_t*)xrealloc(s->thb[h], s->cap_thb[h] * sizeof(thb_t));
  }
  s->thb[h][s->nthb[h]++] = *t;
}

/* generate_tri_block_rows, raster.cpp:41-98. Returns 1 ok, 0 overflow. */
static int gen_tbr(ctx_t* c, bin_scratch* s, int bin, const limits_t* lim, int hard) {
  for (int r = 0; r < 4; ++r) s->ntbr[r] = 0;
  int bxi = bin % c->bx, byi = bin / c->bx;
  int px0 = bxi * BIN, py0 = byi * BIN;
  int px_last = imin(px0 + BIN - 1, c->cam.w - 1);
  int py_last = imin(py0 + BIN - 1, c->cam.h - 1);
  uint32_t nq = c->qcnt[bin], nt = c->tcnt[bin];
  const uint32_t* it = c->items + c->off[bin];
  for (uint32_t i = 0; i < nq * 2 + nt; ++i) {
    uint32_t tri_index = i < nq * 2 ? it[i / 2] * 2 + (i & 1) : it[nq + (i - nq * 2)];
    const tri_setup* t = &c->ts[tri_index];
    if (!t->valid) continue;
    int yb = imax(t->y_min, py0), ye = imin(t->y_max, py_last);
    if (yb > ye) continue;
    for (int r = (yb - py0) / 8; r <= (ye - py0) / 8; ++r) {
      tbr_t rec;
      memset(rec.b, 31, 8);
      memset(rec.l, 0, 8);
      rec.cols = 0;
      rec.tri = tri_index;
      int any = 0;
      for (int ly = 0; ly < 8; ++ly) {
        int py = py0 + r * 8 + ly;
        if (py < yb || py > ye) continue;
        int b, l;
        if (!row_span(t, py, px0, px_last, &b, &l)) continue;
        rec.b[ly] = (uint8_t)(b - px0);
        rec.l[ly] = (uint8_t)(l - px0);
        for (int col = (b - px0) >> 3; col <= (l - px0) >> 3; ++col) rec.cols |= 1u << col;
        any = 1;
      }
      if (!any) continue;
      if (s->ntbr[r] >= lim->max_tbr) {
        if (hard) snprintf(s->err, sizeof s->err, "tri-block-rows per block-row");
        return 0;
      }
      push_tbr(s, r, &rec);
    }
  }
  return 1;
}

/* extract_half_blocks, raster.cpp:100-199 */
static int extract(ctx_t* c, bin_scratch* s, int bin, int block, const limits_t* lim,
                   int hard) {
  int brow = block / 4, bcol = block % 4;
  int bxi = bin % c->bx, byi = bin / c->bx;
  double bpx0 = bxi * BIN + bcol * 8;
  double bpy0 = byi * BIN + brow * 8;
  int upper = block * 2;
  s->nthb[upper] = s->nthb[upper + 1] = 0;
  const tbr_t* rows = s->tbr[brow];
  uint32_t n = 0;
  for (uint32_t i = 0; i < s->ntbr[brow]; ++i) {
    if (!(rows[i].cols & (1u << bcol))) continue;
    if (n >= lim->max_tb) {
      if (hard) snprintf(s->err, sizeof s->err, "tri-blocks per block");
      return 0;
    }
    if (n == s->cap_sr) {
      s->cap_sr = s->cap_sr * 2 + 64;
      s->sr = (sortrec*)xrealloc(s->sr, s->cap_sr * sizeof(sortrec));
    }
    s->sr[n].key = 0;
    s->sr[n].ref = i;
    ++n;
  }
  int packed = lim->max_tb <= 1024;
  uint32_t c0 = (uint32_t)bcol * 8, c1 = (uint32_t)bcol * 8 + 7;
  for (uint32_t k = 0; k < n; ++k) {
    const tbr_t* rw = &rows[s->sr[k].ref];
    uint32_t count = 0, sx = 0, sy = 0;
    for (int ly = 0; ly < 8; ++ly) {
      uint32_t b = rw->b[ly], l = rw->l[ly];
      if (b > l) continue;
      if (b < c0) b = c0;
      if (l > c1) l = c1;
      if (b > l) continue;
      uint32_t m = l - b + 1;
      count += m;
      sx += (b + l) * m / 2 - c0 * m;
      sy += (uint32_t)ly * m;
    }
    uint32_t q;
    if (count == 0) {
      q = 0x3fffffu;
    } else {
      double cx = bpx0 + (double)sx / (double)count + 0.5;
      double cy = bpy0 + (double)sy / (double)count + 0.5;
      q = quantize_depth(fn_eval(c->ts[rw->tri].depth, cx, cy));
    }
    s->sr[k].key = packed ? (uint64_t)((q << 10) | (k & 0x3ffu)) : (((uint64_t)q << 12) | k);
  }
  qsort(s->sr, n, sizeof(sortrec), cmp_sortrec);
  uint32_t prefix[2] = {0, 0};
  for (uint32_t k = 0; k < n; ++k) {
    const tbr_t* rw = &rows[s->sr[k].ref];
    for (int half = 0; half < 2; ++half) {
      thb_t h;
      memset(h.b, 7, 4);
      memset(h.l, 0, 4);
      uint32_t frags = 0;
      for (int ly = 0; ly < 4; ++ly) {
        uint32_t b = rw->b[half * 4 + ly], l = rw->l[half * 4 + ly];
        if (b > l) continue;
        if (b < c0) b = c0;
        if (l > c1) l = c1;
        if (b > l) continue;
        h.b[ly] = (uint8_t)(b - c0);
        h.l[ly] = (uint8_t)(l - c0);
        frags += l - b + 1;
      }
      if (frags == 0) continue;
      int hb = upper + half;
      if (s->nthb[hb] >= lim->max_thb) {
        if (hard) snprintf(s->err, sizeof s->err, "tri-half-blocks per half-block");
        return 0;
      }
      prefix[half] += frags;
      if (prefix[half] > lim->max_frags) {
        if (hard) snprintf(s->err, sizeof s->err, "fragments per half-block");
        return 0;
      }
      h.tri = rw->tri;
      h.prefix = prefix[half];
      push_thb(s, hb, &h);
    }
  }
  return 1;
}

typedef struct {
  uint64_t samples, fragments, thb, segments;
} bin_stats;

/* DepthFilter, depth_filter.hpp:31-92, stored ascending (min first) */
typedef struct {
  uint64_t* key;
  float (*col)[4];
  int n;
  uint64_t max_key;
  int any;
} dfilter;

static void df_insert(dfilter* f, uint64_t key, const float col[4]) {
  int pos = f->n;
  while (pos > 0 && f->key[pos - 1] > key) {
    f->key[pos] = f->key[pos - 1];
    memcpy(f->col[pos], f->col[pos - 1], sizeof f->col[pos]);
    --pos;
  }
  f->key[pos] = key;
  memcpy(f->col[pos], col, sizeof f->col[pos]);
  f->n++;
}

static void df_pop(dfilter* f, uint64_t* key, float col[4], int* ooo) {
  *key = f->key[0];
  memcpy(col, f->col[0], sizeof f->col[0]);
  memmove(f->key, f->key + 1, (size_t)(f->n - 1) * sizeof(uint64_t));
  memmove(f->col, f->col + 1, (size_t)(f->n - 1) * sizeof f->col[0]);
  f->n--;
  *ooo = f->any && *key < f->max_key;
  if (!f->any || *key > f->max_key) f->max_key = *key;
  f->any = 1;
}

/* blend_front_to_back, shading.hpp:62-66 */
static void blend(float acc[4], const float s[4]) {
  float t = 1.0f - acc[3];
  acc[0] = acc[0] + t * s[0];
  acc[1] = acc[1] + t * s[1];
  acc[2] = acc[2] + t * s[2];
  acc[3] = acc[3] + t * s[3];
}

/* make_sample_context (shading.cpp:24-77) + shade_sample (123-139), no
 * textures (array scenes have none). Returns color; *depth_out = depth. */
static void shade(const ctx_t* c, uint32_t tri_index, int px, int py, float out[4],
                  double* depth_out) {
  const tri_setup* t = &c->ts[tri_index];
  const vis_quad* q = &c->vq[tri_index / 2];
  double x = px + 0.5, y = py + 0.5;
  double e0 = fn_eval(t->e[0], x, y), e1 = fn_eval(t->e[1], x, y), e2 = fn_eval(t->e[2], x, y);
  double sum = e0 + e1 + e2;
  double inv = 1.0 / sum;
  float b0 = (float)(e0 * inv), b1 = (float)(e1 * inv), b2 = (float)(e2 * inv);
  *depth_out = fn_eval(t->depth, x, y);
  int k0 = 0, k1 = t->tri == 0 ? 1 : 2, k2 = t->tri == 0 ? 2 : 3;
  float color[4] = {1.0f, 1.0f, 1.0f, 1.0f};
  if (q->has_c) {
    float a[4], b[4], cc[4];
    unpack_color(q->colors[k0], a);
    unpack_color(q->colors[k1], b);
    unpack_color(q->colors[k2], cc);
    for (int i = 0; i < 4; ++i) color[i] = a[i] * b0 + b[i] * b1 + cc[i] * b2;
  }
  float n[3];
  if (q->has_n) {
    for (int i = 0; i < 3; ++i) {
      float a = dec_normal_c((q->normals[k0] >> (10 * i)) & 0x3ffu);
      float b = dec_normal_c((q->normals[k1] >> (10 * i)) & 0x3ffu);
      float cc = dec_normal_c((q->normals[k2] >> (10 * i)) & 0x3ffu);
      n[i] = a * b0 + b * b1 + cc * b2;
    }
  } else {
    for (int i = 0; i < 3; ++i) n[i] = dec_normal_c((t->flat_normal >> (10 * i)) & 0x3ffu);
  }
  /* normalize (float), math.hpp:80-85 */
  float len2 = n[0] * n[0] + n[1] * n[1] + n[2] * n[2];
  if (len2 <= 0.0f) {
    n[0] = n[1] = n[2] = 0.0f;
  } else {
    float inv_len = 1.0f / sqrtf(len2);
    n[0] = n[0] * inv_len;
    n[1] = n[1] * inv_len;
    n[2] = n[2] * inv_len;
  }
  const veil_material* m = &c->sc->materials[t->material];
  float lam = fmaxf_std(0.0f, -(n[0] * c->light[0] + n[1] * c->light[1] + n[2] * c->light[2]));
  float light = fminf_std(1.0f, c->prm->ambient + lam);
  float r = m->base_color[0] * color[0] * 1.0f * light;
  float g = m->base_color[1] * color[1] * 1.0f * light;
  float b = m->base_color[2] * color[2] * 1.0f * light;
  float a = m->opacity * color[3] * 1.0f;
  out[0] = r * a;
  out[1] = g * a;
  out[2] = b * a;
  out[3] = a;
}

static uint64_t sample_key(const ctx_t* c, uint32_t q, uint32_t tri) {
  if (c->extended) return ((uint64_t)q << 32) | tri;
  return ((uint64_t)q << 24) | (tri & 0xffffffu); /* sample_sort_key, raster.hpp:95-97 */
}

/* The sample key in the reference's 24-bit-triangle format whatever the
 * mode: (q << 24) | tri24. In extended mode emit_hash_std hashes these, so a
 * limits-lifted reference build (whose keys are 24-bit) pins the blend order
 * of frames that need only the lifted viewport / bin limits. */
static uint64_t std_key(const ctx_t* c, uint64_t k) {
  if (!c->extended) return k;
  return ((k >> 32) << 24) | (k & 0xffffffu);
}

static void write_pixel(ctx_t* c, int px, int py, const float acc[4], int invalid,
                        uint64_t hash, uint64_t hash_std, uint32_t emitted) {
  float o[4] = {acc[0], acc[1], acc[2], acc[3]};
  /* blend_front_to_back(acc, background) */
  float t = 1.0f - o[3];
  float bgp[4] = {c->bg[0], c->bg[1], c->bg[2], c->bg[3]};
  for (int i = 0; i < 4; ++i) o[i] = o[i] + t * bgp[i];
  size_t pix = (size_t)py * c->cam.w + px;
  for (int i = 0; i < 4; ++i) c->image[pix * 4 + i] = quantize_channel(o[i]);
  c->mask[pix] = invalid ? 1 : 0;
  c->hash[pix] = hash;
  c->hash_std[pix] = hash_std;
  c->emit[pix] = emitted;
}

/* shade_half_block, raster.cpp:201-321 */
static void shade_half_block(ctx_t* c, bin_scratch* s, int bin, int hb, bin_stats* st,
                             dfilter* fl) {
  int bxi = bin % c->bx, byi = bin / c->bx;
  int block = hb / 2, half = hb % 2;
  int px0 = bxi * BIN + (block % 4) * 8;
  int py0 = byi * BIN + (block / 4) * 8 + half * 4;
  float acc[32][4];
  int invalid[32], saturated[32];
  uint64_t hh[32], hs[32];
  uint32_t cnt[32];
  memset(acc, 0, sizeof acc);
  memset(invalid, 0, sizeof invalid);
  memset(saturated, 0, sizeof saturated);
  memset(cnt, 0, sizeof cnt);
  for (int p = 0; p < 32; ++p) {
    hh[p] = hs[p] = kHashSeed;
    fl[p].n = 0;
    fl[p].any = 0;
    fl[p].max_key = 0;
  }
  int nsat = 0, stopped = 0;
  uint64_t enumerated = 0;
  for (uint32_t r = 0; r < s->nthb[hb] && !stopped; ++r) {
    const thb_t* rec = &s->thb[hb][r];
    for (int ly = 0; ly < 4 && !stopped; ++ly) {
      if (rec->b[ly] > rec->l[ly]) continue;
      for (uint32_t cx = rec->b[ly]; cx <= rec->l[ly]; ++cx) {
        int p = ly * 8 + (int)cx;
        ++enumerated;
        float col[4];
        double depth;
        shade(c, rec->tri, px0 + (int)cx, py0 + ly, col, &depth);
        uint64_t key = sample_key(c, quantize_depth(depth), rec->tri);
        df_insert(&fl[p], key, col);
        if (fl[p].n > c->df) {
          uint64_t k2;
          float c2[4];
          int ooo;
          df_pop(&fl[p], &k2, c2, &ooo);
          blend(acc[p], c2);
          hh[p] = (hh[p] ^ k2) * kHashPrime;
          hs[p] = (hs[p] ^ std_key(c, k2)) * kHashPrime;
          ++cnt[p];
          ++st->samples;
          if (ooo) invalid[p] = 1;
          if (c->threshold && !saturated[p] && acc[p][3] >= kAlphaThreshold) {
            saturated[p] = 1;
            if (++nsat == 32) {
              stopped = 1;
              break;
            }
          }
        }
      }
    }
  }
  if (!stopped) {
    for (int p = 0; p < 32; ++p) {
      int done = c->threshold && acc[p][3] >= kAlphaThreshold;
      while (fl[p].n > 0) {
        uint64_t k2;
        float c2[4];
        int ooo;
        df_pop(&fl[p], &k2, c2, &ooo);
        if (done) continue;
        blend(acc[p], c2);
        hh[p] = (hh[p] ^ k2) * kHashPrime;
        hs[p] = (hs[p] ^ std_key(c, k2)) * kHashPrime;
        ++cnt[p];
        ++st->samples;
        if (ooo) invalid[p] = 1;
        if (c->threshold && acc[p][3] >= kAlphaThreshold) done = 1;
      }
    }
  }
  st->segments += (enumerated + 255) / 256;
  for (int ly = 0; ly < 4; ++ly) {
    int py = py0 + ly;
    if (py >= c->cam.h) break;
    for (int lx = 0; lx < 8; ++lx) {
      int px = px0 + lx;
      if (px >= c->cam.w) break;
      int p = ly * 8 + lx;
      write_pixel(c, px, py, acc[p], invalid[p], hh[p], hs[p], cnt[p]);
    }
  }
}

/* rasterize_bin, raster.cpp:323-335 */
static int raster_bin(ctx_t* c, bin_scratch* s, int bin, const limits_t* lim, int hard,
                      bin_stats* st, dfilter* fl) {
  s->err[0] = 0;
  if (!gen_tbr(c, s, bin, lim, hard)) return 0;
  for (int k = 0; k < 16; ++k)
    if (!extract(c, s, bin, k, lim, hard)) return 0;
  memset(st, 0, sizeof *st);
  for (int h = 0; h < 32; ++h) {
    st->thb += s->nthb[h];
    st->fragments += s->nthb[h] ? s->thb[h][s->nthb[h] - 1].prefix : 0;
  }
  for (int h = 0; h < 32; ++h) shade_half_block(c, s, bin, h, st, fl);
  return 1;
}

static void free_scratch(bin_scratch* s) {
  for (int r = 0; r < 4; ++r) free(s->tbr[r]);
  for (int h = 0; h < 32; ++h) free(s->thb[h]);
  free(s->sr);
}

/* ------------------------------------------------------ a-buffer oracle */

typedef struct {
  uint64_t key;
  float col[4];
} frag_t;

static int cmp_frag(const void* a, const void* b) {
  uint64_t x = ((const frag_t*)a)->key, y = ((const frag_t*)b)->key;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* render_reference, oracle.cpp:28-117 (single-threaded) */
static void render_abuffer(ctx_t* c, uint64_t* total_samples) {
  int w = c->cam.w, h = c->cam.h;
  frag_t** lists = (frag_t**)xcalloc((size_t)w, sizeof(frag_t*));
  uint32_t* n = (uint32_t*)xcalloc((size_t)w, 4);
  uint32_t* cap = (uint32_t*)xcalloc((size_t)w, 4);
  *total_samples = 0;
  for (int py = 0; py < h; ++py) {
    memset(n, 0, (size_t)w * 4);
    for (uint64_t t = 0; t < (uint64_t)c->nvis * 2; ++t) {
      const tri_setup* ts = &c->ts[t];
      if (!ts->valid || py < ts->y_min || py > ts->y_max) continue;
      const vis_quad* q = &c->vq[t / 2];
      int x0 = (int)q->x0 * BIN;
      int x1 = imin((int)q->x1 * BIN + BIN - 1, w - 1);
      for (int px = x0; px <= x1; ++px) {
        if (!covers(ts, px, py)) continue;
        float col[4];
        double depth;
        shade(c, (uint32_t)t, px, py, col, &depth);
        if (n[px] == cap[px]) {
          cap[px] = cap[px] * 2 + 8;
          lists[px] = (frag_t*)xrealloc(lists[px], cap[px] * sizeof(frag_t));
        }
        lists[px][n[px]].key = sample_key(c, quantize_depth(depth), (uint32_t)t);
        memcpy(lists[px][n[px]].col, col, sizeof col);
        n[px]++;
      }
    }
    for (int px = 0; px < w; ++px) {
      qsort(lists[px], n[px], sizeof(frag_t), cmp_frag);
      float acc[4] = {0, 0, 0, 0};
      uint64_t hh = kHashSeed, hs = kHashSeed;
      for (uint32_t i = 0; i < n[px]; ++i) {
        blend(acc, lists[px][i].col);
        hh = (hh ^ lists[px][i].key) * kHashPrime;
        hs = (hs ^ std_key(c, lists[px][i].key)) * kHashPrime;
      }
      *total_samples += n[px];
      write_pixel(c, px, py, acc, 0, hh, hs, n[px]);
    }
  }
  for (int px = 0; px < w; ++px) free(lists[px]);
  free(lists);
  free(n);
  free(cap);
}

/* ---------------------------------------------------------------- entry */

static void export_setup(vo_frame* f, ctx_t* c) {
  uint32_t nv = c->nvis;
  uint32_t* src = (uint32_t*)xcalloc(nv, 4);
  uint64_t* aabb = (uint64_t*)xcalloc(nv, 8);
  uint8_t* cls = (uint8_t*)xcalloc(nv, 1);
  uint32_t* attr = (uint32_t*)xcalloc((size_t)nv * 9, 4);
  for (uint32_t i = 0; i < nv; ++i) {
    const vis_quad* q = &c->vq[i];
    src[i] = q->source;
    if (c->extended)
      aabb[i] = (uint64_t)q->x0 | ((uint64_t)q->y0 << 16) | ((uint64_t)q->x1 << 32) |
                ((uint64_t)q->y1 << 48);
    else /* pack_bin_aabb, packing.hpp:77-82 */
      aabb[i] = q->x0 | (q->y0 << 7) | (q->x1 << 14) | (q->y1 << 21) | ((q->cull & 3u) << 28);
    cls[i] = (uint8_t)(q->large | (q->has_c << 1) | (q->has_n << 2) | (q->has_uv << 3) |
                       ((q->cull & 3u) << 4));
    for (int k = 0; k < 4; ++k) attr[i * 9 + k] = q->colors[k];
    for (int k = 0; k < 4; ++k) attr[i * 9 + 4 + k] = q->normals[k];
    attr[i * 9 + 8] = q->material;
  }
  add_array(f, "quad_source", src, nv);
  add_array(f, "quad_aabb", aabb, nv);
  add_array(f, "quad_class", cls, nv);
  add_array(f, "quad_attr", attr, (uint64_t)nv * 9);
  uint64_t nt = (uint64_t)nv * 2;
  uint8_t* valid = (uint8_t*)xcalloc(nt, 1);
  int32_t* yr = (int32_t*)xcalloc(nt * 2, 4);
  double* fn = (double*)xcalloc(nt * 15, 8);
  uint32_t* meta = (uint32_t*)xcalloc(nt * 4, 4);
  for (uint64_t t = 0; t < nt; ++t) {
    const tri_setup* s = &c->ts[t];
    valid[t] = s->valid;
    yr[t * 2] = s->valid ? s->y_min : 0;
    yr[t * 2 + 1] = s->valid ? s->y_max : -1;
    const fn3* fs[5] = {&s->e[0], &s->e[1], &s->e[2], &s->inv_w, &s->depth};
    for (int k = 0; k < 5; ++k) {
      fn[t * 15 + k * 3] = fs[k]->a;
      fn[t * 15 + k * 3 + 1] = fs[k]->b;
      fn[t * 15 + k * 3 + 2] = fs[k]->c;
    }
    meta[t * 4] = s->flat_normal;
    meta[t * 4 + 1] = s->material;
    meta[t * 4 + 2] = s->quad_index;
    meta[t * 4 + 3] = s->tri;
  }
  add_array(f, "tri_valid", valid, nt);
  add_array(f, "tri_yrange", yr, nt * 2);
  add_array(f, "tri_fn", fn, nt * 15);
  add_array(f, "tri_meta", meta, nt * 4);
  uint64_t* st = (uint64_t*)xcalloc(6, 8);
  memcpy(st, c->stats, sizeof c->stats);
  add_array(f, "setup_stats", st, 6);
}

int vo_render(const veil_scene_desc* sc, const veil_render_params* prm, int extended,
              vo_frame** out) {
  vo_frame* f = (vo_frame*)xcalloc(1, sizeof(vo_frame));
  *out = f;
  veil_render_params defaults;
  if (!prm) {
    memset(&defaults, 0, sizeof defaults);
    defaults.depth_filter_size = 3;
    defaults.background[3] = 1.0f;
    defaults.light_dir[0] = 0.3f;
    defaults.light_dir[1] = -0.5f;
    defaults.light_dir[2] = 0.8f;
    defaults.ambient = 0.2f;
    prm = &defaults;
  }
  int st = validate(f, sc, extended);
  if (st != VEIL_OK) return st;
  int reference = (prm->flags & VEIL_RENDER_REFERENCE) != 0;
  if (!reference && prm->depth_filter_size < 1)
    return fail(f, VEIL_ERR_INVALID_ARG, "depth_filter_size must be >= 1");

  ctx_t c;
  memset(&c, 0, sizeof c);
  c.sc = sc;
  c.prm = prm;
  c.extended = extended;
  camera_init(&c.cam, sc);
  c.df = prm->depth_filter_size < 1 ? 1 : prm->depth_filter_size;
  c.threshold = (prm->flags & VEIL_RENDER_ALPHA_THRESHOLD) != 0;
  {
    /* normalize(light_dir), float */
    float l[3] = {prm->light_dir[0], prm->light_dir[1], prm->light_dir[2]};
    float len2 = l[0] * l[0] + l[1] * l[1] + l[2] * l[2];
    if (len2 <= 0.0f) {
      c.light[0] = c.light[1] = c.light[2] = 0.0f;
    } else {
      float inv = 1.0f / sqrtf(len2);
      for (int i = 0; i < 3; ++i) c.light[i] = l[i] * inv;
    }
    float a = prm->background[3];
    c.bg[0] = prm->background[0] * a;
    c.bg[1] = prm->background[1] * a;
    c.bg[2] = prm->background[2] * a;
    c.bg[3] = a;
  }
  size_t npx = (size_t)sc->width * sc->height;
  c.image = (uint8_t*)xcalloc(npx * 4, 1);
  c.mask = (uint8_t*)xcalloc(npx, 1);
  c.hash = (uint64_t*)xcalloc(npx, 8);
  c.hash_std = (uint64_t*)xcalloc(npx, 8);
  c.emit = (uint32_t*)xcalloc(npx, 4);
  for (size_t i = 0; i < npx; ++i) {
    c.hash[i] = c.hash_std[i] = kHashSeed;
    for (int k = 0; k < 4; ++k) c.image[i * 4 + k] = quantize_channel(c.bg[k]);
  }

  st = run_setup(f, &c);
  if (st != VEIL_OK) {
    free(c.image), free(c.mask), free(c.hash), free(c.hash_std), free(c.emit);
    return st;
  }
  export_setup(f, &c);

  uint64_t* counters = (uint64_t*)xcalloc(9, 8);
  if (reference) {
    uint64_t samples = 0;
    render_abuffer(&c, &samples);
    counters[0] = counters[1] = samples;
  } else {
    st = run_binning(f, &c);
    if (st != VEIL_OK) {
      free(counters);
      free(c.image), free(c.mask), free(c.hash), free(c.hash_std), free(c.emit);
      return st;
    }
    int nb = c.nbins;
    int32_t* dims = (int32_t*)xcalloc(2, 4);
    dims[0] = c.bx;
    dims[1] = c.by;
    add_array(f, "bin_dims", dims, 2);
    add_array(f, "bin_quad_counts", c.qcnt, (uint64_t)nb);
    add_array(f, "bin_tri_counts", c.tcnt, (uint64_t)nb);
    add_array(f, "bin_offsets", c.off, (uint64_t)nb);
    add_array(f, "bin_categories", c.cat, (uint64_t)nb);
    add_array(f, "bin_items", c.items, c.nitems);

    /* limits, renderer.cpp:130-142 */
    limits_t low = {1024, 256, 256, 4095}, high = {16384, 4096, 4096, 0xffffffffu};
    if (prm->limit_low_tbr) low.max_tbr = prm->limit_low_tbr;
    if (prm->limit_low_tri_blocks) low.max_tb = low.max_thb = prm->limit_low_tri_blocks;
    if (prm->limit_low_frags) low.max_frags = prm->limit_low_frags;
    if (prm->limit_high_tbr) high.max_tbr = prm->limit_high_tbr;
    if (prm->limit_high_thb) high.max_thb = prm->limit_high_thb;
    if (low.max_tbr > high.max_tbr || low.max_thb > high.max_thb) {
      free(counters);
      free(c.image), free(c.mask), free(c.hash), free(c.hash_std), free(c.emit);
      return fail(f, VEIL_ERR_INVALID_ARG, "low rasterizer limits exceed high limits");
    }

    bin_scratch s;
    memset(&s, 0, sizeof s);
    dfilter fl[32];
    for (int p = 0; p < 32; ++p) {
      fl[p].key = (uint64_t*)xcalloc((size_t)c.df + 1, 8);
      fl[p].col = (float(*)[4])xcalloc((size_t)c.df + 1, 16);
    }
    uint8_t* path = (uint8_t*)xcalloc((size_t)nb, 1);
    uint64_t* thb_off = (uint64_t*)xcalloc((size_t)nb * 32 + 1, 8);
    vec thb_bits = {0}, thb_tri = {0}, thb_pre = {0};
    bin_stats total;
    memset(&total, 0, sizeof total);
    int force_high = (prm->flags & VEIL_RENDER_FORCE_HIGH_PATH) != 0;
    /* low bins first, overflow -> high (renderer.cpp:144-165); bins are
     * independent so a per-bin sequence gives identical results. */
    for (int b = 0; b < nb && st == VEIL_OK; ++b) {
      bin_stats bs;
      if (c.cat[b] == 0) {
        for (int h = 0; h < 32; ++h) thb_off[(size_t)b * 32 + h + 1] = thb_bits.n / 8;
        continue;
      }
      int low_path = c.cat[b] == 1 && !force_high;
      if (low_path && raster_bin(&c, &s, b, &low, 0, &bs, fl)) {
        path[b] = 1;
      } else {
        path[b] = low_path ? 3 : 2;
        if (!raster_bin(&c, &s, b, &high, 1, &bs, fl)) {
          st = fail(f, VEIL_ERR_CAPACITY, "bin (%d,%d) exceeds high-rasterizer limit: %s",
                    b % c.bx, b / c.bx, s.err);
          break;
        }
      }
      total.samples += bs.samples;
      total.fragments += bs.fragments;
      total.thb += bs.thb;
      total.segments += bs.segments;
      for (int h = 0; h < 32; ++h) {
        for (uint32_t i = 0; i < s.nthb[h]; ++i) {
          const thb_t* t = &s.thb[h][i];
          uint64_t bits = 0; /* TriHalfBlock::make, packing.hpp:154-176 */
          for (int ly = 0; ly < 4; ++ly)
            bits |= ((uint64_t)(t->b[ly] & 7u) | ((uint64_t)(t->l[ly] & 7u) << 3)) << (6 * ly);
          bits |= (uint64_t)(t->tri & 0xffffffu) << 24;
          bits |= (uint64_t)(t->prefix & 0xfffu) << 48;
          vec_push(&thb_bits, &bits, 8);
          vec_push(&thb_tri, &t->tri, 4);
          vec_push(&thb_pre, &t->prefix, 4);
        }
        thb_off[(size_t)b * 32 + h + 1] = thb_bits.n / 8;
      }
    }
    free_scratch(&s);
    for (int p = 0; p < 32; ++p) free(fl[p].key), free(fl[p].col);
    add_array(f, "bin_path", path, (uint64_t)nb);
    add_array(f, "thb_offsets", thb_off, (uint64_t)nb * 32 + 1);
    add_array(f, "thb", thb_bits.p, thb_bits.n / 8);
    add_array(f, "thb_tri", thb_tri.p, thb_tri.n / 4);
    add_array(f, "thb_prefix", thb_pre.p, thb_pre.n / 4);
    if (st != VEIL_OK) {
      free(counters);
      free(c.image), free(c.mask), free(c.hash), free(c.hash_std), free(c.emit);
      return st;
    }
    uint64_t inv = 0;
    for (size_t i = 0; i < npx; ++i) inv += c.mask[i];
    if (prm->flags & VEIL_RENDER_VISUALIZE_ERRORS) /* apply_error_overlay, renderer.cpp:56-65 */
      for (size_t i = 0; i < npx; ++i)
        if (c.mask[i]) {
          c.image[i * 4] = 255;
          c.image[i * 4 + 1] = 0;
          c.image[i * 4 + 2] = 255;
          c.image[i * 4 + 3] = 255;
        }
    counters[0] = total.samples;
    counters[1] = total.fragments;
    counters[2] = total.thb;
    counters[3] = total.segments;
    for (int b = 0; b < nb; ++b) {
      counters[4 + c.cat[b]]++;
      if (path[b] == 3) counters[7]++;
    }
    counters[8] = inv;
  }
  add_array(f, "image", c.image, npx * 4);
  add_array(f, "mask", c.mask, npx);
  add_array(f, "emit_hash", c.hash, npx);
  add_array(f, "emit_hash_std", c.hash_std, npx);
  add_array(f, "emit_count", c.emit, npx);
  add_array(f, "counters", counters, 9);
  free(c.vq);
  free(c.ts);
  return VEIL_OK;
}

const void* vo_array(const vo_frame* f, const char* name, uint64_t* count) {
  if (count) *count = 0;
  if (!f || !name) return NULL;
  for (int i = 0; i < f->narrays; ++i)
    if (strcmp(f->arrays[i].name, name) == 0) {
      if (count) *count = f->arrays[i].count;
      return f->arrays[i].data;
    }
  return NULL;
}

const char* vo_message(const vo_frame* f) { return f ? f->message : ""; }

void vo_free(vo_frame* f) {
  if (!f) return;
  for (int i = 0; i < f->narrays; ++i) free(f->arrays[i].data);
  free(f);
}
