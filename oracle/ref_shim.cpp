// Test infrastructure only: a C shim compiled together with the UNMODIFIED
// reference sources (/root/reference/proj/src, see oracle/Makefile) into
// oracle/_ref/libveilref.so. It lets tests and bench.py's CPU-baseline arm
//   * build reference scenes from the same host arrays libveil consumes,
//   * export reference-loaded scenes (e.g. boxes.obj) as arrays,
//   * dump the reference pipeline's intermediate buffers through its public
//     phase hooks (run_setup, run_binning, BinRasterizer::generate_tri_block_rows
//     / extract_half_blocks, raster.hpp:107-119) for bit-exact comparison.
// Nothing on the product path loads this library.
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "veil.h"
#include "veil/binning.hpp"
#include "veil/depth_filter.hpp"
#include "veil/error.hpp"
#include "veil/raster.hpp"
#include "veil/renderer.hpp"
#include "veil/scanline.hpp"
#include "veil/setup.hpp"
#include "veil/shading.hpp"
#include "veil/synthetic.hpp"
#include "veil/thread_pool.hpp"
#include "../include/veil_cuda.h"

// Same definition as proj/src/c_api.cpp:30-32 (one definition rule).
struct veil_scene {
  veil::Scene scene;
};

namespace {

thread_local std::string g_shim_error;

std::map<const veil_scene*, std::vector<veil_material>> g_material_views;

template <typename Fn>
veil_status shim_guard(Fn&& fn) {
  try {
    fn();
    return VEIL_OK;
  } catch (const veil::Error& e) {
    g_shim_error = e.what();
    switch (e.code()) {
      case veil::ErrorCode::io: return VEIL_ERR_IO;
      case veil::ErrorCode::parse: return VEIL_ERR_PARSE;
      case veil::ErrorCode::invalid_argument: return VEIL_ERR_INVALID_ARG;
      case veil::ErrorCode::capacity: return VEIL_ERR_CAPACITY;
      case veil::ErrorCode::internal: return VEIL_ERR_INTERNAL;
    }
    return VEIL_ERR_INTERNAL;
  } catch (const std::exception& e) {
    g_shim_error = e.what();
    return VEIL_ERR_INTERNAL;
  }
}

veil::RenderConfig config_from(const veil_render_params* p) {
  veil::RenderConfig c;
  c.reference = p->flags & VEIL_RENDER_REFERENCE;
  c.alpha_threshold = p->flags & VEIL_RENDER_ALPHA_THRESHOLD;
  c.visualize_errors = p->flags & VEIL_RENDER_VISUALIZE_ERRORS;
  c.force_high_path = p->flags & VEIL_RENDER_FORCE_HIGH_PATH;
  c.backface_culling = p->flags & VEIL_RENDER_BACKFACE_CULLING;
  c.depth_filter_size = p->depth_filter_size;
  c.worker_count = p->thread_count;
  c.background = {p->background[0], p->background[1], p->background[2], p->background[3]};
  c.light_dir = {p->light_dir[0], p->light_dir[1], p->light_dir[2]};
  c.ambient = p->ambient;
  c.limit_low_tbr = p->limit_low_tbr;
  c.limit_low_tri_blocks = p->limit_low_tri_blocks;
  c.limit_low_frags = p->limit_low_frags;
  c.limit_high_tbr = p->limit_high_tbr;
  c.limit_high_thb = p->limit_high_thb;
  return c;
}

struct Array {
  std::vector<uint8_t> bytes;
  uint64_t count = 0;
};

template <typename T>
void put(std::map<std::string, Array>& m, const char* name, const std::vector<T>& v) {
  Array a;
  a.count = v.size();
  a.bytes.resize(v.size() * sizeof(T));
  if (!v.empty()) std::memcpy(a.bytes.data(), v.data(), a.bytes.size());
  m[name] = std::move(a);
}

constexpr uint64_t kHashSeed = 0xcbf29ce484222325ull;
constexpr uint64_t kHashPrime = 0x100000001b3ull;

}  // namespace

struct vref_dump {
  std::map<std::string, Array> arrays;
};

extern "C" {

const char* vref_last_error(void) { return g_shim_error.c_str(); }

veil_status vref_scene_create(const veil_scene_desc* d, veil_scene** out) {
  if (!d || !out) return VEIL_ERR_INVALID_ARG;
  return shim_guard([&] {
    auto s = std::make_unique<veil_scene>();
    veil::Scene& sc = s->scene;
    sc.vertices.resize(d->vertex_count);
    static_assert(sizeof(veil::Vertex) == sizeof(veil_vertex));
    static_assert(sizeof(veil::Quad) == sizeof(veil_quad));
    if (d->vertex_count) std::memcpy(sc.vertices.data(), d->vertices, d->vertex_count * 48);
    sc.quads.resize(d->quad_count);
    if (d->quad_count) std::memcpy(sc.quads.data(), d->quads, d->quad_count * 20);
    for (uint32_t i = 0; i < d->material_count; ++i) {
      const veil_material& m = d->materials[i];
      veil::Material mat;
      mat.base_color = {m.base_color[0], m.base_color[1], m.base_color[2], m.base_color[3]};
      mat.opacity = m.opacity;
      mat.texture = m.texture;
      mat.uses_vertex_colors = m.flags & VEIL_MATERIAL_VERTEX_COLORS;
      mat.uses_vertex_normals = m.flags & VEIL_MATERIAL_VERTEX_NORMALS;
      mat.uses_uvs = m.flags & VEIL_MATERIAL_UVS;
      mat.name = "m" + std::to_string(i);
      sc.materials.push_back(mat);
    }
    sc.has_vertex_normals = d->flags & VEIL_SCENE_HAS_NORMALS;
    sc.has_vertex_colors = d->flags & VEIL_SCENE_HAS_COLORS;
    sc.has_uvs = d->flags & VEIL_SCENE_HAS_UVS;
    for (int i = 0; i < 16; ++i) sc.camera.view_projection.m[i / 4][i % 4] = d->view_projection[i];
    sc.camera.width = d->width;
    sc.camera.height = d->height;
    if (d->has_eye) sc.camera.eye = veil::Vec3d{d->eye[0], d->eye[1], d->eye[2]};
    *out = s.release();
  });
}

veil_status vref_scene_describe(const veil_scene* s, veil_scene_desc* d) {
  if (!s || !d) return VEIL_ERR_INVALID_ARG;
  const veil::Scene& sc = s->scene;
  std::vector<veil_material>& mats = g_material_views[s];
  mats.clear();
  for (const veil::Material& m : sc.materials) {
    veil_material v{};
    v.base_color[0] = m.base_color.x;
    v.base_color[1] = m.base_color.y;
    v.base_color[2] = m.base_color.z;
    v.base_color[3] = m.base_color.w;
    v.opacity = m.opacity;
    v.texture = m.texture;
    v.flags = (m.uses_vertex_colors ? VEIL_MATERIAL_VERTEX_COLORS : 0) |
              (m.uses_vertex_normals ? VEIL_MATERIAL_VERTEX_NORMALS : 0) |
              (m.uses_uvs ? VEIL_MATERIAL_UVS : 0);
    mats.push_back(v);
  }
  std::memset(d, 0, sizeof(*d));
  d->vertices = reinterpret_cast<const veil_vertex*>(sc.vertices.data());
  d->vertex_count = sc.vertices.size();
  d->quads = reinterpret_cast<const veil_quad*>(sc.quads.data());
  d->quad_count = sc.quads.size();
  d->materials = mats.data();
  d->material_count = uint32_t(mats.size());
  d->flags = (sc.has_vertex_normals ? VEIL_SCENE_HAS_NORMALS : 0) |
             (sc.has_vertex_colors ? VEIL_SCENE_HAS_COLORS : 0) |
             (sc.has_uvs ? VEIL_SCENE_HAS_UVS : 0);
  for (int i = 0; i < 16; ++i) d->view_projection[i] = sc.camera.view_projection.m[i / 4][i % 4];
  d->width = sc.camera.width;
  d->height = sc.camera.height;
  if (sc.camera.eye) {
    d->has_eye = 1;
    d->eye[0] = sc.camera.eye->x;
    d->eye[1] = sc.camera.eye->y;
    d->eye[2] = sc.camera.eye->z;
  }
  return VEIL_OK;
}

veil_status vref_dump_run(const veil_scene* s, const veil_render_params* params,
                          vref_dump** out) {
  if (!s || !params || !out) return VEIL_ERR_INVALID_ARG;
  return shim_guard([&] {
    using namespace veil;
    const Scene& scene = s->scene;
    RenderConfig config = config_from(params);
    config.worker_count = 1;
    auto dump = std::make_unique<vref_dump>();
    auto& A = dump->arrays;
    ThreadPool pool(1);

    SetupOutput setup = run_setup(scene, config, pool);
    {
      std::vector<uint32_t> src, attr;
      std::vector<uint64_t> aabb;
      std::vector<uint8_t> cls;
      for (const VisibleQuadRecord& q : setup.quads) {
        src.push_back(q.source_quad);
        aabb.push_back(q.packed_bin_aabb);
        cls.push_back(uint8_t((q.size_class == SizeClass::large ? 1 : 0) |
                              (q.has_colors ? 2 : 0) | (q.has_normals ? 4 : 0) |
                              (q.has_uvs ? 8 : 0) | ((q.packed_bin_aabb >> 28) << 4)));
        for (int i = 0; i < 4; ++i) attr.push_back(q.vertex_colors[i]);
        for (int i = 0; i < 4; ++i) attr.push_back(q.vertex_normals[i]);
        attr.push_back(q.material_id);
      }
      put(A, "quad_source", src);
      put(A, "quad_aabb", aabb);
      put(A, "quad_class", cls);
      put(A, "quad_attr", attr);
      std::vector<uint8_t> valid;
      std::vector<int32_t> yr;
      std::vector<double> fn;
      std::vector<uint32_t> meta;
      for (const TriangleSetup& t : setup.triangles) {
        valid.push_back(t.valid ? 1 : 0);
        yr.push_back(t.y_min);
        yr.push_back(t.y_max);
        const AffineFn* f[5] = {&t.edges[0], &t.edges[1], &t.edges[2], &t.inv_w, &t.depth};
        for (auto* g : f) {
          fn.push_back(g->a);
          fn.push_back(g->b);
          fn.push_back(g->c);
        }
        meta.push_back(t.flat_normal);
        meta.push_back(t.material_id);
        meta.push_back(t.quad_index);
        meta.push_back(t.tri);
      }
      put(A, "tri_valid", valid);
      put(A, "tri_yrange", yr);
      put(A, "tri_fn", fn);
      put(A, "tri_meta", meta);
      std::vector<uint64_t> st = {setup.stats.input_quads,       setup.stats.visible_quads,
                                  setup.stats.culled_degenerate, setup.stats.culled_backfacing,
                                  setup.stats.culled_frustum,    setup.stats.culled_between_samples};
      put(A, "setup_stats", st);
    }

    const Camera& cam = scene.camera;
    BinGrid grid = run_binning(setup, cam.width, cam.height, pool);
    {
      put(A, "bin_dims", std::vector<int32_t>{grid.bins_x, grid.bins_y});
      put(A, "bin_quad_counts", grid.quad_counts);
      put(A, "bin_tri_counts", grid.tri_counts);
      put(A, "bin_offsets", grid.offsets);
      std::vector<uint8_t> cat;
      for (BinCategory c : grid.categories) cat.push_back(uint8_t(c));
      put(A, "bin_categories", cat);
      put(A, "bin_items", grid.items);
    }

    // Phase hooks per bin, in the order render_pipeline applies them
    // (renderer.cpp:117-165): low limits with soft overflow, then high.
    RasterContext ctx;
    Image8 image(cam.width, cam.height);
    std::vector<uint8_t> mask(size_t(cam.width) * cam.height, 0);
    ctx.setup = &setup;
    ctx.grid = &grid;
    ctx.scene = &scene;
    ctx.config = &config;
    ctx.shade.light_dir = normalize(config.light_dir);
    ctx.shade.ambient = config.ambient;
    ctx.shade.textures = scene.textures;
    ctx.frame.color = &image;
    ctx.frame.invalid_mask = &mask;
    Vec4f bg = config.background;
    ctx.frame.background_premultiplied = {bg.x * bg.w, bg.y * bg.w, bg.z * bg.w, bg.w};
    for (size_t i = 0; i < image.rgba.size(); i += 4) {  // fill_background, renderer.cpp:41-54
      image.rgba[i] = quantize_channel(ctx.frame.background_premultiplied.x);
      image.rgba[i + 1] = quantize_channel(ctx.frame.background_premultiplied.y);
      image.rgba[i + 2] = quantize_channel(ctx.frame.background_premultiplied.z);
      image.rgba[i + 3] = quantize_channel(ctx.frame.background_premultiplied.w);
    }

    RasterLimits low = RasterLimits::low(), high = RasterLimits::high();
    if (config.limit_low_tbr) low.max_tbr_per_block_row = config.limit_low_tbr;
    if (config.limit_low_tri_blocks) {
      low.max_tri_blocks_per_block = config.limit_low_tri_blocks;
      low.max_thb_per_half_block = config.limit_low_tri_blocks;
    }
    if (config.limit_low_frags) low.max_frags_per_half_block = config.limit_low_frags;
    if (config.limit_high_tbr) high.max_tbr_per_block_row = config.limit_high_tbr;
    if (config.limit_high_thb) high.max_thb_per_half_block = config.limit_high_thb;

    BinRasterizer worker(ctx);
    const int nb = grid.bin_count();
    std::vector<uint8_t> path(nb, 0);
    std::vector<uint64_t> thb_off(size_t(nb) * 32 + 1, 0), tbr_off(size_t(nb) * 4 + 1, 0);
    std::vector<uint64_t> thb_bits, tbr_bits;
    std::vector<uint32_t> thb_prefix;
    std::vector<uint64_t> hash(size_t(cam.width) * cam.height, kHashSeed);
    std::vector<uint32_t> emit(size_t(cam.width) * cam.height, 0);

    auto run_phases = [&](int b, const RasterLimits& lim, bool hard) {
      if (!worker.generate_tri_block_rows(b, lim, hard)) return false;
      for (int k = 0; k < 16; ++k)
        if (!worker.extract_half_blocks(b, k, lim, hard)) return false;
      return true;
    };

    for (int b = 0; b < nb; ++b) {
      BinCategory c = grid.categories[b];
      if (c == BinCategory::empty) {
        for (int r = 0; r < 4; ++r) tbr_off[size_t(b) * 4 + r + 1] = tbr_bits.size() / 2;
        for (int h = 0; h < 32; ++h) thb_off[size_t(b) * 32 + h + 1] = thb_bits.size();
        continue;
      }
      bool low_path = c == BinCategory::low && !config.force_high_path;
      if (low_path && run_phases(b, low, false)) {
        path[b] = 1;
      } else {
        path[b] = low_path ? 3 : 2;
        run_phases(b, high, true);  // throws the capacity error like the pipeline
      }
      for (int r = 0; r < 4; ++r) {
        for (const TriBlockRow& t : worker.tbr[r]) {
          tbr_bits.push_back(t.lo);
          tbr_bits.push_back(t.hi);
        }
        tbr_off[size_t(b) * 4 + r + 1] = tbr_bits.size() / 2;
      }
      for (int h = 0; h < 32; ++h) {
        for (size_t i = 0; i < worker.thb[h].size(); ++i) {
          thb_bits.push_back(worker.thb[h][i].bits);
          thb_prefix.push_back(worker.thb_prefix[h][i]);
        }
        thb_off[size_t(b) * 32 + h + 1] = thb_bits.size();
      }

      // Per-pixel blend order, re-enumerated from the tri-half-blocks with
      // the reference's public shading and DepthFilter (the loop of
      // raster.cpp:232-284). The image it produces is compared with
      // render_pipeline's below, which pins this re-enumeration.
      const int bx = b % grid.bins_x, by = b / grid.bins_x;
      for (int h = 0; h < 32; ++h) {
        const int block = h / 2, half = h % 2;
        const int px0 = bx * kBinSize + (block % 4) * 8;
        const int py0 = by * kBinSize + (block / 4) * 8 + half * 4;
        std::vector<DepthFilter> filters(32, DepthFilter(std::max(1, config.depth_filter_size)));
        Vec4f acc[32] = {};
        bool invalid[32] = {}, saturated[32] = {};
        uint64_t hh[32];
        uint32_t cnt[32] = {};
        for (auto& v : hh) v = kHashSeed;
        int nsat = 0;
        bool stopped = false;
        for (size_t r = 0; r < worker.thb[h].size() && !stopped; ++r) {
          const TriHalfBlock rec = worker.thb[h][r];
          uint32_t ti = rec.triangle_index();
          const TriangleSetup& tri = setup.triangles[ti];
          const VisibleQuadRecord& quad = setup.quads[ti / 2];
          const Material& mat = scene.materials[tri.material_id];
          for (int ly = 0; ly < 4 && !stopped; ++ly) {
            RowSpan sp = rec.row(ly);
            if (sp.empty()) continue;
            for (uint32_t cx = sp.begin; cx <= sp.last; ++cx) {
              int p = ly * 8 + int(cx);
              SampleContext sc = make_sample_context(tri, quad, px0 + int(cx), py0 + ly);
              Vec4f col = shade_sample(sc, mat, ctx.shade);
              uint64_t key = sample_sort_key(quantize_depth(sc.depth), ti);
              bool ooo = false;
              if (auto e = filters[p].push(key, col, &ooo)) {
                acc[p] = blend_front_to_back(acc[p], e->color);
                hh[p] = (hh[p] ^ e->key) * kHashPrime;
                ++cnt[p];
                if (ooo) invalid[p] = true;
                if (config.alpha_threshold && !saturated[p] &&
                    acc[p].w >= kAlphaThresholdValue) {
                  saturated[p] = true;
                  if (++nsat == 32) {
                    stopped = true;
                    break;
                  }
                }
              }
            }
          }
        }
        if (!stopped) {
          for (int p = 0; p < 32; ++p) {
            bool done = config.alpha_threshold && acc[p].w >= kAlphaThresholdValue;
            filters[p].flush([&](const DepthFilter::Entry& e, bool ooo) {
              if (done) return;
              acc[p] = blend_front_to_back(acc[p], e.color);
              hh[p] = (hh[p] ^ e.key) * kHashPrime;
              ++cnt[p];
              if (ooo) invalid[p] = true;
              if (config.alpha_threshold && acc[p].w >= kAlphaThresholdValue) done = true;
            });
          }
        }
        for (int ly = 0; ly < 4; ++ly) {
          int py = py0 + ly;
          if (py >= cam.height) break;
          for (int lx = 0; lx < 8; ++lx) {
            int px = px0 + lx;
            if (px >= cam.width) break;
            int p = ly * 8 + lx;
            size_t pix = size_t(py) * cam.width + px;
            hash[pix] = hh[p];
            emit[pix] = cnt[p];
            Vec4f o = blend_front_to_back(acc[p], ctx.frame.background_premultiplied);
            uint8_t* dst = image.pixel(px, py);
            dst[0] = quantize_channel(o.x);
            dst[1] = quantize_channel(o.y);
            dst[2] = quantize_channel(o.z);
            dst[3] = quantize_channel(o.w);
            mask[pix] = invalid[p] ? 1 : 0;
          }
        }
      }
    }
    put(A, "bin_path", path);
    put(A, "tbr_offsets", tbr_off);
    put(A, "tbr", tbr_bits);
    put(A, "thb_offsets", thb_off);
    put(A, "thb", thb_bits);
    put(A, "thb_prefix", thb_prefix);
    put(A, "emit_hash", hash);
    put(A, "emit_count", emit);
    if (config.visualize_errors)  // apply_error_overlay, renderer.cpp:56-65
      for (size_t p = 0; p < mask.size(); ++p)
        if (mask[p]) {
          image.rgba[p * 4] = 255;
          image.rgba[p * 4 + 1] = 0;
          image.rgba[p * 4 + 2] = 255;
          image.rgba[p * 4 + 3] = 255;
        }
    put(A, "reenum_image", image.rgba);
    put(A, "reenum_mask", mask);

    // The reference's own full render (renderer.cpp:69-213).
    RenderResult full = render_pipeline(scene, config);
    put(A, "image", full.image.rgba);
    put(A, "mask", full.invalid_mask);
    const RunReport& r = full.report;
    put(A, "counters",
        std::vector<uint64_t>{r.samples, r.fragments, r.tri_half_blocks, r.segments,
                              r.bins_empty, r.bins_low, r.bins_high, r.bins_propagated,
                              r.invalid_pixels});
    *out = dump.release();
  });
}

const void* vref_dump_array(const vref_dump* d, const char* name, uint64_t* count) {
  if (count) *count = 0;
  if (!d || !name) return nullptr;
  auto it = d->arrays.find(name);
  if (it == d->arrays.end()) return nullptr;
  if (count) *count = it->second.count;
  return it->second.bytes.data();
}

void vref_dump_destroy(vref_dump* d) { delete d; }

void vref_scene_forget(const veil_scene* s) { g_material_views.erase(s); }

// generate_synthetic_scene with explicit SyntheticParams (synthetic.hpp:36-47;
// the C API's veil_scene_synthetic uses the defaults) -- the scenes of the
// reference's acceptance criterion 1 (acceptance.cpp:80-101).
veil_status vref_scene_synthetic_params(const char* kind, uint64_t seed, int width, int height,
                                        int layers, int triangles, int sheets, veil_scene** out) {
  if (!kind || !out) return VEIL_ERR_INVALID_ARG;
  return shim_guard([&] {
    auto k = veil::parse_synthetic_kind(kind);
    if (!k) throw veil::Error(veil::ErrorCode::invalid_argument, "unknown synthetic kind");
    veil::SyntheticParams sp;
    sp.width = width;
    sp.height = height;
    if (layers > 0) sp.layers = layers;
    if (triangles > 0) sp.triangles = triangles;
    if (sheets > 0) sp.sheets = sheets;
    auto s = std::make_unique<veil_scene>();
    s->scene = veil::generate_synthetic_scene(*k, seed, sp);
    *out = s.release();
  });
}

// The reference pipeline's max per-pixel sort disorder (RenderConfig::
// measure_disorder, scene.hpp:108; raster.cpp:286-297), which the C API
// cannot reach; acceptance criterion 1 renders with DF = this value.
veil_status vref_measure_disorder(const veil_scene* s, const veil_render_params* p, int* out) {
  if (!s || !p || !out) return VEIL_ERR_INVALID_ARG;
  return shim_guard([&] {
    veil::RenderConfig c = config_from(p);
    c.measure_disorder = true;
    *out = veil::render_pipeline(s->scene, c).report.max_disorder;
  });
}

// The reference's own make_look_at_camera (scene.cpp:128-158), so bench.py's
// reference arm builds its orbit cameras without libveil.
veil_status vref_look_at(const double from[3], const double at[3], const double up[3], double fov_deg,
                         double near_z, double far_z, int width, int height, double out[16]) {
  if (!from || !at || !up || !out) return VEIL_ERR_INVALID_ARG;
  return shim_guard([&] {
    const veil::Camera c = veil::make_look_at_camera({from[0], from[1], from[2]}, {at[0], at[1], at[2]},
                                                     {up[0], up[1], up[2]}, fov_deg, near_z, far_z,
                                                     width, height);
    for (int i = 0; i < 16; ++i) out[i] = c.view_projection.m[i / 4][i % 4];
  });
}

}  // extern "C"
