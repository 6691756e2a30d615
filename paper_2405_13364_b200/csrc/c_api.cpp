// extern "C" boundary of libveil.so: the 18 entry points of the reference's
// veil.h (proj/src/c_api.cpp:85-249) plus the additive veil_cuda.h calls.
// No exception crosses the ABI; failures set a thread-local message
// (reference c_api.cpp:41-74).
#include <cstring>
#include <memory>
#include <string>

#include "veil_internal.hpp"

namespace {

thread_local std::string t_error;

template <typename Fn>
veil_status guard(Fn&& fn) {
  try {
    fn();
    return VEIL_OK;
  } catch (const veil::Error& e) {
    t_error = e.what();
    return e.status();
  } catch (const std::exception& e) {
    t_error = e.what();
    return VEIL_ERR_INTERNAL;
  } catch (...) {
    t_error = "unknown error";
    return VEIL_ERR_INTERNAL;
  }
}

veil_status bad_arg(const char* msg) {
  t_error = msg;
  return VEIL_ERR_INVALID_ARG;
}

veil::RenderOptions options_from(const veil_render_params* params) {
  veil::RenderOptions o;
  veil_render_params_init(&o.params);
  if (params) o.params = *params;
  return o;
}

void finish_render(const veil_scene* scene, const veil::RenderOptions& opt, veil_render* r) {
  const veil::Scene& s = scene->s;
  r->json = veil::report_json(r->out, opt.params, r->out.width, r->out.height,
                              s.degenerate_quad_percent());
}

veil_status do_render(const veil_scene* scene, veil::RenderOptions opt, veil_render** out) {
  return guard([&] {
    auto r = std::make_unique<veil_render>();
    if (opt.params.flags & VEIL_RENDER_REFERENCE)
      veil::render_reference_frame(scene->s, opt, &r->out);
    else
      veil::render_frame(scene->s, opt, &r->out);
    finish_render(scene, opt, r.get());
    *out = r.release();
  });
}

}  // namespace

extern "C" {

const char* veil_status_string(veil_status status) {
  switch (status) {
    case VEIL_OK: return "ok";
    case VEIL_ERR_IO: return "I/O error";
    case VEIL_ERR_PARSE: return "parse error";
    case VEIL_ERR_INVALID_ARG: return "invalid argument";
    case VEIL_ERR_CAPACITY: return "capacity exceeded";
    case VEIL_ERR_INTERNAL: return "internal error";
  }
  return "unknown status";
}

const char* veil_last_error(void) { return t_error.c_str(); }

veil_status veil_scene_load(const char* mesh_path, const char* material_path,
                            const char* camera_path, veil_scene** out_scene) {
  if (!mesh_path || !out_scene) return bad_arg("mesh_path and out_scene are required");
  return guard([&] {
    auto s = std::make_unique<veil_scene>();
    veil::load_obj_scene(&s->s, mesh_path, material_path ? material_path : "",
                         camera_path ? camera_path : "");
    *out_scene = s.release();
  });
}

veil_status veil_scene_synthetic(const char* kind, uint64_t seed, int width, int height,
                                 veil_scene** out_scene) {
  if (!kind || !out_scene) return bad_arg("kind and out_scene are required");
  std::string k = kind;
  if (k != "layered_quads" && k != "intersecting_shells" && k != "random_soup" &&
      k != "dense_bin")
    return bad_arg("unknown synthetic scene kind");
  return guard([&] {
    auto s = std::make_unique<veil_scene>();
    veil::synthetic_scene(&s->s, k, seed, width, height);
    *out_scene = s.release();
  });
}

veil_status veil_scene_group_quads(veil_scene* scene, double* out_degenerate_percent) {
  if (!scene) return bad_arg("scene is required");
  return guard([&] {
    double pct = veil::group_quads(&scene->s);
    if (out_degenerate_percent) *out_degenerate_percent = pct;
  });
}

veil_status veil_scene_set_viewport(veil_scene* scene, int width, int height) {
  if (!scene) return bad_arg("scene is required");
  return guard([&] {
    veil::Camera c = scene->s.camera;
    c.width = width;
    c.height = height;
    veil::validate_camera(c, scene->s.extended);
    scene->s.camera = c;
  });
}

veil_status veil_scene_set_camera(veil_scene* scene, const double matrix[16],
                                  const double eye[3]) {
  if (!scene || !matrix) return bad_arg("scene and matrix are required");
  return guard([&] {
    veil::Camera& c = scene->s.camera;
    for (int i = 0; i < 16; ++i) c.m[i] = matrix[i];
    c.has_eye = eye != nullptr;
    for (int i = 0; i < 3; ++i) c.eye[i] = eye ? eye[i] : 0.0;
  });
}

void veil_scene_destroy(veil_scene* scene) { delete scene; }

void veil_render_params_init(veil_render_params* params) {
  if (!params) return;
  std::memset(params, 0, sizeof(*params));
  params->depth_filter_size = 3;
  params->background[3] = 1.0f;
  params->light_dir[0] = 0.3f;
  params->light_dir[1] = -0.5f;
  params->light_dir[2] = 0.8f;
  params->ambient = 0.2f;
}

veil_status veil_render_scene(const veil_scene* scene, const veil_render_params* params,
                              veil_render** out_render) {
  if (!scene || !out_render) return bad_arg("scene and out_render are required");
  return do_render(scene, options_from(params), out_render);
}

int veil_render_width(const veil_render* r) { return r ? r->out.width : 0; }
int veil_render_height(const veil_render* r) { return r ? r->out.height : 0; }
const uint8_t* veil_render_pixels(const veil_render* r) {
  return r ? r->out.rgba() : nullptr;
}
const uint8_t* veil_render_invalid_mask(const veil_render* r) {
  return r ? r->out.mask() : nullptr;
}
const char* veil_render_report_json(const veil_render* r) { return r ? r->json.c_str() : ""; }

veil_status veil_render_write_png(const veil_render* r, const char* path) {
  if (!r || !path) return bad_arg("render and path are required");
  return guard([&] {
    veil::Image8 img;
    img.width = r->out.width;
    img.height = r->out.height;
    img.rgba.assign(r->out.rgba(), r->out.rgba() + size_t(img.width) * img.height * 4);
    veil::write_png(img, path);
  });
}

void veil_render_destroy(veil_render* r) { delete r; }

veil_status veil_compare_png(const char* a, const char* b, veil_image_diff* out) {
  if (!a || !b || !out) return bad_arg("path_a, path_b and out_diff are required");
  return guard([&] {
    veil::Image8 x = veil::read_png(a), y = veil::read_png(b);
    if (x.width != y.width || x.height != y.height)
      throw veil::Error(VEIL_ERR_INVALID_ARG, "image dimensions differ");
    uint64_t diff = 0;
    int maxd = 0;
    for (size_t p = 0; p < size_t(x.width) * x.height; ++p) {
      int d = 0;
      for (int c = 0; c < 4; ++c) d = std::max(d, std::abs(int(x.rgba[p * 4 + c]) - int(y.rgba[p * 4 + c])));
      if (d > 0) ++diff, maxd = std::max(maxd, d);
    }
    out->differing_pixels = diff;
    out->max_channel_delta = maxd;
    out->width = x.width;
    out->height = x.height;
  });
}

// ------------------------------------------------------------- veil_cuda.h

veil_status veil_scene_create(const veil_scene_desc* d, veil_scene** out) {
  if (!d || !out) return bad_arg("desc and out_scene are required");
  if ((d->vertex_count && !d->vertices) || (d->quad_count && !d->quads) ||
      (d->material_count && !d->materials))
    return bad_arg("scene arrays are required");
  return guard([&] {
    auto s = std::make_unique<veil_scene>();
    veil::Scene& sc = s->s;
    sc.vertices.assign(d->vertices, d->vertices + d->vertex_count);
    sc.quads.assign(d->quads, d->quads + d->quad_count);
    sc.materials.assign(d->materials, d->materials + d->material_count);
    for (uint32_t i = 0; i < d->material_count; ++i) {
      sc.material_names.push_back("m" + std::to_string(i));
      if (sc.materials[i].texture >= 0)
        throw veil::Error(VEIL_ERR_INVALID_ARG, "array scenes carry no textures");
    }
    sc.flags = d->flags;
    for (int i = 0; i < 16; ++i) sc.camera.m[i] = d->view_projection[i];
    sc.camera.width = d->width;
    sc.camera.height = d->height;
    sc.camera.has_eye = d->has_eye != 0;
    for (int i = 0; i < 3; ++i) sc.camera.eye[i] = d->eye[i];
    sc.extended = d->width > veil::kMaxViewportWidth || d->height > veil::kMaxViewportHeight;
    veil::validate_scene(sc);
    *out = s.release();
  });
}

veil_status veil_scene_describe(const veil_scene* scene, veil_scene_desc* d) {
  if (!scene || !d) return bad_arg("scene and out_desc are required");
  const veil::Scene& s = scene->s;
  std::memset(d, 0, sizeof(*d));
  d->vertices = s.vertices.data();
  d->vertex_count = s.vertices.size();
  d->quads = s.quads.data();
  d->quad_count = s.quads.size();
  d->materials = s.materials.data();
  d->material_count = uint32_t(s.materials.size());
  d->flags = s.flags;
  for (int i = 0; i < 16; ++i) d->view_projection[i] = s.camera.m[i];
  d->width = s.camera.width;
  d->height = s.camera.height;
  d->has_eye = s.camera.has_eye;
  for (int i = 0; i < 3; ++i) d->eye[i] = s.camera.eye[i];
  return VEIL_OK;
}

veil_status veil_scene_workload(const char* name, uint64_t seed, int width, int height,
                                veil_scene** out) {
  if (!name || !out) return bad_arg("name and out_scene are required");
  return guard([&] {
    auto s = std::make_unique<veil_scene>();
    veil::workload_scene(&s->s, name, seed, width, height);
    *out = s.release();
  });
}

veil_status veil_camera_look_at(const double from[3], const double at[3], const double up[3],
                                double fov_deg, double near_z, double far_z, int width,
                                int height, double out_matrix[16]) {
  if (!from || !at || !up || !out_matrix) return bad_arg("vectors and out_matrix are required");
  return guard([&] {
    veil::Camera c = veil::look_at_camera(from, at, up, fov_deg, near_z, far_z, width, height);
    for (int i = 0; i < 16; ++i) out_matrix[i] = c.m[i];
  });
}

veil_status veil_scene_set_extended_limits(veil_scene* scene, int enable) {
  if (!scene) return bad_arg("scene is required");
  return guard([&] {
    if (!enable) veil::validate_camera(scene->s.camera, false);
    scene->s.extended = enable != 0;
  });
}

veil_status veil_scene_set_viewport_ext(veil_scene* scene, int width, int height) {
  if (!scene) return bad_arg("scene is required");
  return guard([&] {
    veil::Camera c = scene->s.camera;
    c.width = width;
    c.height = height;
    veil::validate_camera(c, true);
    scene->s.extended = true;
    scene->s.camera = c;
  });
}

veil_status veil_cuda_set_device(int device) {
  return guard([&] { veil::set_current_device(device); });
}

veil_status veil_render_scene_shard(const veil_scene* scene, const veil_render_params* params,
                                    const veil_shard* shard, veil_render** out) {
  if (!scene || !out) return bad_arg("scene and out_render are required");
  veil::RenderOptions o = options_from(params);
  if (shard) {
    if (shard->world_size < 1 || shard->rank < 0 || shard->rank >= shard->world_size)
      return bad_arg("invalid shard");
    o.rank = shard->rank;
    o.world_size = shard->world_size;
  }
  if (o.params.flags & VEIL_RENDER_REFERENCE && o.world_size > 1)
    return bad_arg("the a-buffer renderer does not shard");
  return do_render(scene, o, out);
}

uint64_t veil_shard_tile_count(int bins_x, int bins_y, const veil_shard* shard) {
  if (!shard) return uint64_t(bins_x) * bins_y;
  return veil::shard_tile_count(bins_x, bins_y, shard->rank, shard->world_size);
}

veil_status veil_shard_pack_tiles(const veil_render* r, const veil_shard* shard, uint8_t* out,
                                  uint64_t out_bytes) {
  if (!r || !shard || !out) return bad_arg("render, shard and out are required");
  return guard([&] {
    const int W = r->out.width, H = r->out.height, K = veil::kBinSize;
    int bx = (W + K - 1) / K, by = (H + K - 1) / K;
    uint64_t n = veil::shard_tile_count(bx, by, shard->rank, shard->world_size);
    if (out_bytes < n * 5120) throw veil::Error(VEIL_ERR_INVALID_ARG, "tile buffer too small");
    uint64_t t = 0;
    for (int y = 0; y < by; ++y)
      for (int x = 0; x < bx; ++x) {
        if (!veil::bin_owned(x, y, shard->rank, shard->world_size)) continue;
        uint8_t* dst = out + t * 5120;
        std::memset(dst, 0, 5120);
        for (int ly = 0; ly < K; ++ly) {
          int py = y * K + ly;
          if (py >= H) break;
          int w = std::min(K, W - x * K);
          std::memcpy(dst + ly * K * 4, r->out.rgba() + (size_t(py) * W + x * K) * 4, w * 4);
          std::memcpy(dst + 4096 + ly * K, r->out.mask() + size_t(py) * W + x * K, w);
        }
        ++t;
      }
  });
}

veil_status veil_shard_unpack_tiles(veil_render* r, const veil_shard* shard, const uint8_t* tiles,
                                    uint64_t bytes) {
  if (!r || !shard || !tiles) return bad_arg("render, shard and tiles are required");
  return guard([&] {
    const int W = r->out.width, H = r->out.height, K = veil::kBinSize;
    int bx = (W + K - 1) / K, by = (H + K - 1) / K;
    uint64_t n = veil::shard_tile_count(bx, by, shard->rank, shard->world_size);
    if (bytes < n * 5120) throw veil::Error(VEIL_ERR_INVALID_ARG, "tile buffer too small");
    uint64_t t = 0;
    for (int y = 0; y < by; ++y)
      for (int x = 0; x < bx; ++x) {
        if (!veil::bin_owned(x, y, shard->rank, shard->world_size)) continue;
        const uint8_t* src = tiles + t * 5120;
        for (int ly = 0; ly < K; ++ly) {
          int py = y * K + ly;
          if (py >= H) break;
          int w = std::min(K, W - x * K);
          std::memcpy(r->out.rgba() + (size_t(py) * W + x * K) * 4, src + ly * K * 4, w * 4);
          std::memcpy(r->out.mask() + size_t(py) * W + x * K, src + 4096 + ly * K, w);
        }
        ++t;
      }
  });
}

veil_status veil_render_device(const veil_scene* scene, const veil_render_params* params,
                               const veil_shard* shard) {
  return veil_render_device_timed(scene, params, shard, nullptr, nullptr);
}

veil_status veil_render_device_timed(const veil_scene* scene, const veil_render_params* params,
                                     const veil_shard* shard, void* start_event, void* end_event) {
  if (!scene) return bad_arg("scene is required");
  veil::RenderOptions o = options_from(params);
  o.ev_start = start_event;
  o.ev_end = end_event;
  o.host_readback = false;
  if (o.params.flags & VEIL_RENDER_REFERENCE) return bad_arg("device frames use the pipeline");
  if (shard) {
    if (shard->world_size < 1 || shard->rank < 0 || shard->rank >= shard->world_size)
      return bad_arg("invalid shard");
    o.rank = shard->rank;
    o.world_size = shard->world_size;
  }
  return guard([&] {
    veil::RenderOutput out;
    veil::render_frame(scene->s, o, &out);
  });
}

veil_status veil_measure_disorder(const veil_scene* scene, const veil_render_params* params,
                                  int* max_disorder) {
  if (!scene || !max_disorder) return bad_arg("scene and max_disorder are required");
  veil::RenderOptions o = options_from(params);
  if (o.params.flags & VEIL_RENDER_REFERENCE) return bad_arg("disorder is a property of the pipeline");
  return guard([&] { *max_disorder = veil::measure_disorder(scene->s, o); });
}

veil_status veil_render_scene_multi(const veil_scene* scene, const veil_render_params* params,
                                    const int* devices, int device_count, veil_render** out) {
  if (!scene || !devices || !out) return bad_arg("scene, devices and out_render are required");
  if (device_count < 1 || device_count > 64) return bad_arg("device_count must be in 1..64");
  veil::RenderOptions o = options_from(params);
  if (o.params.flags & VEIL_RENDER_REFERENCE) return bad_arg("the a-buffer renderer does not shard");
  return guard([&] {
    auto r = std::make_unique<veil_render>();
    veil::render_frame_multi(scene->s, o, devices, device_count, &r->out);
    finish_render(scene, o, r.get());
    *out = r.release();
  });
}

veil_status veil_shard_pack_tiles_device(const veil_scene* scene, const veil_shard* shard,
                                         void* dev_tiles, uint64_t bytes) {
  if (!scene || !shard || !dev_tiles) return bad_arg("scene, shard and dev_tiles are required");
  return guard([&] {
    veil::shard_tiles_device(scene->s, shard->rank, shard->world_size, dev_tiles, bytes, false);
  });
}

veil_status veil_shard_unpack_tiles_device(const veil_scene* scene, const veil_shard* shard,
                                           const void* dev_tiles, uint64_t bytes) {
  if (!scene || !shard || !dev_tiles) return bad_arg("scene, shard and dev_tiles are required");
  return guard([&] {
    veil::shard_tiles_device(scene->s, shard->rank, shard->world_size,
                             const_cast<void*>(dev_tiles), bytes, true);
  });
}

veil_status veil_export_framebuffer(const veil_scene* scene, veil_ipc_framebuffer* out) {
  if (!scene || !out) return bad_arg("scene and out are required");
  return guard([&] { veil::export_framebuffer(scene->s, out); });
}

veil_status veil_import_peer_framebuffer(const veil_scene* scene, const veil_ipc_framebuffer* fb) {
  if (!scene) return bad_arg("scene is required");
  return guard([&] { veil::import_peer_framebuffer(scene->s, fb); });
}

veil_status veil_device_framebuffer(const veil_scene* scene, void** rgba, void** mask) {
  if (!scene) return bad_arg("scene is required");
  return guard([&] { veil::device_framebuffer(scene->s, rgba, mask); });
}

void* veil_scene_stream(const veil_scene* scene) {
  return scene ? veil::device_stream(scene->s) : nullptr;
}

veil_status veil_render_stats(const veil_render* r, veil_frame_stats* out) {
  if (!r || !out) return bad_arg("render and out are required");
  *out = r->out.stats;
  return VEIL_OK;
}

veil_status veil_scene_last_stats(const veil_scene* scene, veil_frame_stats* out) {
  if (!scene || !out) return bad_arg("scene and out are required");
  return guard([&] { *out = veil::device_last_stats(scene->s); });
}

veil_status veil_render_scene_dump(const veil_scene* scene, const veil_render_params* params,
                                   veil_render** out) {
  if (!scene || !out) return bad_arg("scene and out_render are required");
  veil::RenderOptions o = options_from(params);
  o.dump = true;
  return do_render(scene, o, out);
}

const void* veil_render_dump_array(const veil_render* r, const char* name, uint64_t* count) {
  if (count) *count = 0;
  if (!r || !name) return nullptr;
  auto it = r->out.dumps.find(name);
  if (it == r->out.dumps.end()) return nullptr;
  if (count) *count = it->second.count;
  static const uint64_t empty = 0;
  return it->second.bytes.empty() ? static_cast<const void*>(&empty) : it->second.bytes.data();
}

}  // extern "C"
