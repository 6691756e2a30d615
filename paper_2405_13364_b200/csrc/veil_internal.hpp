// Host-side data model of libveil (C++17). The scene lives in host arrays
// laid out exactly like the C structures of veil_cuda.h; a device mirror and
// the frame workspace are attached lazily by the CUDA pipeline
// (pipeline.cu). Reference counterparts: proj/include/veil/scene.hpp:33-134.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/veil.h"
#include "../../include/veil_cuda.h"

namespace veil {

// Error categories of the reference (proj/include/veil/error.hpp:22-39); the
// C ABI maps them to veil_status.
class Error : public std::runtime_error {
 public:
  Error(veil_status status, const std::string& message)
      : std::runtime_error(message), status_(status) {}
  veil_status status() const { return status_; }

 private:
  veil_status status_;
};

constexpr int kBinSize = 32;
constexpr int kMaxViewportWidth = 2560;   // reference scene.hpp:90
constexpr int kMaxViewportHeight = 2048;  // reference scene.hpp:91
constexpr int kMaxBins = 5120;            // reference setup.hpp:31
constexpr int kExtMaxViewport = 16384;    // extended-limits mode

struct TextureLevel {
  int width = 0, height = 0;
  std::vector<float> texels;  // straight RGBA, 4 floats per texel
};

struct Texture {
  std::vector<TextureLevel> levels;
};

struct Camera {
  double m[16] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1};  // row-major
  int width = 512, height = 512;
  bool has_eye = false;
  double eye[3] = {0, 0, 0};
};

struct DeviceScene;  // pipeline.cu

struct Scene {
  std::vector<veil_vertex> vertices;
  std::vector<veil_quad> quads;
  std::vector<veil_material> materials;
  std::vector<std::string> material_names;
  std::vector<Texture> textures;
  uint32_t flags = 0;  // veil_scene_flags
  Camera camera;
  bool extended = false;
  uint64_t geometry_version = 1;  // bumped on every geometry/material change
  mutable uint64_t validated_version = 0;  // geometry_version last checked by validate_scene
  mutable uint64_t degenerate_version = 0;  // geometry_version of degenerate_cache
  mutable double degenerate_cache = 0.0;

  Scene();
  ~Scene();
  Scene(const Scene&) = delete;
  Scene& operator=(const Scene&) = delete;

  double degenerate_quad_percent() const;
  mutable DeviceScene* device = nullptr;  // owned; see pipeline.cu
  mutable std::vector<DeviceScene*> shards;  // owned: veil_render_scene_multi workspaces
};

// --- scene ingest (scene_io.cpp) -------------------------------------------
void validate_camera(const Camera& cam, bool extended);
void validate_scene(const Scene& s);
void load_obj_scene(Scene* s, const std::string& mesh, const std::string& mtl,
                    const std::string& cam);
Camera load_camera_file(const std::string& path);
Camera look_at_camera(const double from[3], const double at[3], const double up[3],
                      double fov_deg, double near_z, double far_z, int width, int height);
void synthetic_scene(Scene* s, const std::string& kind, uint64_t seed, int width, int height);
void workload_scene(Scene* s, const std::string& name, uint64_t seed, int width, int height);
double group_quads(Scene* s);
bool mat4_inverse(const double* in, double* out);

// --- images (image_io.cpp) -------------------------------------------------
struct Image8 {
  int width = 0, height = 0;
  std::vector<uint8_t> rgba;
};
Image8 read_png(const std::string& path);
void write_png(const Image8& img, const std::string& path);

// --- rendering -------------------------------------------------------------
struct RenderOptions {
  veil_render_params params;
  int rank = 0, world_size = 1;
  bool dump = false;          // capture parity arrays
  bool host_readback = true;  // copy framebuffer + mask to the host
  bool keep_records = false;  // store every triangle record even in the fused raster
  void* ev_start = nullptr;   // caller's cudaEvent_t pair around the frame's device work
  void* ev_end = nullptr;
};

struct DumpArray {
  std::vector<uint8_t> bytes;
  uint64_t count = 0;
};

// Pinned, pooled host buffer for a frame: RGBA8 (4 B/px) then the invalid
// mask (1 B/px). Returned to the pool when the last owner releases it.
std::shared_ptr<uint8_t> acquire_host_frame(size_t bytes);

struct RenderOutput {
  int width = 0, height = 0;
  std::shared_ptr<uint8_t> host;  // see acquire_host_frame
  uint8_t* rgba() const { return host.get(); }
  uint8_t* mask() const { return host ? host.get() + size_t(width) * height * 4 : nullptr; }
  veil_frame_stats stats{};
  bool reference = false;
  std::map<std::string, DumpArray> dumps;
};

// Runs one frame on the current CUDA device (pipeline.cu).
void render_frame(const Scene& scene, const RenderOptions& opt, RenderOutput* out);
void render_reference_frame(const Scene& scene, const RenderOptions& opt, RenderOutput* out);
void render_frame_multi(const Scene& scene, const RenderOptions& opt, const int* devices, int n,
                        RenderOutput* out);
int measure_disorder(const Scene& scene, const RenderOptions& opt);
void release_device_scene(DeviceScene* d);
void device_framebuffer(const Scene& scene, void** rgba, void** mask);
void export_framebuffer(const Scene& scene, veil_ipc_framebuffer* out);
void import_peer_framebuffer(const Scene& scene, const veil_ipc_framebuffer* fb);
void shard_tiles_device(const Scene& scene, int rank, int world, void* tiles, uint64_t bytes,
                        bool unpack);
void* device_stream(const Scene& scene);
const veil_frame_stats& device_last_stats(const Scene& scene);
void set_current_device(int device);
uint64_t shard_tile_count(int bins_x, int bins_y, int rank, int world);
bool bin_owned(int bx, int by, int rank, int world);

std::string report_json(const RenderOutput& out, const veil_render_params& p, int width,
                        int height, double degenerate_percent);

}  // namespace veil

struct veil_scene {
  veil::Scene s;
};

struct veil_render {
  veil::RenderOutput out;
  std::string json;
};
