/*
 * veil_cuda.h -- additive B200 extensions of libveil.so.
 *
 * Nothing here changes a type or function of veil.h; an embedder of the
 * reference ignores this header. It adds what the reference has no slot
 * for:
 *   - scenes built from host arrays and exported back (the reference only
 *     builds scenes from OBJ files or its own generators, veil.h:48-56),
 *   - the benchmark workloads of BASELINE.json (stack64k, tiny4m,
 *     mixed16m) as deterministic generators,
 *   - extended limits (viewports beyond 2560x2048, proj/include/veil/
 *     scene.hpp:90-91; more than 5120 bins, setup.hpp:31),
 *   - device selection and bin-interleaved screen sharding across GPUs,
 *   - per-stage device timings (CUDA events) and parity dumps of the
 *     intermediate buffers (visible quads, triangle setups, bin lists,
 *     tri-half-block lists, per-pixel blend-order hashes).
 */
#ifndef VEIL_CUDA_H_
#define VEIL_CUDA_H_

#include "veil.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- array scenes --------------------------------------------------------- */

/* Same field order and meaning as the reference's Vertex (scene.hpp:33-38). */
typedef struct veil_vertex {
  float position[3];
  float normal[3];
  float color[4];
  float uv[2];
} veil_vertex; /* 48 bytes */

/* Triangles (v0,v1,v2) and (v0,v2,v3); scene.hpp:42-52. */
typedef struct veil_quad {
  uint32_t v[4];
  uint32_t material;
} veil_quad; /* 20 bytes */

enum veil_material_flags {
  VEIL_MATERIAL_VERTEX_COLORS = 1 << 0,
  VEIL_MATERIAL_VERTEX_NORMALS = 1 << 1,
  VEIL_MATERIAL_UVS = 1 << 2
};

typedef struct veil_material {
  float base_color[4];
  float opacity;
  int32_t texture; /* -1 = none */
  uint32_t flags;  /* veil_material_flags */
} veil_material;

enum veil_scene_flags {
  VEIL_SCENE_HAS_NORMALS = 1 << 0,
  VEIL_SCENE_HAS_COLORS = 1 << 1,
  VEIL_SCENE_HAS_UVS = 1 << 2
};

typedef struct veil_scene_desc {
  const veil_vertex* vertices;
  uint64_t vertex_count;
  const veil_quad* quads;
  uint64_t quad_count;
  const veil_material* materials;
  uint32_t material_count;
  uint32_t flags; /* veil_scene_flags */
  double view_projection[16]; /* row-major */
  int32_t width;
  int32_t height;
  int32_t has_eye;
  int32_t reserved;
  double eye[3];
} veil_scene_desc;

/* Copies the arrays into a new scene (textures are not supported here). */
veil_status veil_scene_create(const veil_scene_desc* desc, veil_scene** out_scene);

/* Read-only view of a scene's host arrays; valid until the scene changes. */
veil_status veil_scene_describe(const veil_scene* scene, veil_scene_desc* out_desc);

/* BASELINE.json workloads: "stack64k" (C2), "tiny4m" (C4),
 * "mixed16m" (C5). width/height <= 0 pick the config's own viewport. */
veil_status veil_scene_workload(const char* name, uint64_t seed, int width, int height,
                                veil_scene** out_scene);

/* make_look_at_camera (proj/src/scene.cpp:128-158) as a C call. */
veil_status veil_camera_look_at(const double from[3], const double at[3], const double up[3],
                                double fov_deg, double near_z, double far_z, int width,
                                int height, double out_matrix[16]);

/* Lifts the reference's structural limits for this scene: viewports up to
 * 16384x16384, any bin count, 32-bit visible-triangle indices. Results are
 * identical to the reference on every scene within its limits. */
veil_status veil_scene_set_extended_limits(veil_scene* scene, int enable);
veil_status veil_scene_set_viewport_ext(veil_scene* scene, int width, int height);

/* ---- device and sharding -------------------------------------------------- */

/* CUDA device used by subsequent calls on this thread (default 0). */
veil_status veil_cuda_set_device(int device);

/* Bin-interleaved screen sharding: rank r of world_size renders the bins it
 * owns (owner(bx,by) = (bx + 3*by) mod world_size). Setup is replicated so
 * visible indices stay global; see DESIGN.md. world_size 1 = whole frame. */
typedef struct veil_shard {
  int32_t rank;
  int32_t world_size;
} veil_shard;

veil_status veil_render_scene_shard(const veil_scene* scene, const veil_render_params* params,
                                    const veil_shard* shard, veil_render** out_render);

/* Owned 32x32 tiles of a sharded render packed densely (RGBA8 then mask):
 * tile i of the rank is bins[i]; 4096 + 1024 bytes each. */
uint64_t veil_shard_tile_count(int bins_x, int bins_y, const veil_shard* shard);
veil_status veil_shard_pack_tiles(const veil_render* render, const veil_shard* shard,
                                  uint8_t* out, uint64_t out_bytes);
veil_status veil_shard_unpack_tiles(veil_render* render, const veil_shard* shard,
                                    const uint8_t* tiles, uint64_t bytes);

/* Device-memory variants on the scene's last device frame (the NCCL gather
 * path): pack this rank's owned tiles into dev_tiles / write tiles received
 * for `shard` into the scene's device framebuffer. Synchronous. */
veil_status veil_shard_pack_tiles_device(const veil_scene* scene, const veil_shard* shard,
                                         void* dev_tiles, uint64_t bytes);
veil_status veil_shard_unpack_tiles_device(const veil_scene* scene, const veil_shard* shard,
                                           const void* dev_tiles, uint64_t bytes);

/* Peer framebuffer gather (one process per GPU on one node): the root rank
 * (shard rank 0) exports its device framebuffer as CUDA IPC handles; every
 * other rank imports them, after which its sharded frames also write their
 * finished pixels straight into the root's framebuffer over NVLink during
 * shading -- no pack, collective or unpack. The caller orders frames with a
 * host barrier after each rank's frame. The handles stay valid while the
 * root keeps its viewport (a larger viewport reallocates the framebuffer:
 * export and import again). Import NULL to detach. */
typedef struct veil_ipc_framebuffer {
  uint8_t rgba[64];
  uint8_t mask[64];
  int32_t width;
  int32_t height;
} veil_ipc_framebuffer;

veil_status veil_export_framebuffer(const veil_scene* scene, veil_ipc_framebuffer* out);
veil_status veil_import_peer_framebuffer(const veil_scene* scene, const veil_ipc_framebuffer* fb);

/* Multi-GPU frame in one process (no IPC, no collective): the frame's bins are
 * interleaved over device_count shards exactly as in veil_render_scene_shard
 * (shard i = rank i, on devices[i]; setup replicated per device). Every shard
 * renders concurrently in its own workspace and host thread, and its shading
 * kernels write their finished pixels straight into devices[0]'s framebuffer
 * (peer memory over NVLink; the same buffer when a device appears twice), so
 * the gather overlaps the shading and the frame is read back once. The
 * render's pixels, mask, report and stats describe the whole frame; stage
 * times in veil_render_stats are the maximum over shards. Requires peer
 * access from every device to devices[0]. Output is identical for any
 * device list. */
veil_status veil_render_scene_multi(const veil_scene* scene, const veil_render_params* params,
                                    const int* devices, int device_count, veil_render** out_render);

/* The pipeline's maximum per-pixel sort disorder for these parameters
 * (reference RenderConfig::measure_disorder, raster.cpp:286-297: over every
 * pixel, the largest i - position-in-sorted-order of its i-th arriving sample),
 * which the reference reports as "max_disorder" but its C ABI cannot request.
 * A depth filter of at least this size renders every pixel in exact order
 * (acceptance.cpp:115-126). One device frame plus an O(n^2)-per-pixel pass. */
veil_status veil_measure_disorder(const veil_scene* scene, const veil_render_params* params,
                                  int* max_disorder);

/* ---- device-resident frame loop ------------------------------------------- */

/* Renders into device memory only (no host copies); for benchmarks that time
 * the device path. Output stays on the scene's device workspace. */
veil_status veil_render_device(const veil_scene* scene, const veil_render_params* params,
                               const veil_shard* shard);
/* veil_render_device that also records two caller-owned CUDA events
 * (cudaEvent_t as void*, either may be NULL) on the scene's stream: `start`
 * immediately before the frame's work (its graph launch) and `end` right after
 * it, before the call waits for the frame. cudaEventElapsedTime(start, end) is
 * then the device time of exactly the frame, without the host's launch
 * preparation or its wake-up after the wait. A frame that re-runs to grow a
 * buffer records them around its last attempt. */
veil_status veil_render_device_timed(const veil_scene* scene, const veil_render_params* params,
                                     const veil_shard* shard, void* start_event, void* end_event);
/* Device pointers of the last veil_render_device() output. */
veil_status veil_device_framebuffer(const veil_scene* scene, void** rgba, void** mask);
/* CUDA stream the scene's kernels run on (cudaStream_t as void*). */
void* veil_scene_stream(const veil_scene* scene);

/* ---- timings and counters ------------------------------------------------- */

typedef struct veil_frame_stats {
  /* CUDA events. low_raster_ms covers low-path extraction and all shading
   * (shade_ms), hi_raster_ms the high-path extraction. */
  double setup_ms, binning_ms, low_raster_ms, hi_raster_ms, total_ms;
  uint64_t samples, fragments, tri_half_blocks, segments;
  uint64_t input_quads, visible_quads;
  uint64_t culled_degenerate, culled_backfacing, culled_frustum, culled_between_samples;
  uint64_t bins_empty, bins_low, bins_high, bins_propagated;
  uint64_t invalid_pixels;
  uint64_t bin_pairs;   /* sum of per-bin list lengths */
  uint64_t small_quads; /* visible small quads */
  uint64_t large_tris;  /* valid triangles of large quads */
  uint64_t kernel_launches;
  double shade_ms; /* CUDA events: shading share of the raster time */
} veil_frame_stats;

veil_status veil_render_stats(const veil_render* render, veil_frame_stats* out);
/* Stats of the last veil_render_device() call on this scene. */
veil_status veil_scene_last_stats(const veil_scene* scene, veil_frame_stats* out);

/* ---- parity dumps (tests) -------------------------------------------------- */

/* Runs a frame with dump capture enabled and keeps the intermediate buffers
 * on the render handle. Names (element type):
 *   quad_source u32, quad_aabb u32, quad_class u8, quad_attr u32[9],
 *   tri_valid u8, tri_yrange i32[2], tri_fn f64[15], tri_meta u32[4],
 *   setup_stats u64[6], bin_dims i32[2], bin_quad_counts u32,
 *   bin_tri_counts u32, bin_offsets u32, bin_categories u8, bin_items u32,
 *   bin_path u8, thb_offsets u64, thb u64, thb_prefix u32, emit_hash u64,
 *   emit_count u32. */
veil_status veil_render_scene_dump(const veil_scene* scene, const veil_render_params* params,
                                   veil_render** out_render);
const void* veil_render_dump_array(const veil_render* render, const char* name,
                                   uint64_t* out_count);

#ifdef __cplusplus
}
#endif

#endif /* VEIL_CUDA_H_ */
