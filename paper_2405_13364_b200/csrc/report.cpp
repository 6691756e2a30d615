// JSON run report with the reference's stable schema (proj/src/report.cpp:
// 21-68: config echo, timings_us, samples, tri_half_blocks, s_per_thb,
// fragments, segments, setup_stats, bins, invalid_pixels) followed by an
// additive "device" object (CUDA-event stage times in ms, kernel launches,
// bin pairs). Keys keep the reference's order.
#include <cmath>
#include <cstdio>
#include <sstream>
#include <thread>

#include "veil_internal.hpp"

namespace veil {

namespace {

// Shortest round-trip decimal; integral values keep a ".0" like nlohmann.
std::string num(double v) {
  if (!std::isfinite(v)) return "null";
  char buf[64];
  for (int p = 1; p <= 17; ++p) {
    std::snprintf(buf, sizeof buf, "%.*g", p, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string s = buf;
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

struct Writer {
  std::ostringstream o;
  int depth = 0;
  bool first = true;
  void indent() {
    o << "\n";
    for (int i = 0; i < depth; ++i) o << "  ";
  }
  void key(const char* k) {
    if (!first) o << ",";
    first = false;
    indent();
    o << "\"" << k << "\": ";
  }
  void open(const char* k) {
    key(k);
    o << "{";
    depth++;
    first = true;
  }
  void close() {
    depth--;
    indent();
    o << "}";
    first = false;
  }
  void u(const char* k, uint64_t v) { key(k), o << v; }
  void i(const char* k, long long v) { key(k), o << v; }
  void d(const char* k, double v) { key(k), o << num(v); }
  void b(const char* k, bool v) { key(k), o << (v ? "true" : "false"); }
};

}  // namespace

std::string report_json(const RenderOutput& out, const veil_render_params& p, int width,
                        int height, double degenerate_percent) {
  const veil_frame_stats& s = out.stats;
  Writer w;
  w.o << "{";
  w.depth = 1;
  int threads = p.thread_count > 0 ? p.thread_count : int(std::thread::hardware_concurrency());
  if (threads <= 0) threads = 1;
  w.open("config");
  w.i("width", width);
  w.i("height", height);
  w.i("depth_filter_size", p.depth_filter_size);
  w.i("threads", threads);
  w.b("alpha_threshold", p.flags & VEIL_RENDER_ALPHA_THRESHOLD);
  w.b("visualize_errors", p.flags & VEIL_RENDER_VISUALIZE_ERRORS);
  w.b("backface_culling", p.flags & VEIL_RENDER_BACKFACE_CULLING);
  w.b("force_high_path", p.flags & VEIL_RENDER_FORCE_HIGH_PATH);
  w.b("reference", out.reference);
  w.close();
  auto us = [](double ms) { return uint64_t(std::llround(ms * 1000.0)); };
  w.open("timings_us");
  w.u("setup", us(s.setup_ms));
  w.u("binning", us(s.binning_ms));
  w.u("low_raster", us(s.low_raster_ms));
  w.u("hi_raster", us(s.hi_raster_ms));
  w.u("total", us(s.total_ms));
  w.close();
  w.u("samples", s.samples);
  w.u("tri_half_blocks", s.tri_half_blocks);
  w.d("s_per_thb", s.tri_half_blocks ? double(s.samples) / double(s.tri_half_blocks) : 0.0);
  w.u("fragments", s.fragments);
  w.u("segments", s.segments);
  w.open("setup_stats");
  w.u("input_quads", s.input_quads);
  w.u("visible_quads", s.visible_quads);
  w.d("visible_percent",
      s.input_quads ? 100.0 * double(s.visible_quads) / double(s.input_quads) : 0.0);
  w.u("culled_degenerate", s.culled_degenerate);
  w.u("culled_backfacing", s.culled_backfacing);
  w.u("culled_frustum", s.culled_frustum);
  w.u("culled_between_samples", s.culled_between_samples);
  w.d("degenerate_quad_percent", degenerate_percent);
  w.close();
  w.open("bins");
  w.u("empty", s.bins_empty);
  w.u("low", s.bins_low);
  w.u("high", s.bins_high);
  w.u("propagated", s.bins_propagated);
  w.close();
  w.open("invalid_pixels");
  w.u("count", s.invalid_pixels);
  double npx = double(width) * double(height);
  w.d("percent", npx > 0 ? 100.0 * double(s.invalid_pixels) / npx : 0.0);
  w.close();
  w.open("device");
  w.d("setup_ms", s.setup_ms);
  w.d("binning_ms", s.binning_ms);
  w.d("low_raster_ms", s.low_raster_ms);
  w.d("hi_raster_ms", s.hi_raster_ms);
  w.d("total_ms", s.total_ms);
  w.u("kernel_launches", s.kernel_launches);
  w.u("bin_pairs", s.bin_pairs);
  w.u("small_quads", s.small_quads);
  w.u("large_tris", s.large_tris);
  w.close();
  w.depth = 0;
  w.indent();
  w.o << "}";
  return w.o.str();
}

}  // namespace veil
