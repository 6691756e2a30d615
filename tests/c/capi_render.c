/* A plain C embedder of the reference's interface (include/veil.h), linked
 * against libveil.so exactly as an application linked against the
 * reference's `veil` library would be (reference tests/test_capi.cpp and
 * tools/veil_cli.cpp use the same calls). Renders a synthetic scene, writes
 * the PNG, the raw RGBA8 + invalid-mask bytes and prints the JSON report.
 *
 *   capi_render <kind> <seed> <width> <height> <depth_filter> <out.png> <out.raw>
 */
#include <stdio.h>
#include <stdlib.h>

#include "veil.h"

static int fail(const char* what, veil_status st) {
  fprintf(stderr, "%s: %s (%s)\n", what, veil_status_string(st), veil_last_error());
  return 2;
}

int main(int argc, char** argv) {
  if (argc != 8) {
    fprintf(stderr, "usage: %s kind seed width height depth_filter out.png out.raw\n", argv[0]);
    return 1;
  }
  veil_scene* scene = NULL;
  veil_render* frame = NULL;
  veil_render_params params;
  veil_status st;
  FILE* f;
  int w, h;

  veil_render_params_init(&params);
  params.depth_filter_size = atoi(argv[5]);
  st = veil_scene_synthetic(argv[1], (uint64_t)strtoull(argv[2], NULL, 10), atoi(argv[3]),
                            atoi(argv[4]), &scene);
  if (st != VEIL_OK) return fail("veil_scene_synthetic", st);
  st = veil_render_scene(scene, &params, &frame);
  if (st != VEIL_OK) return fail("veil_render_scene", st);
  w = veil_render_width(frame);
  h = veil_render_height(frame);
  st = veil_render_write_png(frame, argv[6]);
  if (st != VEIL_OK) return fail("veil_render_write_png", st);
  f = fopen(argv[7], "wb");
  if (!f) return 3;
  fwrite(veil_render_pixels(frame), 1, (size_t)w * (size_t)h * 4, f);
  fwrite(veil_render_invalid_mask(frame), 1, (size_t)w * (size_t)h, f);
  fclose(f);
  printf("%s\n", veil_render_report_json(frame));
  veil_render_destroy(frame);
  veil_scene_destroy(scene);
  /* NULL-safe destroy and error paths, as the reference documents */
  veil_render_destroy(NULL);
  veil_scene_destroy(NULL);
  return 0;
}
