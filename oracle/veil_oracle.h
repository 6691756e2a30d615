/*
 * veil_oracle.h -- CPU restatement of the reference pipeline (TEST
 * INFRASTRUCTURE ONLY).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load liboracle.so, and only as the checker or
 * the timed CPU baseline, never as part of the product path.
 *
 * Parity pinning: the restatement is checked bit-for-bit against the
 * unmodified reference compiled in oracle/_ref (tests/test_oracle_vs_ref.py)
 * and against the committed fixtures in tests/golden/ that the reference
 * produced (oracle/make_golden.py).
 */
#ifndef VEIL_ORACLE_H_
#define VEIL_ORACLE_H_

#include <stdint.h>

#include "../include/veil_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vo_frame vo_frame;

/* Runs the sort-middle pipeline (or the a-buffer renderer when
 * params->flags has VEIL_RENDER_REFERENCE). extended != 0 lifts the viewport /
 * bin / index limits the same way veil_scene_set_extended_limits does.
 * Returns a veil_status; *out is set even on failure (holds the message). */
int vo_render(const veil_scene_desc* scene, const veil_render_params* params, int extended,
              vo_frame** out);

/* Arrays named like veil_render_dump_array (veil_cuda.h), plus "image",
 * "mask", "counters" (u64: samples fragments thb segments bins_empty
 * bins_low bins_high bins_propagated invalid_pixels). */
const void* vo_array(const vo_frame* frame, const char* name, uint64_t* count);
const char* vo_message(const vo_frame* frame);
void vo_free(vo_frame* frame);

#ifdef __cplusplus
}
#endif

#endif
