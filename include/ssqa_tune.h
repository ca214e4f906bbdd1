/*
 * ssqa_tune.h -- engine overrides for parity tests and tuning experiments.
 *
 * Not part of the reference interface and not needed by callers: the engine
 * picks operands, geometry and epilogue itself.  The parity tests use these
 * to force every code path (int8 vs FP4 operands, table vs FP64 epilogue,
 * row splits, CTA pairs) against the oracle.  Process-wide, not thread-safe
 * against concurrent launches; nothing is read from the environment.
 *
 * Keys (value -1 / 0 = engine's choice unless noted):
 *   "tab" 1 table epilogue / 0 FP64 epilogue   "fp4"    0 forces int8 operands
 *   "rs" row parts per column tile             "wide"   trials per wide tile cap
 *   "epi" 12 or 16 epilogue warps              "cta2"   0 disables CTA pairs
 *   "stages" / "nps" smem ring shape           "exp"    ablation bits
 *   "i16" 0 refuses the int16 two-plane path    "tskip"  timeline: first row tile recorded
 *   "nccl1" 1: ssqa_run_row_sharded goes through NCCL even with one device
 */
#ifndef SSQA_TUNE_H
#define SSQA_TUNE_H

#ifdef __cplusplus
extern "C" {
#endif

/* Set one override; SSQA_EINVAL for an unknown key. */
int ssqa_tune_set(const char* key, long value);
/* Timeline dump of block 0 into `path` after each fused launch (NULL: off). */
int ssqa_tune_trace(const char* path);
/* Back to the engine's choices. */
void ssqa_tune_reset(void);

#ifdef __cplusplus
}
#endif

#endif
