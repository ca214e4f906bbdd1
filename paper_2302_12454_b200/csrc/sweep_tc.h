// sweep_tc.h -- the fused tcgen05 sweep engine (SSQA_ENGINE_TCGEN05).
#pragma once

#include <string>

#include "engine.h"
#include "simt_kernels.cuh"

namespace ssqa_engine {

// True when the tcgen05 kernel handles this padded size / replica count.
bool tc_supported(int npad, int r, int delay);
// Operand format a fused run of this batch streams: FP4 (e2m1) or int8.
bool tc_uses_fp4(const ssqa_batch_s* b);
// int8 spin slots -> FP4 (e2m1) slots, `bytes` FP4 bytes (two spins each).
void launch_pack_fp4(const int8_t* src, uint8_t* dst, size_t bytes, cudaStream_t st);
// Full run: cycles 0..sc with scans (state already initialised).
int tc_run(ssqa_batch_s* b, const ScanArgs& sa);
// One sweep at b->cycle without a scan (per-step API).
int tc_sweep(ssqa_batch_s* b, double jperp, double i0);
// GPU row shard: one pass at b->cycle over row tiles [rt0, rt0 + nrt) with
// the batch's operand format (int8 slots, or FP4 slots when tc_uses_fp4:
// sigma(c+1) of those rows, acc), the pass energies' row
// partials added into gE[ccols] (zeroed by the caller); the ring is not
// advanced (the caller merges all shards' rows first).
int tc_shard_pass(ssqa_batch_s* b, int rt0, int nrt, unsigned long long* gE);
// Shard pass with the exchange fused in (sweep_tc.cu, TcParams::npeer).
bool tc_shard_direct_ok(ssqa_batch_s* b);
int tc_shard_pass_direct(ssqa_batch_s* b, int rt0, int nrt, unsigned long long* gE,
                         const long long* peer_delta, unsigned long long* const* peer_E,
                         unsigned* const* peer_flag, int npeer, unsigned epoch,
                         unsigned* push_ctr);
const char* tc_last_error();
// Non-empty after a kernel watchdog fired: who was stuck on which mbarrier.
std::string tc_watchdog_message();

}  // namespace ssqa_engine
