// simt_kernels.cuh -- declarations for lattice init, per-trial scan and the CUDA-core sweep
// engine (SSQA_ENGINE_SIMT).  The tcgen05 engine (sweep_tc.cu) reuses the
// init and scan kernels and the ssqa_device.cuh update arithmetic.
#pragma once

#include <cstdint>

#include "engine.h"
#include "ssqa_device.cuh"
#include <cuda_runtime.h>

namespace ssqa_engine {

using namespace ssqa_dev;

struct ColInfo {
  int t, k;
  bool live;
};

__host__ __device__ __forceinline__ ColInfo decode_col(const Geom& g, int col) {
  ColInfo c;
  const int tile = col / g.tile_cols, w = col - tile * g.tile_cols;
  const int tl = w / g.R;
  c.k = w - tl * g.R;
  c.t = tile * g.tpt + tl;
  c.live = (tl < g.tpt) && (c.t < g.T);
  return c;
}

__host__ __device__ __forceinline__ int col_of(const Geom& g, int t, int k) {
  const int tile = t / g.tpt, tl = t - tile * g.tpt;
  return tile * g.tile_cols + tl * g.R + k;
}


constexpr int kFB = 64;  // field tile of the SIMT engine

struct StepArgs {
  long cycle;
  double jperp, i0, n_rnd, alpha;
  int bidirectional;
  int do_update;
};

struct ScanArgs {
  long cycle, sc;
  double scale, offset;
  int has_target;
  double target_tol;  // target + kTargetTol (annealer.hpp:113), formed on the host
  int stop_at_target;
  int record_trace;
};

void launch_init(const Geom& g, const uint64_t* seeds, int8_t* sig, double* acc,
                 cudaStream_t st);
// GPU row shards: pack rows [row0, row0+rows) of every column of an int8
// spin slot (bit-packed) plus the energy partials into one exchange chunk;
// unpack all shards' chunks into the slot and sum their energy partials.
// Where a shard's exchange chunk goes: n destinations (the caller's own
// buffer, or the shard's slot in every GPU's exchange region through peer
// pointers); counter != nullptr: the last block then raises flag[d] = epoch.
constexpr int kMaxPeers = 8;
struct PeerPush {
  uint8_t* dst[kMaxPeers];
  unsigned* flag[kMaxPeers];
  unsigned* counter;
  unsigned epoch;
  int n;
};
// Before unpacking: wait until flags[0..n) all reach epoch (flags == nullptr: no wait).
struct PeerWait {
  const unsigned* flags;
  unsigned epoch;
  int n;
};
void launch_shard_pack(const Geom& g, const int8_t* slot, int row0, int rows,
                       const unsigned long long* E, const PeerPush& pp, cudaStream_t st);
// FP4 slot variant of launch_shard_pack (tcgen05 FP4 / FP4-pair shard passes).
void launch_shard_pack_fp4(const Geom& g, const uint8_t* slot4, int row0, int rows,
                           const unsigned long long* E, const PeerPush& pp, cudaStream_t st);
// Fused exchange: wait for the peers' flags, sum the nshards int64 partial
// rows (part_stride bytes apart) into E, expand the FP4 slot into the int8
// slot (with_spins).
void launch_shard_merge_direct(const Geom& g, int8_t* slot, const uint8_t* slot4,
                               const void* parts, size_t part_stride, int nshards,
                               bool with_spins, long long* E, const PeerWait& pw,
                               cudaStream_t st);
// slot4 (nullable): also write the FP4 image of the gathered spins.
void launch_shard_unpack(const Geom& g, int8_t* slot, uint8_t* slot4, const void* all,
                         size_t chunk_bytes, int nshards, int rows_per_shard, bool with_spins,
                         long long* E, const PeerWait& pw, cudaStream_t st);
void launch_reset_results(int T, long sc, double* best_e, int* best_k, int* reached,
                          long* first_hit, long* cycles_used, int* active, cudaStream_t st);
void launch_field_simt(const Geom& g, const int8_t* J, const int8_t* sig, int32_t* S,
                       cudaStream_t st);
void launch_energy_update_simt(const Geom& g, const int32_t* S, const int32_t* H, double scale,
                               const uint64_t* seeds, const int8_t* sig_cur,
                               const int8_t* sig_src, int8_t* sig_dst, double* acc,
                               long long* E, const StepArgs& a, cudaStream_t st);
void launch_scan(const Geom& g, const long long* E, const ScanArgs& a, const int8_t* sig_cur,
                 double* best_e, int* best_k, int* reached, long* first_hit, long* cycles_used,
                 int* active, int8_t* best_state, double* trace, cudaStream_t st);

}  // namespace ssqa_engine
