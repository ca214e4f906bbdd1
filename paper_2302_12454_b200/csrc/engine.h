// engine.h -- internal state behind the C ABI (include/ssqa_cuda.h).
//
// HBM layout:
//   J'    int8  [npad][npad]        row i, column j (K-major for the field
//                                    product); zero padding.
//   H'    int32 [npad]
//   sigma int8  [nslots][ccols][npad] spin columns, K-major (column = one
//                                    (trial, replica)); padded spins are 0.
//   acc   f64   [ccols][npad]       clamped accumulators (ReplicaLattice::is_acc)
// Column c = tile*tile_cols + tl*R + k holds replica k of trial
// t = tile*tpt + tl; a tile keeps whole trials so the Trotter neighbour
// k+-1 (mod R) is always inside the tile.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/ssqa_cuda.h"

namespace ssqa_engine {

// Process-wide engine overrides for the parity tests and tuning experiments
// (include/ssqa_tune.h).  Defaults leave every choice to the engine; nothing
// here is read from the environment.
struct TuneOverrides {
  int tab = -1;     // fast epilogue: 1 table, 0 FP64 (update_fast2), -1 engine's choice
  int fp4 = -1;     // 0: force int8 operands
  int rs = 0;       // > 0: row parts per column tile
  int wide = 0;     // > 0: cap on trials per wide tile
  int epi = 0;      // 12 / 16 epilogue warps (0: default)
  int cta2 = -1;    // 0: no CTA pairs
  int stages = 0;   // > 0: operand stages (with nps)
  int nps = 0;      // accumulator-ring slots per subgroup (with stages)
  int exp = 0;      // ablation experiment bits (TcParams::exp_flags)
  int i16 = -1;     // 0: refuse the int16 (two-plane int8) coupling path
  int nccl1 = 0;    // 1: the C++ row-shard driver uses NCCL even for a single device (tests)
  std::string trace;  // timeline dump path (block 0)
  int tskip = 0;      // timeline: first row tile recorded
};
TuneOverrides& tune();

struct Geom {
  int n = 0, npad = 0;     // spins, padded spins (multiple of 128)
  int R = 0, T = 0;        // replicas, trials
  int tpt = 0;             // trials per column tile
  int tile_cols = 0;       // columns per tile (multiple of 16, >= tpt*R)
  int ntiles = 0;          // column tiles
  int ccols = 0;           // ntiles * tile_cols
  // tcgen05 row split: each column tile is processed by rs CTAs, CTA b owning
  // a contiguous range of row tiles (rs = 1: one CTA runs all rows).
  int rs = 1;
};

struct Quantized {
  int n = 0, npad = 0, p = 0, max_abs_j = 0, max_abs_h = 0;
  double offset = 0.0, scale = 1.0;  // scale = 2^-p
  std::vector<int8_t> J;             // [npad*npad]
  std::vector<int32_t> H;            // [npad]
  // FP4 (e2m1) image of J' when every coupling is one of 0, +-1, +-2, +-3,
  // +-4, +-6: two elements per byte, lower K index in the low nibble.
  bool fp4_ok = false;
  // FP4 pair image (fp4x2_ok, when fp4_ok is not): J' = A1 + A2 with both
  // planes e2m1-exact integers (|J'| <= 12, != 11).  Per K chunk of 128
  // couplings a row holds 64 bytes of A1 nibbles, then 64 bytes of A2
  // nibbles, so one 128-byte TMA row feeds both MMAs of the chunk.
  bool fp4x2_ok = false;
  // int16 couplings (127 < max |J'| <= kI16Max): J' = 256 Ahi + Alo with two
  // signed int8 planes; the device image (d_J) holds, per 64-coupling K chunk
  // of a row, 64 bytes of Alo then 64 bytes of Ahi (rows of 2 npad bytes),
  // and the tcgen05 engine runs one kind::i8 MMA per plane into two
  // accumulators, S = D_lo + 256 D_hi.
  bool i16 = false;
  std::vector<uint8_t> J4;           // [npad * npad/2] (fp4_ok) or [npad * npad] (fp4x2_ok)
};

// e2m1 magnitude codes (0, 1, 2, 3, 4, 6 -> 0, 2, 4, 5, 6, 7) of the FP4 pair
// split |v| = a + b, a >= b, for |v| <= 12; -1 where no split exists (11).
constexpr int kFp4x2A[13] = {0, 2, 4, 5, 6, 6, 7, 7, 7, 7, 7, -1, 7};
constexpr int kFp4x2B[13] = {0, 0, 0, 0, 0, 2, 0, 2, 4, 5, 6, -1, 7};
inline bool fp4x2_splittable(int max_abs) { return max_abs <= 12 && max_abs != 11; }
// int16 planes: Alo = the signed low byte, Ahi = (J' - Alo) / 256 in [-128, 127].
constexpr int kI16Max = 127 * 256 + 127;  // 32639
// Byte offsets of coupling j's A1 / A2 nibbles inside a pair-image row, and
// the nibble shift.
inline size_t fp4x2_byte_a(int j) { return size_t(j >> 7) * 128 + size_t((j & 127) >> 1); }
inline int fp4x2_shift(int j) { return 4 * (j & 1); }

// Returns SSQA_OK or SSQA_EUNSUP with *why set.  p_min: lower bound of the
// scale exponent (several instances quantized at one common scale).
int quantize(int n, const double* h, const double* J, double offset, Quantized* q,
             std::string* why, int p_min = 0);
// Smallest p in [0, 62] with v * 2^p integral, or -1 (the quantizer's rule).
int dyadic_exponent_of(double v);
// FP4 pair image of q.J (see Quantized::fp4x2_ok); false if some |J'| has no split.
bool build_fp4x2(const Quantized& q, std::vector<uint8_t>* out);

}  // namespace ssqa_engine

struct ssqa_problem_s {
  ssqa_engine::Quantized q;  // instance 0 (scale, ranges over all instances)
  // Multi-instance problems (ssqa_problem_create_many): `count` models of the
  // same size at one scale 2^-p, stacked in d_J / d_J4 [count][npad][...] and
  // d_H [count][npad]; trial t of a batch anneals instance t.
  int count = 1;
  std::vector<double> offsets;
  double* d_offsets = nullptr;
  int device = 0;
  cudaStream_t stream = nullptr;
  int8_t* d_J = nullptr;
  int32_t* d_H = nullptr;
  uint8_t* d_J4 = nullptr;  // FP4 couplings (q.fp4_ok) or the FP4 pair image (q.fp4x2_ok)
};

struct ssqa_batch_s {
  ssqa_problem_s* prob = nullptr;
  ssqa_params_c p{};
  ssqa_engine::Geom g;
  int engine = SSQA_ENGINE_SIMT;
  int record_trace = 0;
  int d = 0, nslots = 0;
  size_t slot_elems = 0;  // ccols * npad

  // lattice ring: cur = slot of sigma(cycle); phys[s] = slot of the
  // reference history snapshot s (annealer.hpp:75)
  int cur = 0;
  std::vector<int> phys;
  long cycle = 0;

  int8_t* d_sig = nullptr;    // [nslots][ccols][npad]
  uint8_t* d_sig4 = nullptr;  // FP4 spin slots [nslots][ccols][npad/2] (fused FP4 runs)
  bool lattice_stale = false; // spins live in d_sig4 after an FP4 run
  double* d_acc = nullptr;    // [ccols][npad]
  uint64_t* d_seeds = nullptr;
  double* d_jperp = nullptr;  // [sc+1] jperp_schedule table
  // tcgen05 row split (g.rs > 1): cross-CTA state, zeroed per launch --
  //   gE [2][ccols] int64 energy sums, rows [ntiles][npad/128] row-ready
  //   pass stamps, arrive [ntiles] pass arrivals, scan [ntiles] scan stamps
  void* d_split = nullptr;
  size_t split_bytes = 0;
  // GPU row shard (ssqa_batch_set_shard): this batch updates row tiles
  // [shard * nrt / nshards, (shard + 1) * nrt / nshards) of every column
  int shard = 0, nshards = 1;
  int sh_has_target = 0, sh_stop = 0;
  double sh_target_tol = 0.0;
  // SSA batches (annealer.cpp:489-501): R = 1, delay = 0, jperp = 0 and the
  // accumulator bound follows i0_schedule (annealer.cpp:403-408) per cycle.
  bool ssa = false;
  int ssa_tau = 1;
  std::vector<double> ssa_levels;  // SsaParams::i0_levels()
  double* d_i0 = nullptr;          // [sc+1] i0_schedule table (SSA only)
  int32_t* d_S = nullptr;     // SIMT engine: integer fields [ccols][npad]
  long long* d_E = nullptr;
  unsigned* d_push_ctr = nullptr;  // peer push: blocks done in the current pack (ssqa_batch_shard_pass_to)   // per-column integer energy sum E' [ccols]

  // per-trial results
  double* d_best_e = nullptr;
  int* d_best_k = nullptr;
  int* d_reached = nullptr;
  long* d_first_hit = nullptr;
  long* d_cycles_used = nullptr;
  int* d_active = nullptr;
  int8_t* d_best_state = nullptr;  // [T][n]
  uint8_t* d_best_packed = nullptr; // tcgen05: best spin column as stored in a slot [T][npad]
  double* d_trace = nullptr;       // [T][sc+1][R]

  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  long launches = 0;
  bool seeds_set = false;
};
