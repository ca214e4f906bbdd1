// sweep_tc.cu -- the fused tcgen05 SSQA sweep engine (SSQA_ENGINE_TCGEN05).
//
// One persistent CTA per column tile (whole trials, <= 256 replica columns)
// runs every sweep of the batch without leaving the kernel:
//
//   warp 0      TMA producer: J' row tile [128 x 128 B] + spin tile
//               [NT cols x 128 B] per K chunk into a STAGES-deep smem ring
//               (SWIZZLE_128B, K-major), completion on mbarriers.
//   warp 1      TMEM allocator + MMA issuer: one elected thread issues
//               tcgen05.mma.cta_group::1.kind::i8 (M=128 rows i, N=NT columns,
//               K=32) accumulating int32 fields S = J' sigma in TMEM; two
//               accumulator buffers so the epilogue of row tile r overlaps the
//               MMAs of row tile r+1.
//   warps 2..9  epilogue: tcgen05.ld the int32 fields (thread = spin row i,
//               registers = columns), integer energy partials (warp REDUX),
//               counter-RNG noise, delayed Trotter coupling and the exact FP64
//               clamp of update_spins (annealer.cpp:258-300), new spins
//               written K-major for the next sweep's TMA.
//
// Between sweeps the CTA synchronises once, scans its trials
// (annealer.cpp:327-345) and advances the spin-slot ring.  No grid-wide sync:
// a tile's columns depend only on its own spins (F[:, cols] = J' sigma[:, cols]).
#include "devpool.h"
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <vector>

#include "sweep_tc.h"

namespace ssqa_engine {

namespace {

constexpr int kBM = 128;          // rows (spins i) per MMA tile
constexpr int kBK = 128;          // K bytes per stage (one 128B swizzle row)
constexpr int kCW = 8;  // columns per epilogue chunk (one tcgen05.ld .x8)
#ifndef SSQA_ABL
// Timing ablations (scripts/build_ablations.sh), 0 in the product: 16 no energy
// reduction, 32 no spin store, 64 no accumulator store, 128 no accumulator
// stream (stale smem), 256 no TMEM load, 512 no counter RNG (placeholder noise),
// 1024 spin words built but not stored, 2048 no ballots (spin words from one lane).
#define SSQA_ABL 0
#endif
#ifndef SSQA_EPI_V
#define SSQA_EPI_V 1  // FP64 epilogue: 1 issue-lean noise draw (noise_top5 / noise_lut), 0 previous
#endif
#ifndef SSQA_LAZY_NS_MMA
#define SSQA_LAZY_NS_MMA 128   // MMA issuer waiting for a free accumulator buffer
#endif
#ifndef SSQA_LAZY_NS_PROD
#define SSQA_LAZY_NS_PROD 32   // operand producer waiting for a free stage
#endif
#ifndef SSQA_LAZY_NS_LOAD
#define SSQA_LAZY_NS_LOAD 128  // state loaders waiting for a free slot / tile buffer
#endif
#ifndef SSQA_ENERGY_RED
#define SSQA_ENERGY_RED 1  // 1: shuffle transpose-reduce, 0: per-column redux.sync
#endif
constexpr uint32_t kSfCol = 480;  // FP4 scale-factor TMEM columns [480, 512)
constexpr int kMaxDelay = 30;
constexpr int kMaxRowGroups = 64;
constexpr int kMaxCols = 256;
constexpr int kMaxTrialsPerTile = 256;

thread_local std::string g_tc_err;

struct TcParams {
  Geom g;
  const int32_t* H;
  double scale, offset;
  int shift_p;
  const uint64_t* seeds;
  int8_t* sig;
  uint8_t* sig_base;  // slots the kernel reads/writes (d_sig or the FP4 d_sig4)
  size_t slot_elems;
  int nslots, d;
  double* acc;
  const double* jperp_tab;  // per-cycle jperp (run mode)
  const double* i0_tab;     // per-cycle bound (SSA run mode), else nullptr
  double jperp_fixed;       // sweep mode
  double i0, n_rnd, alpha;
  int bidirectional;
  int fast, nr;                 // fast epilogue (host-checked) and n_rnd * 2^p
  int exp_flags;                // ablation experiments (tune "exp"): 1 no epilogue math, 2 no MMA,
                                // 4 no operand TMA (MMAs on stale stages), 8 no J'
                                // loads, 16 no spin loads (single CTAs only)
  double hi_clamp, lo_clamp;    // i0 - alpha, -i0 (formed on the host)
  long c_first, c_last;  // cycles handled: scans/updates for c in [c_first, c_last]
  long sc;               // update iff c < sc
  int run_mode;          // 1: scans + results; 0: plain sweeps (per-step API);
                         // 2: one pass over a row shard (energy partials -> gE, no scan)
  int shard_rt0, shard_nrt;  // run_mode 2: the shard's row tiles
  int multi;                 // multi-instance problem: tile t = trial t = instance t
  const double* offsets;     // multi: per-instance offsets
  int has_target, stop_at_target, record_trace;
  double target_tol;
  int ring_cur;
  int ring_phys[kMaxDelay + 1];
  int stages, nslot;
  int pair;  // FP4 pair operands (Quantized::fp4x2_ok): J' = A1 + A2, spins in SWIZZLE_64B stages
  int i16;   // int16 couplings (Quantized::i16): J' = 256 Ahi + Alo, int8 MMAs into two accumulators
  // Table epilogue (fast mode, tab_w > 0; see TabConsts): integer fields
  // X >= tab_hi / X < tab_lo1 clamp without FP64, the others read
  // fl(fl(X 2^-p + jperp u) [+ jperp d]) from a per-cycle smem table of tab_w
  // entries per neighbour-sign combination
  int tab_lo1, tab_hi, tab_w;
  // Shard passes with the exchange fused in (run_mode 2, npeer > 0; FP4 table
  // epilogue): every spin word also goes to each peer GPU's FP4 slot at the
  // same offset (peer_delta[d] = peer slot base - own slot base, bytes, over
  // NVLink), and the last CTA of the pass pushes the energy partials to
  // peer_E[d] and raises *peer_flag[d] = epoch (system-scope release).
  int npeer;
  long long peer_delta[8];
  unsigned long long* peer_E[8];
  unsigned* peer_flag[8];
  unsigned epoch;
  unsigned* push_ctr;
  int use_tab;  // fast mode: table epilogue (row splits) instead of update_fast2
  int rails_lo; // the clamp rails i0 - alpha and -i0 share their low word (every cycle)
  long long* dbg;  // optional timeline (block 0): [role][rt_global][2] clock64 stamps
  int dbg_rts;     // capacity in row tiles
  int dbg_skip;    // first row tile recorded (tune key "tskip")
  // per-trial results
  double* best_e;
  int* best_k;
  int* reached;
  long* first_hit;
  long* cycles_used;
  int* active;
  int8_t* best_state;
  uint8_t* best_packed;  // [T][npad] bytes: best spin column in slot format
  double* trace;
  // row split (g.rs > 1): see ssqa_batch_s::d_split
  unsigned long long* gE;  // [2][ccols]
  int* g_rows;             // [ntiles][npad/128] pass stamp s+1: rows of pass s written
  unsigned* g_arrive;      // [ntiles] CTAs of the column tile done with their pass
  long long* g_scan;       // [ntiles] (s+1) | stop << 62 once pass s is scanned
};

// Shared bytes of the per-cycle table: TAB (use_tab 1) [combo][tab_w],
// clamped table (use_tab 2) [tab_w + 2][combo].
__host__ __device__ inline int tab_bytes_of(const TcParams& P) {
  const int ncmb = P.bidirectional ? 4 : 2;
  return P.use_tab == 1 ? ncmb * P.tab_w * 8 : (P.use_tab == 2 ? ncmb * (P.tab_w + 2) * 8 : 0);
}

// Bytes per column of one delayed-neighbour tile buffer: the TMA-loaded spin
// rows (int8 128, FP4 64) or, for the clamped-table epilogue, the
// neighbour-sign bytes (128 per plane, a second plane when bidirectional).
__host__ __device__ inline int sig_tile_row(const TcParams& P, bool f4) {
  // (plus half a TMA tile per buffer: one staging tile for the copier warp)
  if (P.fast && P.g.rs == 1 && !P.i16 && ((P.use_tab == 0 && P.rails_lo) || P.use_tab == 2))
    return 128 * (P.bidirectional ? 2 : 1) + (f4 ? 32 : 64);
  return f4 ? 64 : 128;
}

// gpu-scope release/acquire helpers for the row-split protocol
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ long long ld_acquire_gpu(const long long* p) {
  long long v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu(long long* p, long long v) {
  asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try(uint32_t a, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(a), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ bool mbar_try_sleep(uint32_t a, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(a), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}

// Watchdog record in mapped host memory (set by tc_watchdog_init): a wait
// that makes no progress for ~20 s writes who is stuck and traps instead of
// hanging the device; the host prints the record when the launch fails.
// No printf: a vprintf call in the kernel makes ptxas budget every role at
// the smallest setmaxnreg count; a plain out-of-line function (the cold
// path) keeps the per-role budgets and the hot loops short.
struct WatchdogRec {
  int fired, block, warp, lane;
  unsigned addr, parity;
};
__device__ WatchdogRec* g_watchdog = nullptr;

__device__ __noinline__ void watchdog_fire(uint32_t a, uint32_t parity) {
  WatchdogRec* w = g_watchdog;
  if (w && atomicCAS(&w->fired, 0, 1) == 0) {
    volatile WatchdogRec* v = w;
    v->block = blockIdx.x;
    v->warp = threadIdx.x >> 5;
    v->lane = threadIdx.x & 31;
    v->addr = a;
    v->parity = parity;
    __threadfence_system();
  }
  __trap();
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try(a, parity)) return;
  // sleep in try_wait (suspend hint 1 ms)
  const long long t0 = clock64();
  while (!mbar_try_sleep(a, parity))
    if (clock64() - t0 > 20000000000ll) watchdog_fire(a, parity);
}

// Waits of the control warps (MMA issuer, producers, loaders) that are
// expected to be long: poll with a plain try_wait and back off with
// nanosleep, so a waiting control warp does not take issue slots from the
// epilogue warps of its scheduler (a suspend-hinted try_wait wakes on every
// barrier event of the CTA and re-runs the poll loop).
__device__ __forceinline__ void mbar_wait_lazy(uint64_t* bar, uint32_t parity, uint32_t ns) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try(a, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try(a, parity)) {
    __nanosleep(ns);
    if (clock64() - t0 > 20000000000ll) watchdog_fire(a, parity);
  }
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

// Same with an L2 cache-policy hint (createpolicy descriptor).
__device__ __forceinline__ void tma_load_2d_hint(const CUtensorMap* map, uint64_t* bar, void* dst,
                                                 int x, int y, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "l"(policy)
      : "memory");
}

// 3D tile load (accumulator chunks: {rows 0..31, columns, 32-row blocks}).
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// K-major, SWIZZLE_128B UMMA shared-memory descriptor (sm100 layout:
// start>>4 [0,14), LBO>>4 [16,30) (=1, unused for swizzled K-major),
// SBO>>4 [32,46) (=1024 B between 8-row groups), version 1 [46,48),
// layout type 2 = SWIZZLE_128B [61,64)).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}

// K-major, SWIZZLE_64B descriptor (FP4 pair spin stages: 64-byte rows, 8-row
// atoms of 512 B; layout type 4).
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;
  d |= uint64_t(512 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(4) << 61;
  return d;
}

// Instruction descriptor, kind::i8: D = s32 (c_format 2), A = B = signed
// int8 (format 1), both K-major, N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) |
         (uint32_t(M >> 4) << 24);
}


// kind::mxf4 block-scaled MMA (A, B e2m1 packed, ue8m0 scales in TMEM).
__host__ __device__ constexpr uint32_t idesc_mxf4(int M, int N) {
  return (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (1u << 23) |
         (uint32_t(M >> 4) << 24);
}


__device__ __forceinline__ void tmem_st16_const(uint32_t taddr, uint32_t v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
      "%1};" ::"r"(taddr),
      "r"(v));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}


// ---- MMA issue from a whole, converged warp: one lane is elected inside the
// asm, so every operand stays warp-uniform (uniform registers, no per-MMA
// R2UR / elect loop around a single-lane branch).  Measured on B200
// (scripts/mma_peak.cu): a single-lane issuer sustains ~66 % (N = 224) /
// ~43 % (N = 144) of the kind::mxf4 rate behind per-stage mbarriers, the
// warp-wide issuer 100 % / 95 %.
// CTA pairs (cta_group::2): two CTAs of a cluster run M = 256 MMAs, each
// holding its own 128 J' rows and half of the spin columns; the leader (rank
// 0) issues the MMAs, whose commits arrive on both CTAs' barriers.
template <bool CTA2>
__device__ __forceinline__ void mma_i8_w(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                         uint32_t idesc, uint32_t accumulate) {
  if (CTA2)
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
  else
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

template <bool CTA2>
__device__ __forceinline__ void mma_mxf4_w(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate, uint32_t sf_tmem) {
  if (CTA2)
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], "
        "[%5], p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(sf_tmem));
  else
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], "
        "[%5], p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(sf_tmem));
}

// Commit (from the whole warp, one elected lane); with CTA pairs the arrive
// lands on the barrier at the same smem offset in both CTAs.
template <bool CTA2>
__device__ __forceinline__ void mma_commit_w(uint64_t* bar) {
  if (CTA2)
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
        "h"(uint16_t(3))
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
            smem_u32(bar))
        : "memory");
}

// J' tile multicast to the CTAs of `mask` (same smem offset and barrier in each)
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// shared::cluster address of the same smem location in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}

// TMA tile load into this CTA's smem whose completion (complete_tx) is
// counted on the pair leader's barrier (cluster address).
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, uint32_t bar_cluster,
                                                 void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair_hint(const CUtensorMap* map, uint32_t bar_cluster,
                                                      void* dst, int x, int y, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(x), "r"(y), "l"(policy)
      : "memory");
}


__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int32_t (&v)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

template <int EPI>
__device__ __forceinline__ void epi_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(EPI * 32) : "memory");
}

// Spin-slot ring (same rule as the host's pick_free in capi.cu).
__host__ __device__ inline int ring_free(int cur, const int* phys, int d, int nslots) {
  for (int s = 0; s < nslots; ++s) {
    if (s == cur) continue;
    bool used = false;
    for (int q = 0; q <= d; ++q) used |= (phys[q] == s);
    if (!used) return s;
  }
  return -1;
}

// ------------------------------------------------------------- shared state
// Per-column tables in smem, NT entries each:
//   c_col  what the epilogue reads per update, one 16-byte load (ColTab)
//   c_key  CounterRng(seed_t, kStreamSweepNoise).key()
//   c_kt   replica k | (trial-in-tile << 16);  c_flag bit0 live
//   c_E    integer energy partials per TMEM lane quarter [4][NT]
struct __align__(16) ColTab {
  uint64_t base;  // key + spin_counter(cycle, k, 0) * golden + golden (mix64's first add)
  uint32_t off;   // column * npad: element offset of the column inside a spin slot
  uint32_t nbr;   // up | dn << 16: delayed Trotter neighbours k+1, k-1 (mod R) as byte
                  // offsets into the delayed-spin tile; bit 31 = update this column
};
constexpr int kColBytes = 16 + 8 + 4 * 2;

// warp sum without the compiler's divergence-check wrapper (all lanes converge)
__device__ __forceinline__ int redux_add(int v) {
  int r;
  asm volatile("redux.sync.add.s32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
  return r;
}
__device__ __forceinline__ void red_add_u32_if(uint32_t* p, uint32_t v, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
      "@q red.shared.add.u32 [%0], %1;\n\t}" ::"r"(smem_u32(p)),
      "r"(v), "r"(int(pred)));
}
__device__ __forceinline__ uint32_t ld_u8(const uint8_t* p) {
  uint32_t v;
  asm volatile("ld.global.u8 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_u8_if(uint8_t* p, uint32_t v, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
      "@q st.global.u8 [%0], %1;\n\t}" ::"l"(p),
      "r"(v), "r"(int(pred)));
}
__device__ __forceinline__ int ld_s8(const int8_t* p) {
  int v;
  asm volatile("ld.global.s8 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_f64_stream(const double* p) {
  double v;
  asm volatile("ld.global.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_f64_stream(double* p, double v) {
  asm volatile("st.global.L1::no_allocate.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void st_f64_if(double* p, double v, bool pred, uint64_t pol) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
      "@q st.global.L1::no_allocate.L2::cache_hint.f64 [%0], %1, %3;\n\t}" ::"l"(p),
      "d"(v), "r"(int(pred)), "l"(pol));
}
// The global stores / shared reductions of the epilogue carry no "memory"
// clobber: nothing in the thread reads those addresses back, and the
// ordering that matters -- proxy fences, mbarrier arrives, named barriers --
// is between volatile asm statements, which keep their relative order.  A
// clobber would stop the compiler from hoisting the next element's shared
// loads above each store (C3: the spin-word and accumulator stores cost ~30 %).

// Ballot of a register != 0 in plain PTX: no divergence check, and the
// predicate never has to survive to a deferred VOTE.
__device__ __forceinline__ uint32_t ballot_nz(uint32_t v) {
  uint32_t r;
  asm(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t"
      "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\t}"
      : "=r"(r)
      : "r"(v));
  return r;
}
// Warp collectives in plain PTX (no compiler divergence checks / predicate
// juggling around them; the epilogue's warps are always converged here).
#ifndef SSQA_PTX_COLL
#define SSQA_PTX_COLL 1  // bit 0: PTX ballot (C3: -2.6 %/sweep), bit 1: PTX shuffles
#endif
__device__ __forceinline__ int shfl_xor_i(int v, int m) {
#if SSQA_PTX_COLL & 2
  int r;
  asm volatile("shfl.sync.bfly.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=r"(r) : "r"(v), "r"(m));
  return r;
#else
  return __shfl_xor_sync(0xffffffffu, v, m);
#endif
}
__device__ __forceinline__ uint32_t ballot_neg(uint32_t neg) {
#if SSQA_PTX_COLL & 1
  return ballot_nz(neg);
#else
  return __ballot_sync(0xffffffffu, neg != 0u);
#endif
}
__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 v;
  asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ void st_u32_if(uint32_t* p, uint32_t v, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
      "@q st.global.u32 [%0], %1;\n\t}" ::"l"(p),
      "r"(v), "r"(int(pred)));
}
__device__ __forceinline__ void st_s8_if(int8_t* p, int v, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
      "@q st.global.s8 [%0], %1;\n\t}" ::"l"(p),
      "r"(v), "r"(int(pred)));
}

__device__ __forceinline__ int lds_s8(uint32_t a) {
  int v;
  asm volatile("ld.shared.s8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}

struct TrialTab {
  double best_e;
  long first_hit, cycles_used;
  int best_k, reached, active, improved;
};

struct SmemCtl {
  uint64_t full[8];    // operand stages: TMA -> MMA
  uint64_t empty[8];   // operand stages: MMA -> TMA
  uint64_t tfull[2];   // accumulator: MMA -> epilogue
  uint64_t tempty[2];  // accumulator: epilogue -> MMA
  uint64_t afull[16];  // accumulator-state chunks: loader -> epilogue
  uint64_t aempty[16]; // accumulator-state chunks: epilogue -> loader
  uint64_t sfull[2];   // delayed-spin tile: loader -> epilogue
  uint64_t sempty[2];  // delayed-spin tile: epilogue -> loader
  // "rows ready": the epilogue has written (and proxy-fenced) spin rows and
  // accumulators of row-tile group b in the current pass; the producer, MMA
  // issuer and state loader of the next pass wait on it (one phase per pass).
  uint64_t rready[kMaxRowGroups];
  uint64_t done;       // epilogue finished (TMEM may be released)
  uint64_t stg;        // clamped-table path: staged delayed spin rows (TMA -> copier)
  int8_t nz_lut[32];   // integer noise per top-five-bit draw (noise_lut)
  uint8_t umask[kMaxCols / kCW];  // per chunk: bit j = column 8 ch + j updates this cycle
  uint32_t tmem_base;
  long last_pass;  // last cycle any role may start (stop-at-target drain)
  int scan_me;     // row split: this CTA scans the pass (last arrival)
  int scan_stop;   // row split: the column tile's trials have all stopped
  // slot ring per role (producer, loader, epilogue, neighbour-tile copier):
  // [0] = cur, [1 + q] = phys[q]
  int ring[4][kMaxDelay + 2];
};

__device__ __forceinline__ void ring_advance(int* r, long c, int d, int nslots) {
  const int dst = ring_free(r[0], r + 1, d, nslots);
  r[1 + int(c % (d + 1))] = dst;
  r[0] = dst;
}

struct Layout {
  int stages, nslot;
  uint32_t a_bytes, b_bytes, acc_off, sig_off, ctl_off, tab_off, ytab_off, total;
};

// b_row: operand bytes per spin column and stage (kBK; 64 for FP4 pairs);
// b_cols: spin columns per operand stage (NT; NT/2 for CTA pairs).
__host__ __device__ inline Layout make_layout(int NT, int tpt, int stages, int nslot,
                                              int tile_row = kBM, int b_row = kBK,
                                              int b_cols = -1, int tab_bytes = 0) {
  Layout L;
  L.stages = stages;
  L.nslot = nslot;
  L.a_bytes = kBM * kBK;
  L.b_bytes = uint32_t(b_cols < 0 ? NT : b_cols) * uint32_t(b_row);
  uint32_t o = uint32_t(stages) * (L.a_bytes + L.b_bytes);
  L.acc_off = o;
  o += uint32_t(nslot) * kCW * kBM * 8;
  L.sig_off = o;
  o += 2u * uint32_t(NT) * uint32_t(tile_row);
  L.ctl_off = o;
  o += uint32_t((sizeof(SmemCtl) + 127) / 128 * 128);
  L.tab_off = o;
  o += uint32_t(NT) * (kColBytes + 8 * 4) + 8 + uint32_t(tpt) * uint32_t(sizeof(TrialTab));
  o = (o + 15u) & ~15u;
  L.ytab_off = o;
  o += uint32_t(tab_bytes);
  L.total = o + 1024;  // alignment slack
  return L;
}

// Per-thread row context for one row tile of the epilogue.
struct EpiRow {
  uint64_t acc_i;           // &acc[i] (+ column offset * 8)
  uint64_t dst_i, cur_i;    // int8 slots: &sigma[i]; FP4 slots: &sigma4[i/2] (+ offset/2)
  const uint8_t* st_i;      // delayed-spin tile, row il (FP4: byte il/2)
  int h1, h2;
  uint32_t nib_shift;       // FP4: 4 * (i & 1)
  uint64_t iG;              // i * golden
  uint32_t iG_lo, iG_hi;    // the same, pinned in registers (opaque to rematerialisation)
  uint64_t pol_stream;      // L2 evict_first policy for the accumulator stream
  bool w_row;               // spin row exists (i < n)
  uint8_t* dst_w;           // FP4 word stores: byte of rows (warp row 0) + 8*(lane&3)
  uint32_t nib_live;        // FP4 word stores: nibble mask of the live rows of that word
  int npeer;                // fused shard exchange: peers that get every spin word too
  const long long* peer_delta;  // TcParams::peer_delta
  uint32_t hi_off;          // int16 couplings: TMEM column offset of D_hi (0: none)
  // issue-lean FP64 epilogue (noise_top5 / noise_lut / update_fast3)
  uint32_t i_u32;           // global spin row i
  uint32_t p4, p32;         // 4 and 32 in registers (noise_top5)
  uint32_t h1x;             // h1 + noise-free bias + 2^31 (update_fast3)
  const int8_t* nz_lut;     // SmemCtl::nz_lut
};

// Table epilogue constants for one cycle.  With X = S + H' + noise * NR the
// integer field, the reference's update is y = fl(fl(X 2^-p + jperp u)
// [+ jperp d]), s = fl(acc + y), then the clamp.  For X >= hi the sum s is
// at least i0 whatever acc and the neighbours are (host bound, 1 of margin
// over every rounding), for X < lo1 it is below -i0: no FP64 at all.  In
// between y comes from ytab[combo * w + X - lo1] (combo: bit 0 = sigma_up
// negative, bit 1 = sigma_dn negative), built per cycle with the reference's
// own operations, and the only FP64 instruction left is s = acc + y; the
// clamp compares the bit patterns (i0 > 0 > -i0, no NaN, no -0.0).  The
// FP64 units share the tensor core's issue path on B200: while MMAs run an
// FP64 add costs ~10x (scripts/dadd_probe.cu).
struct TabConsts {
  int lo1, hi, w;
  long long i0_bits;          // s >= i0   <=>  (int64) bits(s) >= i0_bits
  unsigned long long lo_bits; // s < -i0   <=>  (uint64) bits(s) > lo_bits
  long long hic_bits;         // bits(i0 - alpha), bits(-i0)
  long long loc_bits;
  const double* ytab;
};

// a + (hi:lo) as one add / add-with-carry pair
__device__ __forceinline__ uint64_t add64_pair(uint64_t a, uint32_t lo, uint32_t hi) {
  uint64_t r;
  asm("{\n\t.reg .u32 l, h;\n\tmov.b64 {l, h}, %1;\n\tadd.cc.u32 l, l, %2;\n\t"
      "addc.u32 h, h, %3;\n\tmov.b64 %0, {l, h};\n\t}"
      : "=l"(r)
      : "l"(a), "r"(lo), "r"(hi));
  return r;
}

// Spread the 8 bits of b to bit 4k+3 of a word of e2m1 +-1 nibbles (0x2 / 0xA).
__device__ __forceinline__ uint32_t nibbles_pm1(uint32_t b) {
  uint32_t x = (b | (b << 12)) & 0x000F000Fu;
  x = (x | (x << 6)) & 0x03030303u;
  x = (x | (x << 3)) & 0x11111111u;
  return (x << 3) | 0x22222222u;
}

// All of this warp's kCW-column chunks of one row tile: TMEM fields,
// staged accumulators, delayed neighbours -> exact update, predicated
// stores, per-column warp energy sums.  Template switches are hoisted out of
// the column loop:
//   BIDIR   couple to k-1 as well as k+1
//   SIGACC  sigma(c) = sign(acc(c)) instead of a load (all but the first sweep)
//   FAST    host-checked table epilogue (TabConsts), int32 energy partials
//   F4      FP4 operands: fp32 fields in TMEM, spins stored as e2m1 nibbles
template <bool BIDIR, bool SIGACC, bool FAST, bool F4, bool TAB>
__device__ __forceinline__ void epi_chunks(const EpiRow& er, const UpdateConsts& uc,
                                           const FastConsts& fc, const TabConsts& tc,
                                           const I2D& i2d, SmemCtl* ctl,
                                           double* acc_ring, const ColTab* c_col,
                                           long long* q_sum, uint32_t trow, int sub,
                                           int nsubs, int nchunk, int nps, uint32_t cnt0, int il,
                                           int lane) {
  // this subgroup's ring position: slot sub*nps + cnt % nps, parity (cnt / nps) & 1
  int sidx = int(cnt0 % uint32_t(nps));
  uint32_t ph = (cnt0 / uint32_t(nps)) & 1;
  // FP4 spin words: lane L writes 8 rows of column L >> 2
  constexpr bool kWordSt = F4 && FAST;
  const int wj = lane >> 2;
  for (int ch = sub; ch < nchunk; ch += nsubs) {
    const int cb = ch * kCW;
    const int slot = sub * nps + sidx;
    int32_t v[kCW];
    if (SSQA_ABL & 256) {
#pragma unroll
      for (int j = 0; j < kCW; ++j) v[j] = int(trow) + cb + j;
    } else {
      tmem_ld8(trow + uint32_t(cb), v);
      if (er.hi_off) {
        // int16 couplings: S = D_lo + 256 D_hi
        int32_t vh[kCW];
        tmem_ld8(trow + er.hi_off + uint32_t(cb), vh);
#pragma unroll
        for (int j = 0; j < kCW; ++j) v[j] += vh[j] * 256;
      }
    }
    if (!(SSQA_ABL & 128)) mbar_wait(&ctl->afull[slot], ph);
    if (++sidx == nps) {
      sidx = 0;
      ph ^= 1;
    }
    // slot layout [column][128 rows] (2D accumulator map)
    double* ab = acc_ring + size_t(slot) * kCW * kBM + il;
    int ep[kCW];
    uint32_t ball[kCW];
    if (FAST && TAB) {
      // table epilogue (TabConsts); pass 1: integer fields, energies, table positions
      int X[kCW];
      double ao[kCW];
      uint32_t cmb = 0, midm = 0;
#pragma unroll
      for (int j = 0; j < kCW; ++j) {
        const uint4 ct = lds128(c_col + cb + j);
        const uint64_t cbase = (uint64_t(ct.y) << 32) | ct.x;
        const double a_old = ab[j * kBM];
        ao[j] = a_old;
        const int S = F4 ? __float_as_int(__int_as_float(v[j]) + 12582912.0f) : v[j];
        const int s2 = S + er.h2;
        if (SIGACC) {
          // sign of a finite, never -0.0 accumulator: s2 * (+-1) on the FMA pipe
          ep[j] = s2 * ((__double2hiint(a_old) >> 30) | 1);
        } else {
          int sg;
          if (F4) {
            const uint32_t bc = ld_u8(reinterpret_cast<const uint8_t*>(er.cur_i + (ct.z >> 1)));
            sg = ((bc >> er.nib_shift) & 8u) ? -1 : 1;
          } else {
            sg = ld_s8(reinterpret_cast<const int8_t*>(er.cur_i + ct.z));
          }
          ep[j] = sg * s2;
        }
        uint32_t neg_up, neg_dn = 0;
        if (F4) {
          neg_up = (uint32_t(er.st_i[ct.w & 0xffffu]) >> er.nib_shift) >> 3 & 1u;
          if (BIDIR) neg_dn = (uint32_t(er.st_i[(ct.w >> 16) & 0x7fffu]) >> er.nib_shift) >> 3 & 1u;
        } else {
          neg_up = uint32_t(int8_t(er.st_i[ct.w & 0xffffu])) >> 31;
          if (BIDIR) neg_dn = uint32_t(int8_t(er.st_i[(ct.w >> 16) & 0x7fffu])) >> 31;
        }
        const uint32_t top = (SSQA_ABL & 512) ? uint32_t(cbase) ^ er.iG_lo
                                              : mix64_top32_pre(add64_pair(cbase, er.iG_lo, er.iG_hi));
        const int nzi = top < 0x70000000u ? 0 : (top < 0xB8000000u ? -fc.nr : fc.nr);
        X[j] = S + er.h1 + nzi;
        cmb |= (neg_up | (neg_dn << 1)) << (2 * j);
        midm |= uint32_t(unsigned(X[j] - tc.lo1) < unsigned(tc.w)) << j;
      }
      // pass 2: new accumulators; the table path only where a lane needs it
      const bool any_mid = ballot_nz(midm) != 0u;
#pragma unroll
      for (int j = 0; j < kCW; ++j) {
        const uint2 cw = *reinterpret_cast<const uint2*>(&c_col[cb + j].off);
        const bool pos = X[j] >= tc.hi;
        long long res = pos ? tc.hic_bits : tc.loc_bits;
        if (any_mid) {
          const bool mid = (midm >> j) & 1u;
          const int e = int((cmb >> (2 * j)) & 3u) * tc.w + (mid ? X[j] - tc.lo1 : 0);
          const double sd = __dadd_rn(ao[j], tc.ytab[e]);
          const long long sb = __double_as_longlong(sd);
          const bool ge = sb >= tc.i0_bits;
          const bool lt = static_cast<unsigned long long>(sb) > tc.lo_bits;
          const long long r2 = ge ? tc.hic_bits : (lt ? tc.loc_bits : sb);
          res = mid ? r2 : res;
        }
        const uint32_t neg = uint32_t(static_cast<unsigned long long>(res) >> 63);
        const bool w = (cw.y & 0x80000000u) && er.w_row;
        if (!(SSQA_ABL & 64))
          st_f64_if(reinterpret_cast<double*>(er.acc_i + uint64_t(cw.x) * 8u),
                    __longlong_as_double(res), w, er.pol_stream);
        if (SSQA_ABL & 32) {
        } else if (kWordSt) {
          ball[j] = (SSQA_ABL & 2048) ? neg : ballot_neg(neg);
        } else if (F4) {
          const uint32_t nib = 2u | (neg << 3);
          const uint32_t hi = __shfl_xor_sync(0xffffffffu, nib, 1);
          st_u8_if(reinterpret_cast<uint8_t*>(er.dst_i + (cw.x >> 1)), nib | (hi << 4),
                   w && !(lane & 1));
        } else {
          st_s8_if(reinterpret_cast<int8_t*>(er.dst_i + uint64_t(cw.x)), int(1 - 2 * int(neg)), w);
        }
      }
    } else if (FAST) {
      // FP64 epilogue (update_fast2): fewer instructions than the table path,
      // best where the MMAs leave the FP64 units mostly free (no row split)
#pragma unroll
      for (int j = 0; j < kCW; ++j) {
        const uint4 ct = lds128(c_col + cb + j);
        const uint64_t cbase = (uint64_t(ct.y) << 32) | ct.x;
        const uint32_t coff = ct.z;
        const uint32_t nb = ct.w;
        const double a_old = ab[j * kBM];
        const int S = F4 ? __float_as_int(__int_as_float(v[j]) + 12582912.0f) : v[j];
        const int s2 = S + er.h2;
        if (SIGACC) {
          ep[j] = s2 * ((__double2hiint(a_old) >> 30) | 1);
        } else {
          int sg;
          if (F4) {
            const uint32_t bc = ld_u8(reinterpret_cast<const uint8_t*>(er.cur_i + (coff >> 1)));
            sg = ((bc >> er.nib_shift) & 8u) ? -1 : 1;
          } else {
            sg = ld_s8(reinterpret_cast<const int8_t*>(er.cur_i + coff));
          }
          ep[j] = sg * s2;
        }
        int up, dn = 0;
        if (F4) {
          // update_fast2 only reads the sign bit: move the nibble's bit 3 there
          up = int(uint32_t(er.st_i[nb & 0xffffu]) << (28u - er.nib_shift));
          if (BIDIR) dn = int(uint32_t(er.st_i[(nb >> 16) & 0x7fffu]) << (28u - er.nib_shift));
        } else {
          up = int8_t(er.st_i[nb & 0xffffu]);
          if (BIDIR) dn = int8_t(er.st_i[(nb >> 16) & 0x7fffu]);
        }
#if SSQA_EPI_V
        const uint32_t t5 = noise_top5(cbase, er.i_u32, er.p4, er.p32);
        const double nv = update_fast3<BIDIR>(fc, i2d, uint32_t(S) + er.h1x +
                                                           uint32_t(noise_lut(er.nz_lut, t5)),
                                              up, dn, a_old);
#else
        const uint32_t top = (SSQA_ABL & 512) ? uint32_t(cbase) ^ er.iG_lo
                                              : mix64_top32_pre(add64_pair(cbase, er.iG_lo, er.iG_hi));
        const double nv = update_fast2<BIDIR>(fc, i2d, S + er.h1, top, up, dn, a_old);
#endif
        const uint32_t neg = uint32_t(__double2hiint(nv)) >> 31;
        const bool w = (nb & 0x80000000u) && er.w_row;
        if (!(SSQA_ABL & 64))
          st_f64_if(reinterpret_cast<double*>(er.acc_i + uint64_t(coff) * 8u), nv, w, er.pol_stream);
        if (SSQA_ABL & 32) {
        } else if (kWordSt) {
          ball[j] = (SSQA_ABL & 2048) ? neg : ballot_neg(neg);
        } else if (F4) {
          const uint32_t nib = 2u | (neg << 3);
          const uint32_t hi = __shfl_xor_sync(0xffffffffu, nib, 1);
          st_u8_if(reinterpret_cast<uint8_t*>(er.dst_i + (coff >> 1)), nib | (hi << 4),
                   w && !(lane & 1));
        } else {
          st_s8_if(reinterpret_cast<int8_t*>(er.dst_i + uint64_t(coff)), int(1 - 2 * int(neg)), w);
        }
      }
    } else {
      // exact path for any finite or non-finite double (hand-written lattices)
#pragma unroll
      for (int j = 0; j < kCW; ++j) {
        const int cl = cb + j;
        const uint4 ct = lds128(c_col + cl);
        const uint64_t cbase = (uint64_t(ct.y) << 32) | ct.x;
        const uint32_t coff = ct.z;
        const uint32_t nb = ct.w;
        const double a_old = ab[j * kBM];
        // FP4: the fp32 accumulator holds a small exact integer (|S| < 2^22);
        // its bits after adding 1.5*2^23 are 0x4B400000 + S, and the bias is
        // folded into the per-row constants h1/h2 (EpiRow).
        const int S = F4 ? __float_as_int(__int_as_float(v[j]) + 12582912.0f) : v[j];
        const int s2 = S + er.h2;
        int sg;
        if (SIGACC) {
          sg = a_old >= 0.0 ? 1 : -1;
        } else if (F4) {
          const uint32_t bc = ld_u8(reinterpret_cast<const uint8_t*>(er.cur_i + (coff >> 1)));
          sg = ((bc >> er.nib_shift) & 8u) ? -1 : 1;
        } else {
          sg = ld_s8(reinterpret_cast<const int8_t*>(er.cur_i + coff));
        }
        // energy partials of every column, padding included: the scan reads
        // only live columns, and padded rows contribute 0 (J', H' rows are zero)
        ep[j] = sg * s2;
        int up, dn = 0;
        if (F4) {
          const uint32_t bu = er.st_i[nb & 0xffffu];
          up = ((bu >> er.nib_shift) & 8u) ? -1 : 1;
          if (BIDIR) dn = ((uint32_t(er.st_i[(nb >> 16) & 0x7fffu]) >> er.nib_shift) & 8u) ? -1 : 1;
        } else {
          up = int8_t(er.st_i[nb & 0xffffu]);
          if (BIDIR) dn = int8_t(er.st_i[(nb >> 16) & 0x7fffu]);
        }
        const double field = scaled_i32(S + er.h1, i2d);
        const uint32_t t5 = mix64_top5_pre(cbase + er.iG);
        const double nv = update_fast(uc, field, t5, up, dn, BIDIR, a_old);
        const uint32_t neg = nv >= 0.0 ? 0u : 1u;
        const bool w = (nb & 0x80000000u) && er.w_row;
        if (!(SSQA_ABL & 64))
          st_f64_if(reinterpret_cast<double*>(er.acc_i + uint64_t(coff) * 8u), nv, w, er.pol_stream);
        if (SSQA_ABL & 32) {
        } else if (F4) {
          // e2m1 +1 = 0x2, -1 = 0xA; even lanes store the byte of rows (i, i+1)
          const uint32_t nib = 2u | (neg << 3);
          const uint32_t hi = __shfl_xor_sync(0xffffffffu, nib, 1);
          st_u8_if(reinterpret_cast<uint8_t*>(er.dst_i + (coff >> 1)), nib | (hi << 4),
                   w && !(lane & 1));
        } else {
          st_s8_if(reinterpret_cast<int8_t*>(er.dst_i + uint64_t(coff)), int(1 - 2 * int(neg)), w);
        }
      }
    }
    if (kWordSt && !(SSQA_ABL & 32)) {
      // ball[j] bit r = sign of row r of column cb+j; lane L stores the e2m1
      // nibbles of rows 8*(L&3) .. +7 of column cb + (L>>2) as one 32-bit word
      const uint32_t a0 = (wj & 1) ? ball[1] : ball[0], a1 = (wj & 1) ? ball[3] : ball[2];
      const uint32_t a2 = (wj & 1) ? ball[5] : ball[4], a3 = (wj & 1) ? ball[7] : ball[6];
      const uint32_t b0 = (wj & 2) ? a1 : a0, b1 = (wj & 2) ? a3 : a2;
      const uint32_t mm = (wj & 4) ? b1 : b0;
      const uint32_t word = nibbles_pm1((mm >> (8 * (lane & 3))) & 0xffu) & er.nib_live;
      const uint2 cw = *reinterpret_cast<const uint2*>(&c_col[cb + wj].off);
      if (SSQA_ABL & 1024) {
      } else {
        st_u32_if(reinterpret_cast<uint32_t*>(er.dst_w + (cw.x >> 1)), word,
                  (cw.y & 0x80000000u) && er.nib_live);
        if (TAB && er.npeer) {
          // fused shard exchange: the same word into every peer's slot
          for (int d = 0; d < er.npeer; ++d)
            st_u32_if(reinterpret_cast<uint32_t*>(er.dst_w + er.peer_delta[d] + (cw.x >> 1)), word,
                      (cw.y & 0x80000000u) && er.nib_live);
        }
      }
    }
    __syncwarp();
    if (lane == 0 && !(SSQA_ABL & 128)) mbar_arrive(&ctl->aempty[slot]);
    if (SSQA_ABL & 16) {
    } else if (FAST && (SSQA_ENERGY_RED == 1)) {
      // transpose-reduce the 8 column partials across the warp with shuffles:
      // after the five butterfly stages lane L holds the warp sum of column
      // (L >> 2) & 7; lanes with L % 4 == 0 add it to the quarter's partial.
      int a4[4], a2[2], a1;
      const bool b16 = lane & 16, b8 = lane & 8, b4 = lane & 4;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int keep = b16 ? ep[k + 4] : ep[k];
        const int send = b16 ? ep[k] : ep[k + 4];
        a4[k] = keep + shfl_xor_i(send, 16);
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int keep = b8 ? a4[k + 2] : a4[k];
        const int send = b8 ? a4[k] : a4[k + 2];
        a2[k] = keep + shfl_xor_i(send, 8);
      }
      {
        const int keep = b4 ? a2[1] : a2[0];
        const int send = b4 ? a2[0] : a2[1];
        a1 = keep + shfl_xor_i(send, 4);
      }
      a1 += shfl_xor_i(a1, 2);
      a1 += shfl_xor_i(a1, 1);
      // lane bits 4,3,2 select column bits 2,1,0
      const int col = (b16 ? 4 : 0) + (b8 ? 2 : 0) + (b4 ? 1 : 0);
      red_add_u32_if(reinterpret_cast<uint32_t*>(q_sum) + cb + col, uint32_t(a1),
                     (lane & 3) == 0);
    } else {
#pragma unroll
      for (int j = 0; j < kCW; ++j) {
        const int wsum = redux_add(ep[j]);
        if (FAST) {
          red_add_u32_if(reinterpret_cast<uint32_t*>(q_sum) + cb + j, uint32_t(wsum), lane == 0);
        } else {
          if (lane == 0) q_sum[cb + j] += wsum;
        }
      }
    }
  }
}

// Neighbour-sign tiles of the clamped-table path: [column][128 rows] bytes,
// up plane value 8 where sigma_{k+1}(c-d) < 0, then (bidirectional) the down
// plane with value 16 -- the byte offsets of the table entry.
constexpr int kCtTileRow = 128;

__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint64_t lds_u64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void tmem_ld8_nw(uint32_t taddr, int32_t (&v)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const int32_t (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Sum each of the 8 column partials over the warp's 32 rows (shuffle
// transpose-reduce) and add it to the lane quarter's column sums.
__device__ __forceinline__ void reduce8_to_quarter(const int (&ep)[kCW], long long* q_sum, int cb,
                                                   int lane) {
  int a4[4], a2[2], a1;
  const bool b16 = lane & 16, b8 = lane & 8, b4 = lane & 4;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int keep = b16 ? ep[k + 4] : ep[k];
    const int send = b16 ? ep[k] : ep[k + 4];
    a4[k] = keep + shfl_xor_i(send, 16);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int keep = b8 ? a4[k + 2] : a4[k];
    const int send = b8 ? a4[k] : a4[k + 2];
    a2[k] = keep + shfl_xor_i(send, 8);
  }
  {
    const int keep = b4 ? a2[1] : a2[0];
    const int send = b4 ? a2[0] : a2[1];
    a1 = keep + shfl_xor_i(send, 4);
  }
  a1 += shfl_xor_i(a1, 2);
  a1 += shfl_xor_i(a1, 1);
  const int col = (b16 ? 4 : 0) + (b8 ? 2 : 0) + (b4 ? 1 : 0);
  red_add_u32_if(reinterpret_cast<uint32_t*>(q_sum) + cb + col, uint32_t(a1), (lane & 3) == 0);
}

// ---- Issue-lean FP64 epilogue (use_tab 0, no row split) ------------------
// update_fast2's exact arithmetic (magic-number field, the reference's three
// FP64 adds, the clamp) with the ALU work cut down -- the hot loop is bound by
// instruction issue and the ALU pipe:
//  * counter RNG with the 64-bit counter sum pinned, high-word shifts on the
//    FMA pipe, and the noise level from a byte table (noise_lut);
//  * the 2^31 bias of the magic conversion folded into the row constant;
//  * neighbour signs from the copier warp's permuted sign tile: one signed
//    byte load at a fixed offset whose bit 31 is the sign (no address math);
//  * the energy sign from the accumulator's high word on the FMA pipe, the
//    partials kept in TMEM across the row tiles (one warp reduction per pass);
//  * the clamp with three selects (the rails share their low word).
struct V4Row {
  uint32_t iG_lo, iG_hi, p4, p32;
  uint32_t h1x;              // h1 (+ FP4 bias) + 2^31
  int h2;
  uint32_t nbt;              // shared address of row il of sign-tile column 0
  uint32_t lut;
  uint32_t e_tmem;
  int e_mode;                // energy partials in TMEM: 0 reduce every chunk, 1 first row tile
                             // (store), 2 middle (load, add, store), 3 last (load, add, reduce)
  uint64_t acc_col;          // &acc[col0 * npad + i]
  uint32_t col_stride32;     // npad * 8 bytes
  uint8_t* dst_w;
  uint32_t nib_live;
  uint64_t cur_i, dst_i;
  uint32_t nib_shift;
  bool w_row;
  uint32_t jp_hi, jp_lo, hic_hi, loc_hi, rail_lo;
  uint64_t pol;
  int h1c, ct_max;           // TBL: clamped table index = clamp(S + h1c + noise, 0, ct_max)
  uint32_t ytab;
  int exp;                   // timing ablations (TcParams::exp_flags): 64 no accumulator stores
};

template <bool BIDIR, bool SIGACC, bool F4, bool TBL = false>
__device__ __forceinline__ void epi_v4(const V4Row& r, const FastConsts& fc, const I2D& i2d,
                                       SmemCtl* ctl, const double* acc_ring, const ColTab* c_col,
                                       const uint8_t* c_umask, long long* q_sum, uint32_t trow,
                                       int sub, int nsubs, int nchunk, int nps, uint32_t cnt0,
                                       int il, int lane) {
  int sidx = int(cnt0 % uint32_t(nps));
  uint32_t ph = (cnt0 / uint32_t(nps)) & 1;
  const int wj = lane >> 2;
  const uint32_t colt = smem_u32(c_col);
  constexpr uint32_t kRow = BIDIR ? 2u * kCtTileRow : uint32_t(kCtTileRow);
  for (int ch = sub; ch < nchunk; ch += nsubs) {
    const int cb = ch * kCW;
    const int slot = sub * nps + sidx;
    int32_t v[kCW], e[kCW];
    tmem_ld8_nw(trow + uint32_t(cb), v);
    if (r.e_mode >= 2) tmem_ld8_nw(r.e_tmem + uint32_t(cb), e);
    else
#pragma unroll
      for (int j = 0; j < kCW; ++j) e[j] = 0;
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    mbar_wait(&ctl->afull[slot], ph);
    if (++sidx == nps) {
      sidx = 0;
      ph ^= 1;
    }
    const double* ab = acc_ring + size_t(slot) * kCW * kBM + il;
    const uint32_t umask = c_umask[ch];
    const uint32_t nbq = r.nbt + uint32_t(cb) * kRow;
    uint32_t ball[kCW];
#pragma unroll
    for (int j = 0; j < kCW; ++j) {
      const uint64_t cbase = lds_u64(colt + uint32_t(cb + j) * uint32_t(sizeof(ColTab)));
      const double a_old = ab[j * kBM];
      const int S = F4 ? __float_as_int(__int_as_float(v[j]) + 12582912.0f) : v[j];
      const int s2 = S + r.h2;
      if (SIGACC) {
        // sign(acc) = 2 (hi >> 31) + 1, high product on the FMA pipe
        const int t = __mulhi(__double2hiint(a_old), 2);
        e[j] += s2 * (2 * t + 1);
      } else {
        const uint32_t coff = c_col[cb + j].off;
        int sg;
        if (F4) {
          const uint32_t bc = ld_u8(reinterpret_cast<const uint8_t*>(r.cur_i + (coff >> 1)));
          sg = ((bc >> r.nib_shift) & 8u) ? -1 : 1;
        } else {
          sg = ld_s8(reinterpret_cast<const int8_t*>(r.cur_i + coff));
        }
        e[j] += sg * s2;
      }
      const uint32_t up = uint32_t(lds_s8(nbq + uint32_t(j) * kRow));
      const uint32_t t5 = noise_top5_v4(cbase, r.iG_lo, r.iG_hi, r.p4, r.p32);
      double input;
      if (TBL) {
        // y = fl(X 2^-p + jperp u [+ jperp d]) from the per-cycle clamped table
        // (use_tab 2 layout [row][combo], 8-byte entries)
        const int xi = min(max(S + r.h1c + lds_s8(r.lut + t5), 0), r.ct_max);
        uint32_t cmbo = (up >> 28) & 8u;
        if (BIDIR) cmbo |= (uint32_t(lds_s8(nbq + uint32_t(j) * kRow + kCtTileRow)) >> 27) & 16u;
        input = lds_f64(r.ytab + (uint32_t(xi) << (BIDIR ? 5 : 4)) + cmbo);
      } else {
        const uint32_t xb = uint32_t(S) + r.h1x + uint32_t(lds_s8(r.lut + t5));
        input = __dsub_rn(__hiloint2double(int(i2d.magic_hi), int(xb)), i2d.magic);
        input = __dadd_rn(input, __hiloint2double(int(r.jp_hi ^ (up & 0x80000000u)), int(r.jp_lo)));
        if (BIDIR) {
          const uint32_t dn = uint32_t(lds_s8(nbq + uint32_t(j) * kRow + kCtTileRow));
          input = __dadd_rn(input, __hiloint2double(int(r.jp_hi ^ (dn & 0x80000000u)), int(r.jp_lo)));
        }
      }
      const double sd = __dadd_rn(a_old, input);
      const bool p_lo = sd < fc.lo_clamp, p_hi = sd >= fc.i0;
      const int nhi = p_hi ? int(r.hic_hi) : (p_lo ? int(r.loc_hi) : __double2hiint(sd));
      const int nlo = (p_hi || p_lo) ? int(r.rail_lo) : __double2loint(sd);
      const double nv = __hiloint2double(nhi, nlo);
      uint64_t addr;
      asm("mad.wide.u32 %0, %1, %2, %3;"
          : "=l"(addr)
          : "r"(uint32_t(cb + j)), "r"(r.col_stride32), "l"(r.acc_col));
      st_f64_if(reinterpret_cast<double*>(addr), nv, ((umask >> j) & 1u) && !(r.exp & 64), r.pol);
      if (F4) {
        ball[j] = __ballot_sync(0xffffffffu, nhi < 0);
      } else {
        const uint32_t coff = c_col[cb + j].off;
        st_s8_if(reinterpret_cast<int8_t*>(r.dst_i + uint64_t(coff)), nhi < 0 ? -1 : 1,
                 ((umask >> j) & 1u) && r.w_row);
      }
    }
    if (F4) {
      const uint32_t a0 = (wj & 1) ? ball[1] : ball[0], a1 = (wj & 1) ? ball[3] : ball[2];
      const uint32_t a2 = (wj & 1) ? ball[5] : ball[4], a3 = (wj & 1) ? ball[7] : ball[6];
      const uint32_t b0 = (wj & 2) ? a1 : a0, b1 = (wj & 2) ? a3 : a2;
      const uint32_t mm = (wj & 4) ? b1 : b0;
      const uint32_t word = nibbles_pm1((mm >> (8 * (lane & 3))) & 0xffu) & r.nib_live;
      const uint32_t coffw = c_col[cb + wj].off;
      st_u32_if(reinterpret_cast<uint32_t*>(r.dst_w + (coffw >> 1)), word,
                ((umask >> wj) & 1u) && r.nib_live);
    }
    if (r.e_mode == 1 || r.e_mode == 2) tmem_st8(r.e_tmem + uint32_t(cb), e);
    else reduce8_to_quarter(e, q_sum, cb, lane);
    __syncwarp();
    if (lane == 0) mbar_arrive(&ctl->aempty[slot]);
  }
}

// Best-state snapshots during the run copy the packed spin column (npad
// bytes int8, npad/2 bytes FP4; 16-byte aligned) with vector loads/stores;
// expand_best_state turns it into the int8 +-1 best_state once at the end.
template <bool F4>
__device__ __forceinline__ void snap_best_state(const TcParams& P, int cur, size_t colg,
                                                int trial, int npad, int lane) {
  const size_t nb = F4 ? size_t(npad) / 2 : size_t(npad);
  const uint4* src = reinterpret_cast<const uint4*>(P.sig_base + size_t(cur) * (F4 ? P.slot_elems / 2 : P.slot_elems) + colg * nb);
  uint4* dst = reinterpret_cast<uint4*>(P.best_packed + size_t(trial) * npad);
  const int nv = int(nb / 16);
  for (int v0 = 0; v0 < nv; v0 += 128) {
    uint4 r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int v = v0 + u * 32 + lane;
      if (v < nv) r[u] = src[v];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int v = v0 + u * 32 + lane;
      if (v < nv) dst[v] = r[u];
    }
  }
}

template <bool F4>
__device__ __forceinline__ void expand_best_state(const TcParams& P, int trial, int n, int npad,
                                                  int lane) {
  const uint8_t* src = P.best_packed + size_t(trial) * npad;
  int8_t* dst = P.best_state + size_t(trial) * n;
  for (int i = lane; i < n; i += 32) {
    const uint32_t b = src[F4 ? i >> 1 : i];
    dst[i] = F4 ? (((b >> (4 * (i & 1))) & 8u) ? -1 : 1) : int8_t(b);
  }
}

// Debug timeline: role 0 MMA (start, commit), 1 loader (start, all issued),
// 2 epilogue warp 3 (start incl. waits, done), 3 epilogue warp 3 (operands
// ready, -).  Block 0, lane 0 only; no cost when P.dbg is null.
#define DBG_STAMP(role, rtg, which)                                                    \
  do {                                                                                 \
    if (P.dbg && blockIdx.x == 0 && lane == 0 && int(rtg) >= P.dbg_skip &&            \
        int(rtg) - P.dbg_skip < P.dbg_rts)                                             \
      P.dbg[(size_t(role) * P.dbg_rts + ((rtg) - P.dbg_skip)) * 2 + (which)] = clock64(); \
  } while (0)

// Registers per thread after setmaxnreg: control warpgroup / epilogue
// warpgroups.  setmaxnreg moves registers inside the CTA's launch pool, so
// (EPI * kEpi + 4 * kCtl) * 32 must not exceed (EPI + 4) * 32 * launch regs:
// EPI 12 launches at 128 (pool 65536 -> 160), EPI 16 at 96 (pool 61440 -> 112).
constexpr int kCtlRegs = 32;
template <int EPI> struct EpiRegs { static constexpr int value = EPI == 16 ? 112 : 160; };
static_assert((12 * EpiRegs<12>::value + 4 * kCtlRegs) * 32 <= 16 * 32 * 128, "EPI 12 pool");
static_assert((16 * EpiRegs<16>::value + 4 * kCtlRegs) * 32 <= 20 * 32 * 96, "EPI 16 pool");

// Warp roles: 0 .. EPI-1 epilogue (EPI/4 warps per TMEM lane quarter),
// EPI operand TMA producer, EPI+1 TMEM allocator + MMA issuer, EPI+2 state
// loader (TMA of accumulator chunks and delayed-spin tiles).
// CL: cluster mode -- 0 none; 1 CTA pairs (clusters of 2 row parts sharing
// M = 256 MMAs).
template <int EPI, bool F4, int CL>
__global__ void __launch_bounds__(32 * (4 + EPI), 1)
    k_sweep_tc(const __grid_constant__ CUtensorMap tmJ, const __grid_constant__ CUtensorMap tmS,
               const __grid_constant__ CUtensorMap tmSe, const __grid_constant__ CUtensorMap tmA,
               const TcParams P) {
  constexpr bool CTA2 = CL == 1;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-align by offsetting into the shared array itself, so every derived
  // pointer keeps the shared address space (no generic loads)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const Geom& g = P.g;
  const int NT = g.tile_cols;
  constexpr int kTileRow = F4 ? kBM / 2 : kBM;  // bytes per spin-tile row (128 spins)
  // FP4 pairs: a stage is K = 128 couplings -- one 128-byte J'' row holding
  // 64 bytes of A1 and 64 bytes of A2 nibbles -- against 64 bytes of spins
  const bool pair = F4 && P.pair != 0;
  // int16 planes (Quantized::i16): a stage is K = 64 couplings -- one 128-byte
  // row of 64 Alo bytes then 64 Ahi bytes -- against 64 spin bytes; the MMAs of
  // the two planes accumulate into D_lo (columns [buf NT]) and D_hi ([2 NT + buf NT])
  const bool i16 = !F4 && P.i16 != 0;
  const int b_row = (pair || i16) ? kBK / 2 : kBK;
  const Layout L = make_layout(NT, g.tpt, P.stages, P.nslot, sig_tile_row(P, F4), b_row,
                               CTA2 ? NT / 2 : NT, tab_bytes_of(P));
  const int stages = L.stages, nslot = L.nslot;
  uint8_t* sA = smem;
  uint8_t* sB = smem + size_t(stages) * L.a_bytes;
  double* acc_ring = reinterpret_cast<double*>(smem + L.acc_off);  // [nslot][kCW][kBM]
  uint8_t* sig_tiles = smem + L.sig_off;  // [2][NT][kTileRow] delayed-spin tiles
  SmemCtl* ctl = reinterpret_cast<SmemCtl*>(smem + L.ctl_off);
  uint8_t* tabs = smem + L.tab_off;
  ColTab* c_col = reinterpret_cast<ColTab*>(tabs);
  uint64_t* c_key = reinterpret_cast<uint64_t*>(c_col + NT);
  long long* c_E = reinterpret_cast<long long*>(c_key + NT);  // [4][NT]
  int* c_kt = reinterpret_cast<int*>(c_E + 4 * NT);
  int* c_flag = c_kt + NT;
  TrialTab* trials = reinterpret_cast<TrialTab*>(c_flag + NT + (NT & 1));
  double* ytab = reinterpret_cast<double*>(smem + L.ytab_off);  // TabConsts::ytab

  // warp index broadcast from lane 0: provably warp-uniform for ptxas (role
  // branches and setmaxnreg must be warp-uniform)
  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  // The single-lane pipeline roles take the highest warp indices: the warp
  // scheduler favours higher warp ids, so the TMA producer, MMA issuer and
  // state loader are never starved by the EPI busy epilogue warps.
  constexpr int kWarpProducer = EPI, kWarpMma = EPI + 1, kWarpLoader = EPI + 2;
  // CTA = (column tile, row part): with a row split (g.rs > 1) the rs CTAs of
  // a column tile share its columns and own contiguous ranges of row tiles.
  const int RS = g.rs;
  const bool split = RS > 1;
  const int tile = int(blockIdx.x) / RS;
  const int part = int(blockIdx.x) % RS;
  const int col0 = tile * NT;
  const int ntl = max(0, min(g.tpt, g.T - tile * g.tpt));
  const int NRT_all = g.npad / kBM;
  const bool scan_mode = P.run_mode == 1;   // scans, results, row-split protocol
  const bool shard_mode = P.run_mode == 2;  // one pass over the rows of a GPU shard
  const int rt_base = shard_mode ? P.shard_rt0 : 0;
  const int rt_span = shard_mode ? P.shard_nrt : NRT_all;
  // CTA pairs: parts 2p, 2p+1 of a column tile form a cluster (rank = part & 1,
  // the leader is rank 0); pair p owns row tiles [2 u_lo, 2 u_hi), rank 0 the
  // first half and rank 1 the second -- equal counts, as one M = 256 MMA
  // covers a row tile of each.
  const uint32_t crank = CTA2 ? uint32_t(part & 1) : 0u;
  const bool leader = crank == 0;
  const int u_lo = int((long long)(rt_span / 2) * (part / 2) / (RS / 2 > 0 ? RS / 2 : 1));
  const int u_hi = int((long long)(rt_span / 2) * (part / 2 + 1) / (RS / 2 > 0 ? RS / 2 : 1));
  const int rt_lo = CTA2 ? rt_base + 2 * u_lo + int(crank) * (u_hi - u_lo)
                         : rt_base + int((long long)rt_span * part / RS);
  const int NRT = CTA2 ? u_hi - u_lo
                       : rt_base + int((long long)rt_span * (part + 1) / RS) - rt_lo;  // this CTA's
  // one stage = 128 bytes of K per row: 128 int8 or 256 e2m1 couplings/spins
  // (an FP4 row of npad = 128 is a partial chunk: TMA zero-fills the rest)
  const int NKC = (F4 && !pair) ? (g.npad + 2 * kBK - 1) / (2 * kBK)
                                : (i16 ? g.npad / (kBK / 2) : g.npad / kBK);
  // multi-instance problems: this tile's trial anneals its own J', H', offset
  const int j_row0 = P.multi ? tile * g.npad : 0;
  const int nchunk = NT / kCW;
  const int acc_cols = NT;
  constexpr int nsubs = EPI / 4;         // epilogue subgroups (4 warps each)
  const int nps = nslot / nsubs;         // ring slots per subgroup
  auto chunks_of = [&](int sb) { return (nchunk - sb + nsubs - 1) / nsubs; };
  // row tiles per "rows ready" barrier (at most kMaxRowGroups barriers)
  const int rgroup = (NRT + kMaxRowGroups - 1) / kMaxRowGroups;
  const int nrg = (NRT + rgroup - 1) / rgroup;
  // spin rows covered by one K chunk of the operand stream
  const int kKRows = (F4 && !pair) ? 2 * kBK : (i16 ? kBK / 2 : kBK);
  // clamped-table epilogue (use_tab 2, never with a row split): neighbour-sign
  // tiles built by the copier warp, energy partials kept in TMEM columns
  // [2 NT, 3 NT) across the row tiles when they fit below the scale factors
  // Fast epilogues without a row split take their neighbour signs from a
  // permuted sign tile built by the copier warp (nbt_mode): the clamped table
  // (use_tab 2, ct_mode) and the issue-lean FP64 epilogue (use_tab 0, epi_v4).
  const bool nbt_mode = P.fast && !split && !P.i16 && ((P.use_tab == 0 && P.rails_lo) || P.use_tab == 2);
  const bool ct_mode = nbt_mode && P.use_tab == 2;
  const uint32_t ct_tile_bytes = uint32_t(NT) * kCtTileRow * (P.bidirectional ? 2u : 1u);
  const bool e_tmem = nbt_mode && 3 * NT <= (F4 ? int(kSfCol) : 512);

  // ---- one-time setup ----
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&ctl->full[s], 1);
      mbar_init(&ctl->empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ctl->tfull[b], 1);
      mbar_init(&ctl->tempty[b], CTA2 ? 2 * EPI : EPI);  // pair: both CTAs' epilogues
      mbar_init(&ctl->sfull[b], nbt_mode ? 32u : 1u);  // copier warp: every lane arrives
      mbar_init(&ctl->sempty[b], EPI);
    }
    for (int s = 0; s < nslot; ++s) {
      mbar_init(&ctl->afull[s], 1);
      mbar_init(&ctl->aempty[s], 4);
    }
    for (int b = 0; b < nrg; ++b)
      mbar_init(&ctl->rready[b], EPI * (min(NRT, (b + 1) * rgroup) - b * rgroup));
    mbar_init(&ctl->done, EPI);
    mbar_init(&ctl->stg, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int r = 0; r < 4; ++r) {
      ctl->ring[r][0] = P.ring_cur;
      for (int q = 0; q <= P.d; ++q) ctl->ring[r][1 + q] = P.ring_phys[q];
    }
    ctl->last_pass = P.c_last;
  }
  if (threadIdx.x < 32) fill_noise_lut(ctl->nz_lut, P.nr, int(threadIdx.x));
  if (warp == kWarpProducer && lane == 0) {
    prefetch_tmap(&tmJ);
    prefetch_tmap(&tmS);
  }
  if (warp == kWarpLoader && lane == 0) {
    prefetch_tmap(&tmSe);
    prefetch_tmap(&tmA);
  }
  if (warp == kWarpMma) {
    const uint32_t ncols = (F4 || nbt_mode || i16 || 2 * acc_cols > 256) ? 512u : 256u;
    if (CTA2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&ctl->tmem_base)),
                   "r"(ncols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&ctl->tmem_base)),
                   "r"(ncols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  for (int c = threadIdx.x; c < NT; c += blockDim.x) {
    const ColInfo ci = decode_col(g, col0 + c);
    const int tl = ci.t - tile * g.tpt;
    c_key[c] = ci.live ? rng_key(P.seeds[ci.t], kStreamSweepNoise) : 0;
    const int kup = (ci.k + 1 == g.R) ? 0 : ci.k + 1;
    const int kdn = (ci.k == 0) ? g.R - 1 : ci.k - 1;
    c_col[c].base = 0;
    c_col[c].off = uint32_t(col0 + c) * uint32_t(g.npad);
    c_col[c].nbr = uint32_t(tl * g.R + kup) * kTileRow | (uint32_t(tl * g.R + kdn) * kTileRow << 16);
    c_kt[c] = ci.k | (tl << 16);
    c_flag[c] = ci.live ? 1 : 0;
  }
  for (int t = threadIdx.x; t < ntl; t += blockDim.x) {
    const int tg = tile * g.tpt + t;
    TrialTab tt{};
    tt.active = 1;
    tt.improved = -1;
    if (P.run_mode) {
      tt.best_e = P.best_e[tg];
      tt.best_k = P.best_k[tg];
      tt.reached = P.reached[tg];
      tt.first_hit = P.first_hit[tg];
      tt.cycles_used = P.cycles_used[tg];
      tt.active = P.active[tg];
    }
    trials[t] = tt;
  }
  tc_fence_before();
  // clusters: barriers initialised and TMEM allocated in every CTA before any
  // cross-CTA arrive, commit or TMA
  if (CL) cluster_sync_all();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = ctl->tmem_base;
  constexpr int kMmaM = CTA2 ? 2 * kBM : kBM;
  const uint32_t idesc = F4 ? idesc_mxf4(kMmaM, NT) : idesc_i8(kMmaM, NT);
  const uint32_t sf_tmem = tmem_base + kSfCol;  // unit (2^0) block scales for FP4
  if (F4) {
    // every ue8m0 scale factor is 127 = 2^0: fill the whole scale region
    if (warp < 4) tmem_st16_const(tmem_base + (uint32_t(warp * 32) << 16) + kSfCol, 0x7F7F7F7Fu),
                  tmem_st16_const(tmem_base + (uint32_t(warp * 32) << 16) + kSfCol + 16, 0x7F7F7F7Fu);
    tc_fence_before();
    if (CTA2) cluster_sync_all();  // the leader's MMAs read both CTAs' scales
    else __syncthreads();
    tc_fence_after();
  }

  // Register split between the warpgroups (inside each role's branch, so
  // ptxas budgets each role's code separately): the control warpgroup
  // (producer, MMA issuer, loader, one idle warp) runs single-lane loops in
  // few registers and hands the rest to the epilogue warpgroups.
#define SSQA_CTL_REGS() asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kCtlRegs))
#define SSQA_EPI_REGS() asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(EpiRegs<EPI>::value))

  uint32_t it = 0;      // operand stage sequence (producer == MMA)
  uint32_t acc_it = 0;  // accumulator / row-tile sequence (MMA == loader == epilogue)

  // Passes are pipelined across roles: pass c+1's operand loads, MMAs and
  // state loads start as soon as the rows they read were written in pass c
  // (ctl->rready, one phase per pass), while the epilogue is still finishing
  // pass c and scanning it.  A pass that starts before the scan of the pass
  // before it has decided to stop is drained by the epilogue without work.
  // rows_wait(s, b): group b of pass index s (= c - c_first) is complete.
  auto rows_wait = [&](long s, int b) { mbar_wait(&ctl->rready[b], uint32_t(s) & 1u); };
  // the control warps' form (long waits, no issue-slot polling)
  auto rows_wait_lazy = [&](long s, int b) { mbar_wait_lazy(&ctl->rready[b], uint32_t(s) & 1u, 256); };
  auto stop_at = [&](long c) { return c > *reinterpret_cast<volatile long*>(&ctl->last_pass); };

  if (warp == kWarpProducer) {
    // ===== operand TMA producer =====
    SSQA_CTL_REGS();
    if (lane == 0) {
      int* ring = ctl->ring[0];
      const uint64_t pol_keep = policy_evict_last();
      for (long c = P.c_first; c <= P.c_last; ++c) {
        const long s = c - P.c_first;
        int waited = 0;
        if (s > 0) {
          rows_wait_lazy(s - 1, 0);
          waited = 1;
          if (stop_at(c)) break;
        }
        const int yS = ring[0] * g.ccols + col0;
        for (int rt = 0; rt < NRT; ++rt) {
          for (int kc = 0; kc < NKC; ++kc, ++it) {
            if (s > 0 && rt == 0) {
              // the spin rows of this K chunk were written by pass c-1
              if (split) {
                // ... by the CTAs owning them (row-ready pass stamps)
                const int r1 = min(NRT_all, ((kc + 1) * kKRows + kBM - 1) / kBM);
                for (int r = kc * kKRows / kBM; r < r1; ++r)
                  while (ld_acquire_gpu(&P.g_rows[tile * NRT_all + r]) < int(s)) __nanosleep(64);
                asm volatile("fence.proxy.async.global;" ::: "memory");
              } else {
                const int need = min(nrg - 1, min(NRT - 1, ((kc + 1) * kKRows - 1) / kBM) / rgroup);
                while (waited <= need) rows_wait_lazy(s - 1, waited++);
              }
            }
            const int st = it % stages;
            const uint32_t ph = (it / stages) & 1;
            mbar_wait_lazy(&ctl->empty[st], ph ^ 1, SSQA_LAZY_NS_PROD);
            if (P.exp_flags & 4) {
              if (!CTA2 || leader) mbar_arrive(&ctl->full[st]);
            } else if (CTA2) {
              // both CTAs' tiles complete on the leader's barrier: its own J'
              // rows and half of the spin columns from each CTA
              const uint32_t bar = mapa_rank(smem_u32(&ctl->full[st]), 0);
              if (leader) mbar_expect_tx(&ctl->full[st], 2 * (L.a_bytes + L.b_bytes));
              tma_load_2d_pair_hint(&tmJ, bar, sA + size_t(st) * L.a_bytes, kc * kBK,
                                    j_row0 + (rt_lo + rt) * kBM, pol_keep);
              tma_load_2d_pair(&tmS, bar, sB + size_t(st) * L.b_bytes, kc * b_row,
                               yS + int(crank) * (NT / 2));
            } else {
              // ablations 8 / 16: skip the J' / spin loads (stale smem operands)
              const bool la = !(P.exp_flags & 8), lb = !(P.exp_flags & 16);
              mbar_expect_tx(&ctl->full[st], (la ? L.a_bytes : 0u) + (lb ? L.b_bytes : 0u));
              if (la)
                tma_load_2d_hint(&tmJ, &ctl->full[st], sA + size_t(st) * L.a_bytes, kc * kBK,
                                 j_row0 + (rt_lo + rt) * kBM, pol_keep);
              if (lb)
                tma_load_2d(&tmS, &ctl->full[st], sB + size_t(st) * L.b_bytes, kc * b_row, yS);
            }
          }
        }
        if (c < P.sc) ring_advance(ring, c, P.d, P.nslots);
      }
    }
    __syncwarp();
    if (CL) cluster_sync_all();  // no CTA leaves while its cluster may still signal it
  } else if (warp == kWarpMma) {
    // ===== MMA issuer (the pair's leader only; the whole warp runs the loop,
    // one elected lane issues) =====
    SSQA_CTL_REGS();
    if (!CTA2 || leader) {
      for (long c = P.c_first; c <= P.c_last; ++c) {
        const long s = c - P.c_first;
        if (s > 0) {
          rows_wait_lazy(s - 1, 0);
          if (stop_at(c)) break;
        }
        for (int rt = 0; rt < NRT; ++rt, ++acc_it) {
          const int buf = acc_it & 1;
          const uint32_t aph = (acc_it >> 1) & 1;
          mbar_wait_lazy(&ctl->tempty[buf], aph ^ 1, SSQA_LAZY_NS_MMA);
          tc_fence_after();
          DBG_STAMP(0, acc_it, 0);
          const uint32_t d_tmem = tmem_base + uint32_t(buf * acc_cols);
          for (int kc = 0; kc < NKC; ++kc, ++it) {
            const int st = it % stages;
            const uint32_t ph = (it / stages) & 1;
            mbar_wait(&ctl->full[st], ph);
            tc_fence_after();
            // descriptors of the stage; the K sub-blocks advance the start
            // address by 32 B (+2 in the >>4 field)
            const uint64_t ad = umma_desc_sw128(smem_u32(sA + size_t(st) * L.a_bytes));
            const uint32_t b0 = smem_u32(sB + size_t(st) * L.b_bytes);
            if (i16 && !(P.exp_flags & 2)) {
              // A sub-blocks [Alo k0, Alo k1, Ahi k0, Ahi k1] against spin
              // sub-blocks [k0, k1, k0, k1]: D_lo = Alo sigma, D_hi = Ahi sigma
              const uint64_t bd = umma_desc_sw64(b0);
#pragma unroll
              for (int k = 0; k < kBK / 32; ++k)
                mma_i8_w<CTA2>(k < 2 ? d_tmem : d_tmem + uint32_t(2 * acc_cols), ad + uint64_t(2 * k),
                               bd + uint64_t(2 * (k & 1)), idesc, (kc | (k & 1)) ? 1u : 0u);
            } else if (pair && !(P.exp_flags & 2)) {
              // A sub-blocks [A1 k0, A1 k1, A2 k0, A2 k1] against spin
              // sub-blocks [k0, k1, k0, k1]: S = A1 sigma + A2 sigma
              const uint64_t bd = umma_desc_sw64(b0);
#pragma unroll
              for (int k = 0; k < kBK / 32; ++k)
                mma_mxf4_w<CTA2>(d_tmem, ad + uint64_t(2 * k), bd + uint64_t(2 * (k & 1)), idesc,
                                 (kc | k) ? 1u : 0u, sf_tmem);
            } else if (!(P.exp_flags & 2)) {
              const uint64_t bd = umma_desc_sw128(b0);
#pragma unroll
              for (int k = 0; k < kBK / 32; ++k) {
                if (F4)
                  mma_mxf4_w<CTA2>(d_tmem, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc,
                                   (kc | k) ? 1u : 0u, sf_tmem);
                else
                  mma_i8_w<CTA2>(d_tmem, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc,
                                 (kc | k) ? 1u : 0u);
              }
            }
            mma_commit_w<CTA2>(&ctl->empty[st]);
          }
          mma_commit_w<CTA2>(&ctl->tfull[buf]);
          DBG_STAMP(0, acc_it, 1);
        }
      }
    }
    __syncwarp();
    mbar_wait_lazy(&ctl->done, 0, 1000);
    tc_fence_after();
    const uint32_t ncols = (F4 || nbt_mode || i16 || 2 * acc_cols > 256) ? 512u : 256u;
    if (CTA2) {
      cluster_sync_all();  // both CTAs' epilogues are done with the pair's TMEM
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(ncols));
    } else {
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(ncols));
    }
  } else if (warp == kWarpLoader) {
    // ===== state loader: delayed-spin tile + accumulator chunks.  Lane sb
    // feeds epilogue subgroup sb's accumulator ring on its own, so one slow
    // subgroup never holds back the others' loads; lane 0 also loads the
    // delayed-spin tiles and keeps the slot ring. =====
    SSQA_CTL_REGS();
    if (lane < nsubs) {
      const int sb2 = lane;
      int* ring = ctl->ring[1];
      const uint64_t pol_first = policy_evict_first();
      const uint32_t my_chunks = uint32_t(chunks_of(sb2));
      for (long c = P.c_first; c <= P.c_last; ++c) {
        const long s = c - P.c_first;
        int waited = 0;
        if (s > 0) {
          rows_wait_lazy(s - 1, 0);
          waited = 1;
          if (stop_at(c)) break;
        }
        const int ySrc = ring[1 + int(c % (P.d + 1))] * g.ccols + col0;
        for (int rt = 0; rt < NRT; ++rt, ++acc_it) {
          // accumulators (and, for delay 0, the neighbour spins) of these rows
          // were written by pass c-1
          if (s > 0)
            while (waited <= rt / rgroup) rows_wait_lazy(s - 1, waited++);
          if (sb2 == 0 && split) {  // (without a row split warp EPI+3 loads these tiles)
            const int sb = acc_it & 1;
            const uint32_t sph = (acc_it >> 1) & 1;
            mbar_wait(&ctl->sempty[sb], sph ^ 1);
            DBG_STAMP(1, acc_it, 0);
            mbar_expect_tx(&ctl->sfull[sb], uint32_t(NT) * kTileRow);
            tma_load_2d(&tmSe, &ctl->sfull[sb], sig_tiles + size_t(sb) * NT * kTileRow,
                        (rt_lo + rt) * kTileRow, ySrc);
          }
          // chunk ch belongs to epilogue subgroup ch % nsubs and lands in that
          // subgroup's own ring (slots [sub*nps, sub*nps + nps)): each slot is
          // consumed, in order, by a single subgroup, so no consumer can ever
          // wait on a slot barrier two phases ahead (parity aliasing).
          for (int ch = sb2; ch < nchunk && !(SSQA_ABL & 128); ch += nsubs) {
            const uint32_t cnt = acc_it * my_chunks + uint32_t(ch / nsubs);
            const int slot = sb2 * nps + int(cnt % uint32_t(nps));
            const uint32_t ph = (cnt / uint32_t(nps)) & 1;
            mbar_wait_lazy(&ctl->aempty[slot], ph ^ 1, SSQA_LAZY_NS_LOAD);
            mbar_expect_tx(&ctl->afull[slot], kCW * kBM * 8);
            tma_load_2d_hint(&tmA, &ctl->afull[slot], acc_ring + size_t(slot) * kCW * kBM,
                             (rt_lo + rt) * kBM, col0 + ch * kCW, pol_first);
          }
          if (sb2 == 0) DBG_STAMP(1, acc_it, 1);
        }
        // every lane has read this cycle's ring entry before lane 0 moves it
        __syncwarp((1u << nsubs) - 1u);
        if (sb2 == 0 && c < P.sc) ring_advance(ring, c, P.d, P.nslots);
        __syncwarp((1u << nsubs) - 1u);
      }
    }
    __syncwarp();
    if (CL) cluster_sync_all();
  } else if (warp >= EPI) {
    // ===== row-ready publisher (row split only): once this CTA's epilogue has
    // written a group of its row tiles in pass c, stamp them for the other
    // CTAs of the column tile (their producers load all rows of sigma) =====
    SSQA_CTL_REGS();
    if (nbt_mode) {
      // ===== neighbour-sign tiles of the clamped-table epilogue: for row tile
      // rt, byte [column][row] = 8 where sigma_{k+1}(c-d) of that row is
      // negative (up plane), 16 where sigma_{k-1}(c-d) is (down plane,
      // bidirectional only), copied from the delayed spin slot with the
      // neighbour permutation applied (column p holds its neighbour's signs) =====
      int* ring = ctl->ring[3];
      const bool bidir = P.bidirectional != 0;
      const uint32_t rowstride = uint32_t(kCtTileRow) * (bidir ? 2u : 1u);
      // staging for the TMA-loaded spin rows (one tile, behind the two sign buffers)
      uint8_t* stg = sig_tiles + 2 * size_t(ct_tile_bytes);
      uint32_t it2 = 0, sph = 0;
      for (long c = P.c_first; c <= P.c_last; ++c) {
        const long s = c - P.c_first;
        int waited = 0;
        if (s > 0) {
          rows_wait_lazy(s - 1, 0);
          waited = 1;
          if (stop_at(c)) break;
        }
        const int ySrc = ring[1 + int(c % (P.d + 1))] * g.ccols + col0;
        for (int rt = 0; rt < NRT; ++rt, ++it2) {
          if (s > 0)
            while (waited <= rt / rgroup) rows_wait_lazy(s - 1, waited++);
          if (lane == 0) {
            mbar_expect_tx(&ctl->stg, uint32_t(NT) * kTileRow);
            tma_load_2d(&tmSe, &ctl->stg, stg, (rt_lo + rt) * kTileRow, ySrc);
          }
          const int buf = int(it2 & 1u);
          mbar_wait_lazy(&ctl->sempty[buf], ((it2 >> 1) & 1u) ^ 1u, SSQA_LAZY_NS_LOAD);
          mbar_wait(&ctl->stg, sph);
          sph ^= 1u;
          uint8_t* dst = sig_tiles + size_t(buf) * ct_tile_bytes;
          if (P.exp_flags & 32) {
            // timing ablation: stale neighbour signs (no copy)
          } else if (F4) {
            // 64 bytes (128 rows) per column: 4 x 16 bytes, each -> 32 sign bytes
            for (int u = lane; u < NT * 4; u += 32) {
              const int pcol = u >> 2, part = u & 3;
              const uint32_t nbr = c_col[pcol].nbr;
              int su = int((nbr & 0xffffu) / uint32_t(kTileRow));
              su = su < NT ? su : pcol;
              const uint4 w = *reinterpret_cast<const uint4*>(stg + size_t(su) * kTileRow + part * 16);
              const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
              uint32_t o[8];
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const uint32_t t = wv[k] & 0x88888888u;
                const uint32_t ev = (t << 4) & 0x80808080u, od = t & 0x80808080u;
                o[2 * k] = __byte_perm(ev, od, 0x5140);
                o[2 * k + 1] = __byte_perm(ev, od, 0x7362);
              }
              uint4* d = reinterpret_cast<uint4*>(dst + size_t(pcol) * rowstride + uint32_t(part) * 32u);
              d[0] = make_uint4(o[0], o[1], o[2], o[3]);
              d[1] = make_uint4(o[4], o[5], o[6], o[7]);
              if (bidir) {
                int sd = int(((nbr >> 16) & 0x7fffu) / uint32_t(kTileRow));
                sd = sd < NT ? sd : pcol;
                const uint4 w2 = *reinterpret_cast<const uint4*>(stg + size_t(sd) * kTileRow + part * 16);
                const uint32_t wv2[4] = {w2.x, w2.y, w2.z, w2.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  const uint32_t t = wv2[k] & 0x88888888u;
                  const uint32_t ev = (t << 4) & 0x80808080u, od = t & 0x80808080u;
                  o[2 * k] = __byte_perm(ev, od, 0x5140);
                  o[2 * k + 1] = __byte_perm(ev, od, 0x7362);
                }
                uint4* d2 = reinterpret_cast<uint4*>(dst + size_t(pcol) * rowstride + kCtTileRow +
                                                     uint32_t(part) * 32u);
                d2[0] = make_uint4(o[0], o[1], o[2], o[3]);
                d2[1] = make_uint4(o[4], o[5], o[6], o[7]);
              }
            }
          } else {
            // int8 +-1 rows: 128 bytes per column, 8 x 16 bytes
            for (int u = lane; u < NT * 8; u += 32) {
              const int pcol = u >> 3, part = u & 7;
              const uint32_t nbr = c_col[pcol].nbr;
              int su = int((nbr & 0xffffu) / uint32_t(kTileRow));
              su = su < NT ? su : pcol;
              const uint4 w = *reinterpret_cast<const uint4*>(stg + size_t(su) * kTileRow + part * 16);
              uint4* d = reinterpret_cast<uint4*>(dst + size_t(pcol) * rowstride + uint32_t(part) * 16u);
              *d = make_uint4(w.x & 0x80808080u, w.y & 0x80808080u, w.z & 0x80808080u,
                              w.w & 0x80808080u);
              if (bidir) {
                int sd = int(((nbr >> 16) & 0x7fffu) / uint32_t(kTileRow));
                sd = sd < NT ? sd : pcol;
                const uint4 w2 = *reinterpret_cast<const uint4*>(stg + size_t(sd) * kTileRow + part * 16);
                uint4* d2 = reinterpret_cast<uint4*>(dst + size_t(pcol) * rowstride + kCtTileRow +
                                                     uint32_t(part) * 16u);
                *d2 = make_uint4(w2.x & 0x80808080u, w2.y & 0x80808080u, w2.z & 0x80808080u,
                                 w2.w & 0x80808080u);
              }
            }
          }
          __syncwarp();  // the staging tile is read before the next TMA overwrites it
          mbar_arrive(&ctl->sfull[buf]);  // every lane (count 32): its stores are done
        }
        __syncwarp();
        if (lane == 0 && c < P.sc) ring_advance(ring, c, P.d, P.nslots);
        __syncwarp();
      }
    } else if (!split) {
      // ===== delayed-neighbour spin tiles (TMA), on their own warp so they never
      // queue behind the accumulator loads of an epilogue subgroup =====
      if (lane == 0) {
        int* ring = ctl->ring[3];
        uint32_t it2 = 0;
        for (long c = P.c_first; c <= P.c_last; ++c) {
          const long s = c - P.c_first;
          int waited = 0;
          if (s > 0) {
            rows_wait_lazy(s - 1, 0);
            waited = 1;
            if (stop_at(c)) break;
          }
          const int ySrc = ring[1 + int(c % (P.d + 1))] * g.ccols + col0;
          for (int rt = 0; rt < NRT; ++rt, ++it2) {
            if (s > 0)
              while (waited <= rt / rgroup) rows_wait_lazy(s - 1, waited++);
            const int sb = int(it2 & 1u);
            mbar_wait_lazy(&ctl->sempty[sb], ((it2 >> 1) & 1u) ^ 1u, SSQA_LAZY_NS_LOAD);
            mbar_expect_tx(&ctl->sfull[sb], uint32_t(NT) * kTileRow);
            tma_load_2d(&tmSe, &ctl->sfull[sb], sig_tiles + size_t(sb) * NT * kTileRow,
                        (rt_lo + rt) * kTileRow, ySrc);
          }
          if (c < P.sc) ring_advance(ring, c, P.d, P.nslots);
        }
      }
      __syncwarp();
    } else if (split && scan_mode && lane == 0) {
      for (long c = P.c_first; c <= P.c_last; ++c) {
        const long s = c - P.c_first;
        if (s > 0 && stop_at(c)) break;
        for (int b = 0; b < nrg; ++b) {
          rows_wait_lazy(s, b);
          __threadfence();
          const int r1 = min(NRT, (b + 1) * rgroup);
          for (int r = b * rgroup; r < r1; ++r)
            st_release_gpu(&P.g_rows[tile * NRT_all + rt_lo + r], int(s + 1));
        }
      }
    }
    __syncwarp();
    if (CL) cluster_sync_all();
  } else {
    // ===== epilogue =====
    SSQA_EPI_REGS();
    const int ew = warp;  // 0 .. EPI-1
    const int q = warp & 3;   // TMEM lane quarter this warp may access
    const int sub = ew >> 2;
    constexpr int kSubs = EPI / 4;
    int* ring = ctl->ring[2];
    bool drain = false;  // every trial of the tile has stopped: consume only
    for (long c = P.c_first; c <= P.c_last; ++c) {
      if (stop_at(c)) break;
      const bool do_update = c < P.sc;
      const int cur = ring[0];
      const int dst = do_update ? ring_free(cur, ring + 1, P.d, P.nslots) : cur;
      if (!drain && P.fast && P.use_tab == 2) {
        // clamped table (use_tab 2): row x = 0 .. tab_w + 1 holds X = tab_lo1 - 1 + x,
        // entry [x][combo] = fl(fl(X 2^-p + jperp u) [+ jperp d]) with the
        // reference's own operations (annealer.cpp:276-284); rows 0 and tab_w + 1
        // are decided fields (low / high) and stand for every field beyond them
        const double jp = P.run_mode ? P.jperp_tab[c] : P.jperp_fixed;
        const double jpos = __dmul_rn(jp, 1.0), jneg = __dmul_rn(jp, -1.0);
        const I2D i2 = make_i2d(P.shift_p);
        const int ncmb = P.bidirectional ? 4 : 2;
        for (int e = ew * 32 + lane; e < ncmb * (P.tab_w + 2); e += EPI * 32) {
          const int x = e / ncmb, cmb = e - x * ncmb;
          double in = scaled_i32(P.tab_lo1 - 1 + x, i2);
          in = __dadd_rn(in, (cmb & 1) ? jneg : jpos);
          if (P.bidirectional) in = __dadd_rn(in, (cmb & 2) ? jneg : jpos);
          ytab[e] = in;
        }
      }
      if (!drain && P.fast && P.use_tab == 1) {
        // this cycle's table of fl(fl(X 2^-p + jperp u) [+ jperp d]) (TabConsts),
        // with the reference's own operations (annealer.cpp:276-284)
        const double jp = P.run_mode ? P.jperp_tab[c] : P.jperp_fixed;
        const double jpos = __dmul_rn(jp, 1.0), jneg = __dmul_rn(jp, -1.0);
        const I2D i2 = make_i2d(P.shift_p);
        const int ncmb = P.bidirectional ? 4 : 2;
        for (int e = ew * 32 + lane; e < ncmb * P.tab_w; e += EPI * 32) {
          const int cmb = e / P.tab_w;
          double in = scaled_i32(P.tab_lo1 + (e - cmb * P.tab_w), i2);
          in = __dadd_rn(in, (cmb & 1) ? jneg : jpos);
          if (P.bidirectional) in = __dadd_rn(in, (cmb & 2) ? jneg : jpos);
          ytab[e] = in;
        }
      }
      if (!drain) {
        for (int c0 = ew * 32; c0 < NT; c0 += EPI * 32) {
          const int cl = c0 + lane;
          uint32_t upd = 0;
          if (cl < NT) {
            const int k = c_kt[cl] & 0xffff, tl = c_kt[cl] >> 16;
            // key + spin_counter(c, k, 0) * golden, plus mix64's initial += golden
            c_col[cl].base = c_key[cl] + spin_counter(uint64_t(c), uint32_t(k), 0) * kGolden + kGolden;
            const uint32_t live = uint32_t(c_flag[cl] & 1);
            upd = live && do_update && (!P.run_mode || trials[tl].active);
            c_col[cl].nbr = (c_col[cl].nbr & 0x7fffffffu) | (upd << 31);
            for (int qq = 0; qq < 4; ++qq) c_E[qq * NT + cl] = 0;
          }
          // per-chunk update masks (bit j: column 8 ch + j updates)
          const uint32_t bal = __ballot_sync(0xffffffffu, upd != 0u);
          if (lane < 4 && c0 + 8 * lane < NT) ctl->umask[c0 / 8 + lane] = uint8_t(bal >> (8 * lane));
        }
      }
      long long* q_sum = c_E + q * NT;
      epi_bar<EPI>();
      const double jperp = P.run_mode ? P.jperp_tab[c] : P.jperp_fixed;
      const double i0c = (P.run_mode && P.i0_tab) ? P.i0_tab[c] : P.i0;
      const UpdateConsts uc = make_consts(P.n_rnd, jperp, i0c, P.alpha);
      const I2D i2d = make_i2d(P.shift_p);
      const bool bidir = P.bidirectional != 0;
      const bool fast = P.fast != 0;
      FastConsts fc;
      fc.nr = P.nr;
      fc.jp_hi = uint32_t(__double2hiint(uc.jp_pos));
      fc.jp_lo = uint32_t(__double2loint(uc.jp_pos));
      fc.i0 = i0c;
      fc.hi_clamp = (P.run_mode && P.i0_tab) ? __dsub_rn(i0c, P.alpha) : P.hi_clamp;
      fc.lo_clamp = -i0c;
      TabConsts tc;
      tc.lo1 = P.tab_lo1;
      tc.hi = P.tab_hi;
      tc.w = P.tab_w;
      tc.i0_bits = __double_as_longlong(i0c);
      tc.lo_bits = static_cast<unsigned long long>(__double_as_longlong(fc.lo_clamp));
      tc.hic_bits = __double_as_longlong(fc.hi_clamp);
      tc.loc_bits = __double_as_longlong(fc.lo_clamp);
      tc.ytab = ytab;
      // sigma(c) is sign(acc(c)) once this kernel has updated the lattice;
      // on the first cycle it comes from the spin slot (init / written state).
      const bool sig_from_acc = c > P.c_first;
      const uint64_t pol_first = policy_evict_first();
      // spin slots: int8 [ccols][npad], or FP4 nibbles [ccols][npad/2]
      const size_t slot_bytes = F4 ? P.slot_elems / 2 : P.slot_elems;
      const uint8_t* sig_cur = P.sig_base + size_t(cur) * slot_bytes;
      uint8_t* sig_dst = P.sig_base + size_t(dst) * slot_bytes;
      for (int rt = 0; rt < NRT; ++rt, ++acc_it) {
        const int buf = acc_it & 1;
        const uint32_t aph = (acc_it >> 1) & 1;
        const int il = q * 32 + lane;  // row within the tile
        const int i = (rt_lo + rt) * kBM + il;
        const bool row_live = i < g.n;
        const uint32_t trow = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(buf * acc_cols);
        const uint8_t* stile = sig_tiles + size_t(buf) * NT * kTileRow;
        if (warp == 0) DBG_STAMP(2, acc_it, 0);
        mbar_wait(&ctl->sfull[buf], aph);
        mbar_wait(&ctl->tfull[buf], aph);
        tc_fence_after();
        if (warp == 0) DBG_STAMP(3, acc_it, 0);
        const uint32_t cnt0 = acc_it * uint32_t(chunks_of(sub));
        if (drain || (P.exp_flags & 1)) {
          // consume the chunks without the update arithmetic (drain, or the
          // ablation of the update math)
          uint32_t cnt = cnt0;
          for (int ch = sub; ch < nchunk; ch += kSubs, ++cnt) {
            const int slot = sub * nps + int(cnt % uint32_t(nps));
            mbar_wait(&ctl->afull[slot], (cnt / uint32_t(nps)) & 1);
            if (!drain) {
              int32_t v[kCW];
              tmem_ld8(trow + uint32_t(ch * kCW), v);
              const double* ab = acc_ring + size_t(slot) * kCW * kBM + il;
#pragma unroll
              for (int j = 0; j < kCW; ++j) {
                const uint32_t coff = c_col[ch * kCW + j].off;
                st_f64_if(reinterpret_cast<double*>(P.acc + i + uint64_t(coff)),
                          ab[j * kBM] + double(v[j]), false, pol_first);
              }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&ctl->aempty[slot]);
          }
        } else if ((rt_lo + rt) * kBM + q * 32 >= g.n) {
          // every row of this warp is padding (n is not a multiple of 128:
          // C2's last row tile has 16 live rows): nothing to update or store,
          // zero energy; hand the staged chunks back and keep the energy
          // partials in TMEM consistent (first tile: zero; last: reduce)
          const uint32_t e_tm = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(2 * acc_cols);
          const int e_mode = (!nbt_mode || !e_tmem || NRT == 1)
                                 ? 0 : (rt == 0 ? 1 : (rt == NRT - 1 ? 3 : 2));
          uint32_t cnt = cnt0;
          for (int ch = sub; ch < nchunk; ch += kSubs, ++cnt) {
            const int slot = sub * nps + int(cnt % uint32_t(nps));
            mbar_wait(&ctl->afull[slot], (cnt / uint32_t(nps)) & 1);
            if (e_mode == 1) {
              int32_t z[kCW];
#pragma unroll
              for (int j = 0; j < kCW; ++j) z[j] = 0;
              tmem_st8(e_tm + uint32_t(ch * kCW), z);
            } else if (e_mode == 3) {
              int32_t e[kCW];
              tmem_ld8_nw(e_tm + uint32_t(ch * kCW), e);
              asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
              reduce8_to_quarter(e, q_sum, ch * kCW, lane);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&ctl->aempty[slot]);
          }
        } else {
          const int h1 = row_live ? P.H[j_row0 + i] : 0;
          const int h2 = 2 * h1;
          EpiRow er;
          er.acc_i = reinterpret_cast<uint64_t>(P.acc + i);
          er.dst_i = reinterpret_cast<uint64_t>(sig_dst + (F4 ? i / 2 : i));
          er.cur_i = reinterpret_cast<uint64_t>(sig_cur + (F4 ? i / 2 : i));
          er.st_i = stile + (F4 ? il / 2 : il);
          er.nib_shift = 4u * uint32_t(i & 1);
          er.h1 = F4 ? h1 - 0x4B400000 : h1;
          er.h2 = F4 ? h2 - 0x4B400000 : h2;
          er.iG = uint64_t(i) * kGolden;
          asm volatile("mov.b32 %0, %1;" : "=r"(er.iG_lo) : "r"(uint32_t(er.iG)));
          asm volatile("mov.b32 %0, %1;" : "=r"(er.iG_hi) : "r"(uint32_t(er.iG >> 32)));
          er.pol_stream = pol_first;
          er.w_row = row_live;
          {
            const int r0 = (rt_lo + rt) * kBM + q * 32 + 8 * (lane & 3);  // first row of the word
            const int nl = min(8, max(0, g.n - r0));
            er.nib_live = nl >= 8 ? 0xffffffffu : ((1u << (4 * nl)) - 1u);
            er.dst_w = sig_dst + ((rt_lo + rt) * kBM + q * 32) / 2 + 4 * (lane & 3);
          }
          er.npeer = P.npeer;
          er.peer_delta = P.peer_delta;
          er.hi_off = i16 ? uint32_t(2 * acc_cols) : 0u;
          er.i_u32 = uint32_t(i);
          asm volatile("mov.b32 %0, %1;" : "=r"(er.p4) : "r"(4u));
          asm volatile("mov.b32 %0, %1;" : "=r"(er.p32) : "r"(32u));
          er.h1x = uint32_t(er.h1) + 0x80000000u;
          er.nz_lut = ctl->nz_lut;
#define SSQA_EPI(B, S, F, T)                                                               \
  epi_chunks<B, S, F, F4, T>(er, uc, fc, tc, i2d, ctl, acc_ring, c_col, q_sum, trow, \
                             sub, kSubs, nchunk, nps, cnt0, il, lane)
#define SSQA_EPI_FAST(B, S)                  \
  if (P.use_tab == 1) SSQA_EPI(B, S, true, true); \
  else SSQA_EPI(B, S, true, false)
          if (ct_mode) {
            V4Row vr;
            vr.iG_lo = er.iG_lo;
            vr.iG_hi = er.iG_hi;
            vr.p4 = er.p4;
            vr.p32 = er.p32;
            vr.h1x = er.h1x;
            vr.h2 = er.h2;
            vr.h1c = er.h1 - (P.tab_lo1 - 1);
            vr.ct_max = P.tab_w + 1;
            vr.ytab = smem_u32(ytab);
            vr.nbt = smem_u32(sig_tiles) + uint32_t(buf) * ct_tile_bytes + uint32_t(il);
            vr.lut = smem_u32(ctl->nz_lut);
            vr.e_tmem = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(2 * acc_cols);
            vr.e_mode = (!e_tmem || NRT == 1) ? 0 : (rt == 0 ? 1 : (rt == NRT - 1 ? 3 : 2));
            vr.acc_col = reinterpret_cast<uint64_t>(P.acc + size_t(col0) * g.npad + i);
            vr.col_stride32 = uint32_t(g.npad) * 8u;
            vr.dst_w = er.dst_w;
            vr.nib_live = er.nib_live;
            vr.cur_i = er.cur_i;
            vr.dst_i = er.dst_i;
            vr.nib_shift = er.nib_shift;
            vr.w_row = row_live;
            vr.jp_hi = fc.jp_hi;
            vr.jp_lo = fc.jp_lo;
            vr.hic_hi = uint32_t(__double2hiint(fc.hi_clamp));
            vr.loc_hi = uint32_t(__double2hiint(fc.lo_clamp));
            vr.rail_lo = uint32_t(__double2loint(fc.hi_clamp));
            vr.pol = pol_first;
            vr.exp = P.exp_flags;
#define SSQA_V4T(B, S)                                                                            \
  epi_v4<B, S, F4, true>(vr, fc, i2d, ctl, acc_ring, c_col, ctl->umask, q_sum, trow, sub, kSubs, \
                         nchunk, nps, cnt0, il, lane)
            if (sig_from_acc) {
              if (bidir) SSQA_V4T(true, true);
              else SSQA_V4T(false, true);
            } else {
              if (bidir) SSQA_V4T(true, false);
              else SSQA_V4T(false, false);
            }
#undef SSQA_V4T
          } else if (nbt_mode) {
            V4Row vr;
            vr.iG_lo = er.iG_lo;
            vr.iG_hi = er.iG_hi;
            vr.p4 = er.p4;
            vr.p32 = er.p32;
            vr.h1x = er.h1x;
            vr.h2 = er.h2;
            vr.nbt = smem_u32(sig_tiles) + uint32_t(buf) * ct_tile_bytes + uint32_t(il);
            vr.lut = smem_u32(ctl->nz_lut);
            vr.e_tmem = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(2 * acc_cols);
            vr.e_mode = (!e_tmem || NRT == 1) ? 0 : (rt == 0 ? 1 : (rt == NRT - 1 ? 3 : 2));
            vr.acc_col = reinterpret_cast<uint64_t>(P.acc + size_t(col0) * g.npad + i);
            vr.col_stride32 = uint32_t(g.npad) * 8u;
            vr.dst_w = er.dst_w;
            vr.nib_live = er.nib_live;
            vr.cur_i = er.cur_i;
            vr.dst_i = er.dst_i;
            vr.nib_shift = er.nib_shift;
            vr.w_row = row_live;
            vr.jp_hi = fc.jp_hi;
            vr.jp_lo = fc.jp_lo;
            vr.hic_hi = uint32_t(__double2hiint(fc.hi_clamp));
            vr.loc_hi = uint32_t(__double2hiint(fc.lo_clamp));
            vr.rail_lo = uint32_t(__double2loint(fc.hi_clamp));  // == loc's (fast_ok)
            vr.pol = pol_first;
            vr.exp = P.exp_flags;
#define SSQA_V4(B, S)                                                                       \
  epi_v4<B, S, F4>(vr, fc, i2d, ctl, acc_ring, c_col, ctl->umask, q_sum, trow, sub, kSubs, \
                   nchunk, nps, cnt0, il, lane)
            if (sig_from_acc) {
              if (bidir) SSQA_V4(true, true);
              else SSQA_V4(false, true);
            } else {
              if (bidir) SSQA_V4(true, false);
              else SSQA_V4(false, false);
            }
#undef SSQA_V4
          } else if (fast && sig_from_acc) {
            if (bidir) SSQA_EPI_FAST(true, true);
            else SSQA_EPI_FAST(false, true);
          } else if (fast) {
            if (bidir) SSQA_EPI_FAST(true, false);
            else SSQA_EPI_FAST(false, false);
          } else if (sig_from_acc) {
            if (bidir) SSQA_EPI(true, true, false, false);
            else SSQA_EPI(false, true, false, false);
          } else {
            if (bidir) SSQA_EPI(true, false, false, false);
            else SSQA_EPI(false, false, false, false);
          }
#undef SSQA_EPI_FAST
#undef SSQA_EPI
        }
        tc_fence_before();
        // this warp's spin rows and accumulators of row tile rt are in global
        // memory: make them visible to the TMA (async proxy) reads of pass c+1
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __syncwarp();
        if (warp == 0) DBG_STAMP(2, acc_it, 1);
        if (lane == 0) {
          if (CTA2 && !leader) mbar_arrive_cluster(mapa_rank(smem_u32(&ctl->tempty[buf]), 0));
          else mbar_arrive(&ctl->tempty[buf]);
          mbar_arrive(&ctl->sempty[buf]);
          mbar_arrive(&ctl->rready[rt / rgroup]);
        }
      }
      epi_bar<EPI>();
      const long s_idx = c - P.c_first;
      // energy partial sum of tile column cl over this CTA's rows
      auto cta_energy = [&](int cl) -> long long {
        long long ep = 0;
        for (int qq = 0; qq < 4; ++qq)
          ep += P.fast ? (long long)reinterpret_cast<const int*>(c_E + qq * NT)[cl]
                       : c_E[qq * NT + cl];
        return ep;
      };
      unsigned long long* gE_pass = split ? P.gE + size_t(s_idx & 1) * g.ccols + col0 : nullptr;
      bool do_scan = scan_mode && !drain;
      if (shard_mode) {
        // GPU row shard: this CTA's row partials of the pass energies; the
        // host all-gathers them with the shard's spin rows and scans
        for (int cl = ew * 32 + lane; cl < NT; cl += EPI * 32)
          atomicAdd(P.gE + col0 + cl, static_cast<unsigned long long>(cta_energy(cl)));
        if (P.npeer) {
          // fused exchange: this CTA's spin words (peer stores) and energy
          // atomics are done; the last CTA of the pass pushes the summed
          // partials to every peer and raises their flags
          epi_bar<EPI>();
          if (ew == 0 && lane == 0) {
            __threadfence_system();
            const unsigned done = atomicAdd(P.push_ctr, 1u);
            __threadfence();
            ctl->scan_me = done == gridDim.x - 1u;
          }
          epi_bar<EPI>();
          if (ctl->scan_me) {
            for (int col = ew * 32 + lane; col < g.ccols; col += EPI * 32) {
              const unsigned long long v = __ldcg(P.gE + col);
              for (int d = 0; d < P.npeer; ++d) P.peer_E[d][col] = v;
            }
            epi_bar<EPI>();
            if (ew == 0 && lane == 0) {
              __threadfence_system();
              for (int d = 0; d < P.npeer; ++d)
                asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(P.peer_flag[d]),
                             "r"(P.epoch)
                             : "memory");
              *P.push_ctr = 0u;  // next pass
            }
          }
        }
      }
      if (split && scan_mode && !drain) {
        // Row split: add this CTA's row partials to the column tile's pass
        // sums; the last CTA of the tile to arrive scans the pass.
        for (int cl = ew * 32 + lane; cl < NT; cl += EPI * 32)
          atomicAdd(gE_pass + cl, static_cast<unsigned long long>(cta_energy(cl)));
        __threadfence();
        epi_bar<EPI>();
        if (ew == 0 && lane == 0) {
          const unsigned old = atom_add_acq_rel_gpu(&P.g_arrive[tile], 1u);
          ctl->scan_me = old == unsigned((s_idx + 1) * RS - 1);
        }
        epi_bar<EPI>();
        do_scan = ctl->scan_me != 0;
        if (do_scan) {
          // the trial table as the previous pass's scanner left it
          for (int t = ew * 32 + lane; t < ntl; t += 32 * EPI) {
            const int tg = tile * g.tpt + t;
            trials[t].best_e = __ldcg(P.best_e + tg);
            trials[t].best_k = __ldcg(P.best_k + tg);
            trials[t].reached = __ldcg(P.reached + tg);
            trials[t].first_hit = __ldcg(reinterpret_cast<const long long*>(P.first_hit) + tg);
            trials[t].cycles_used = __ldcg(reinterpret_cast<const long long*>(P.cycles_used) + tg);
            trials[t].active = __ldcg(P.active + tg);
          }
          epi_bar<EPI>();
        }
      }

      // ===== scan (annealer.cpp:327-345), one warp per trial, lanes over replicas =====
      if (do_scan) {
        for (int t = ew; t < ntl; t += EPI) {
          TrialTab& tt = trials[t];
          if (!tt.active) continue;
          const int tg = tile * g.tpt + t;
          // The reference walks k = 0..R-1 keeping the first strict improvement;
          // that is the first k reaching min_k e_k, if that beats best_e.
          double bmin = __longlong_as_double(0x7ff0000000000000LL);  // +inf
          int bk = 0x7fffffff;
          for (int k = lane; k < g.R; k += 32) {
            const long long ep = split ? (long long)__ldcg(gE_pass + t * g.R + k)
                                       : cta_energy(t * g.R + k);
            const double ek = __dadd_rn(__dmul_rn(-0.5, scaled(ep, P.scale)),
                                        P.multi ? P.offsets[tg] : P.offset);
            if (P.record_trace) P.trace[(size_t(tg) * (P.sc + 1) + c) * g.R + k] = ek;
            if (ek < bmin) {
              bmin = ek;
              bk = k;
            }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bmin, o);
            const int ok = __shfl_xor_sync(0xffffffffu, bk, o);
            if (ov < bmin || (ov == bmin && ok < bk)) {
              bmin = ov;
              bk = ok;
            }
          }
          const int improved = bmin < tt.best_e ? bk : -1;
          __syncwarp();
          if (lane == 0 && improved >= 0) {
            tt.best_e = bmin;
            tt.best_k = improved;
            if (P.has_target && !tt.reached && bmin <= P.target_tol) {
              tt.reached = 1;
              tt.first_hit = c;
            }
          }
          if (lane == 0 && P.stop_at_target && tt.reached && c < P.sc) {
            tt.active = 0;
            tt.cycles_used = c;
          }
          if (improved >= 0)
            snap_best_state<F4>(P, cur, size_t(col0 + t * g.R + improved), tg, g.npad, lane);
          __syncwarp();
        }
      }
      epi_bar<EPI>();
      if (split && scan_mode && !drain) {
        if (do_scan) {
          // publish the scan: trial table -> global, clear the pass sums
          for (int t = ew * 32 + lane; t < ntl; t += 32 * EPI) {
            const int tg = tile * g.tpt + t;
            P.best_e[tg] = trials[t].best_e;
            P.best_k[tg] = trials[t].best_k;
            P.reached[tg] = trials[t].reached;
            P.first_hit[tg] = trials[t].first_hit;
            P.cycles_used[tg] = trials[t].cycles_used;
            P.active[tg] = trials[t].active;
          }
          for (int cl = ew * 32 + lane; cl < NT; cl += EPI * 32) gE_pass[cl] = 0ull;
          __threadfence();
          epi_bar<EPI>();
          if (ew == 0 && lane == 0) {
            int any = 0;
            for (int t = 0; t < ntl; ++t) any |= trials[t].active;
            st_release_gpu(&P.g_scan[tile], (s_idx + 1) | (any ? 0ll : (1ll << 62)));
          }
        }
        // every CTA of the column tile: the scan of this pass decides which
        // trials still update
        if (ew == 0 && lane == 0) {
          long long v;
          while (((v = ld_acquire_gpu(&P.g_scan[tile])) & ((1ll << 62) - 1)) < s_idx + 1)
            __nanosleep(128);
          ctl->scan_stop = int((v >> 62) & 1);
        }
        epi_bar<EPI>();
        if (!do_scan)
          for (int t = ew * 32 + lane; t < ntl; t += 32 * EPI)
            trials[t].active = __ldcg(P.active + tile * g.tpt + t);
      }
      epi_bar<EPI>();
      if (ew == 0 && lane == 0) {
        if (do_update) ring_advance(ring, c, P.d, P.nslots);
        if (scan_mode && !drain) {
          int any = 0;
          if (split) any = !ctl->scan_stop;
          else
            for (int t = 0; t < ntl; ++t) any |= trials[t].active;
          // nothing left to anneal: the other roles may already be in pass
          // c+1 -- let it run (drained) and stop everyone after it
          if (!any && c < P.c_last) ctl->last_pass = c + 1;
        }
      }
      epi_bar<EPI>();
      if (scan_mode && !drain &&
          c + 1 == *reinterpret_cast<volatile long*>(&ctl->last_pass) &&
          c + 1 <= P.c_last) {
        int any = 0;
        if (split) any = !ctl->scan_stop;
        else
          for (int t = 0; t < ntl; ++t) any |= trials[t].active;
        drain = !any;
      }
    }
    // results of this CTA's trials (the epilogue warps own the trial table)
    epi_bar<EPI>();
    if (scan_mode && part == 0) {
      for (int t = ew; t < ntl; t += EPI)
        expand_best_state<F4>(P, tile * g.tpt + t, g.n, g.npad, lane);
    }
    if (scan_mode && !split) {  // with a row split the scanners keep global current
      for (int t = ew * 32 + lane; t < ntl; t += 32 * EPI) {
        const int tg = tile * g.tpt + t;
        P.best_e[tg] = trials[t].best_e;
        P.best_k[tg] = trials[t].best_k;
        P.reached[tg] = trials[t].reached;
        P.first_hit[tg] = trials[t].first_hit;
        P.cycles_used[tg] = trials[t].cycles_used;
        P.active[tg] = trials[t].active;
      }
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&ctl->done);
    if (CL) cluster_sync_all();
  }
  // No code after the role branches: each role runs to the end on its own
  // register budget (the MMA warp releases TMEM once the epilogue is done).
}
#undef SSQA_CTL_REGS
#undef SSQA_EPI_REGS

// ------------------------------------------------------------------- host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

// 2D map over a row-major [rows][inner] array of `esize`-byte elements,
// box {box_inner, box_rows}.
bool make_map(CUtensorMap* m, void* base, CUtensorMapDataType dt, uint32_t esize,
              uint64_t inner, uint64_t rows, uint32_t box_inner, uint32_t box_rows,
              CUtensorMapSwizzle swz) {
  EncodeFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {inner * esize};
  cuuint32_t box[2] = {box_inner, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, dt, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Operand stages and per-subgroup state-ring depth inside ~226 KB: prefer
// deep accumulator rings (up to 3 slots per subgroup, so the loader runs
// chunks ahead of the HBM latency), then as many operand stages (<= 4) as fit.
// deep: operand-feed-bound shapes (row splits, FP4 pairs) -- as many operand
// stages as fit (up to 8: the bytes in flight set the J' / spin stream
// rate), then accumulator-ring slots.
Layout pick_layout(int NT, int tpt, int nsubs, int tile_row, int b_row, int b_cols,
                   int tab_bytes, bool deep) {
  const uint32_t cap = 226 * 1024;  // of 227 KB dynamic shared memory per CTA
  const int max_stages = deep ? 8 : 4;
  if (deep)
    for (int stages = max_stages; stages >= 4; --stages)
      for (int nps = 3; nps >= 1; --nps) {
        if (nps * nsubs > 16) continue;
        Layout L = make_layout(NT, tpt, stages, nps * nsubs, tile_row, b_row, b_cols, tab_bytes);
        if (L.total <= cap) return L;
      }
  for (int nps = 3; nps >= 1; --nps)
    for (int stages = max_stages; stages >= 2; --stages) {
      if (nps * nsubs > 16) continue;
      Layout L = make_layout(NT, tpt, stages, nps * nsubs, tile_row, b_row, b_cols, tab_bytes);
      // the epilogue-bound shapes want the accumulator stream deep (C3: 3 ring
      // slots per subgroup and 2 operand stages 218 us/sweep, 2 and 3: 222)
      if (L.total <= cap) return L;
    }
  return make_layout(NT, tpt, 2, nsubs, tile_row, b_row, b_cols, tab_bytes);
}

// Fast epilogue without a row split: 2 clamped table, 0 FP64 (update_fast2).
#ifndef SSQA_NOSPLIT_EPI
#define SSQA_NOSPLIT_EPI 0
#endif
constexpr int kDefaultNoSplitEpi = SSQA_NOSPLIT_EPI;

// 16 epilogue warps (4 per scheduler): the update chain is latency-bound,
// so more resident warps beat more registers per warp (C3: -5 %/sweep vs 12).
constexpr int kDefaultEpi = 16;

// A fused run with a row split (run_mode 1, g.rs > 1) spin-waits across the
// CTAs of a column tile, so every CTA must be resident at once: those
// launches are cooperative (the driver refuses a grid that cannot be
// co-resident -- also next to other work on the device -- instead of letting
// it deadlock) and checked against the occupancy first; the caller falls back
// to rs = 1 on cudaErrorNotSupported.
template <int EPI, bool F4>
cudaError_t launch_variant(int grid, int smem, cudaStream_t st, const CUtensorMap* maps,
                           const TcParams& P) {
  auto kern = k_sweep_tc<EPI, F4, 0>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const bool coop = P.run_mode == 1 && P.g.rs > 1;
  if (coop) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * (4 + EPI), smem);
    if (e != cudaSuccess) return e;
    if (per_sm * sms < grid) return cudaErrorNotSupported;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(32 * (4 + EPI));
  cfg.dynamicSmemBytes = size_t(smem);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = coop ? 1 : 0;
  e = cudaLaunchKernelEx(&cfg, kern, maps[0], maps[1], maps[2], maps[3], P);
  if (e == cudaErrorCooperativeLaunchTooLarge) return cudaErrorNotSupported;
  return e;
}

// CTA pairs (CL 1, clusters of 2).  Every CTA must be resident at once (the
// row split synchronises across CTAs), so the launch is refused
// (cudaErrorNotSupported) unless all grid / 2 clusters fit on the device.
template <bool F4, int CL>
cudaError_t launch_variant_pair(int grid, int smem, cudaStream_t st, const CUtensorMap* maps,
                                const TcParams& P) {
  auto kern = k_sweep_tc<16, F4, CL>;
  constexpr int csize = 2;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(32 * (4 + 16));
  cfg.dynamicSmemBytes = size_t(smem);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = unsigned(csize);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int clusters = 0;
  e = cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg);
  if (e != cudaSuccess) return e;
  if (csize * clusters < grid) return cudaErrorNotSupported;
  return cudaLaunchKernelEx(&cfg, kern, maps[0], maps[1], maps[2], maps[3], P);
}

// int8 spin slot -> FP4 (e2m1) slot: +1 -> 0x2, -1 -> 0xA, 0 -> 0x0.
__global__ void k_pack_fp4(const int8_t* __restrict__ src, uint8_t* __restrict__ dst,
                           size_t nbytes) {
  for (size_t b = blockIdx.x * size_t(blockDim.x) + threadIdx.x; b < nbytes;
       b += size_t(gridDim.x) * blockDim.x) {
    auto code = [](int v) { return v > 0 ? 0x2u : (v < 0 ? 0xAu : 0x0u); };
    dst[b] = uint8_t(code(src[2 * b]) | (code(src[2 * b + 1]) << 4));
  }
}

// Mapped host record of the device watchdog (see watchdog_fire); one per
// process, bound to every device the engine launches on.
WatchdogRec* g_host_wd = nullptr;
unsigned long long g_wd_devices = 0;  // bit d: g_watchdog set on device d

void watchdog_bind(int device) {
  if (device < 0 || device >= 64 || (g_wd_devices >> device) & 1ull) return;
  if (!g_host_wd) {
    void* h = nullptr;
    if (cudaHostAlloc(&h, sizeof(WatchdogRec), cudaHostAllocMapped | cudaHostAllocPortable) !=
        cudaSuccess)
      return;
    std::memset(h, 0, sizeof(WatchdogRec));
    g_host_wd = static_cast<WatchdogRec*>(h);
  }
  void* d = nullptr;
  if (cudaHostGetDevicePointer(&d, g_host_wd, 0) != cudaSuccess) return;
  if (cudaMemcpyToSymbol(g_watchdog, &d, sizeof(d)) == cudaSuccess)
    g_wd_devices |= 1ull << device;
}

int launch(ssqa_batch_s* b, TcParams& P, bool f4) {
  watchdog_bind(b->prob->device);
  const Geom& g = P.g;  // the batch geometry (a shard pass may use its own row split)
  // Table epilogue for row splits: their MMAs keep the tensor core busy, and
  // the FP64 units share its issue path; the FP64 epilogue is cheaper where
  // they are mostly free (C3: 1146 vs 1178 ms/step).  Tune key "tab" forces.
  // clamped-table epilogue elsewhere (two FP64 adds fewer than update_fast2).
  // Tune key "tab": 0 FP64 epilogue, 1 table epilogue, 2 clamped table.
  const bool tab_ok = P.fast && P.tab_w > 0;
  P.use_tab = tab_ok ? ((g.rs > 1 || P.npeer) ? 1 : kDefaultNoSplitEpi) : 0;
  if (tune().tab >= 0) P.use_tab = tab_ok ? std::min(2, tune().tab) : 0;
  if (P.fast && g.rs == 1 && !P.i16 && (P.use_tab == 2 || (P.use_tab == 0 && P.rails_lo))) {
    // the sign tiles of the copier warp must fit next to the smallest pipeline
    const bool pr = f4 && b->prob->q.fp4x2_ok;
    const Layout Lmin = make_layout(g.tile_cols, g.tpt, 2, 4, sig_tile_row(P, f4),
                                    pr ? kBK / 2 : kBK, g.tile_cols, tab_bytes_of(P));
    if (Lmin.total > 226u * 1024u) {
      P.use_tab = 0;
      P.rails_lo = 0;  // plain FP64 epilogue, spin tiles by TMA
    }
  }
  CUtensorMap maps[4];
  const uint64_t srows = uint64_t(b->nslots) * g.ccols;
  // FP4 rows are npad/2 bytes (two e2m1 values per byte)
  const uint64_t row_bytes = f4 ? uint64_t(g.npad) / 2 : uint64_t(g.npad);
  void* Jsrc = f4 ? static_cast<void*>(b->prob->d_J4) : static_cast<void*>(b->prob->d_J);
  // FP4 pair image: rows of npad bytes (two planes); spin stages of 64 bytes
  const bool pair = f4 && b->prob->q.fp4x2_ok;
  P.pair = pair ? 1 : 0;
  // int16 couplings: plane image rows of 2 npad bytes, 64-byte spin stages
  const bool i16 = !f4 && b->prob->q.i16;
  P.i16 = i16 ? 1 : 0;
  const uint64_t j_row_bytes = pair ? uint64_t(g.npad) : (i16 ? 2 * uint64_t(g.npad) : row_bytes);
  const uint32_t b_row = (pair || i16) ? kBK / 2 : kBK;
  void* Ssrc = f4 ? static_cast<void*>(b->d_sig4) : static_cast<void*>(b->d_sig);
  const uint32_t tile_row = f4 ? kBM / 2 : kBM;
  P.sig_base = static_cast<uint8_t*>(Ssrc);
  if (!make_map(&maps[0], Jsrc, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, j_row_bytes,
                uint64_t(g.npad) * b->prob->count, kBK, kBM, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_map(&maps[1], Ssrc, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, row_bytes, srows, b_row,
                g.tile_cols, (pair || i16) ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_map(&maps[2], Ssrc, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, row_bytes, srows, tile_row,
                g.tile_cols, CU_TENSOR_MAP_SWIZZLE_NONE) ||
      !make_map(&maps[3], b->d_acc, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, g.npad, g.ccols, kBM, kCW,
                CU_TENSOR_MAP_SWIZZLE_NONE)) {
    g_tc_err = "cuTensorMapEncodeTiled failed";
    return SSQA_ECUDA;
  }
  if (g.rs > 1 && P.run_mode == 1) {
    // row-split synchronisation state, zeroed for every launch
    const int nrt_all = g.npad / kBM;
    const size_t bytes = size_t(2) * g.ccols * 8 + size_t(g.ntiles) * 8 +
                         size_t(g.ntiles) * nrt_all * 4 + size_t(g.ntiles) * 4 + 64;
    if (b->split_bytes < bytes) {
      if (b->d_split) {
        cudaStreamSynchronize(b->prob->stream);  // the last launch may still use it
        pool_free(b->d_split);
      }
      b->d_split = nullptr;
      b->split_bytes = 0;
      if (pmalloc(&b->d_split, bytes) != cudaSuccess) {
        g_tc_err = "row-split state allocation failed";
        return SSQA_ECUDA;
      }
      b->split_bytes = bytes;
    }
    cudaMemsetAsync(b->d_split, 0, bytes, b->prob->stream);
    uint8_t* base = static_cast<uint8_t*>(b->d_split);
    P.gE = reinterpret_cast<unsigned long long*>(base);
    P.g_scan = reinterpret_cast<long long*>(base + size_t(2) * g.ccols * 8);
    P.g_rows = reinterpret_cast<int*>(base + size_t(2) * g.ccols * 8 + size_t(g.ntiles) * 8);
    P.g_arrive = reinterpret_cast<unsigned*>(P.g_rows + size_t(g.ntiles) * nrt_all);
  }
  // 12 epilogue warps (160 registers each) for the issue-lean epilogue without
  // a row split (C3: 213.9 vs 216.9 us/sweep with 16), 16 elsewhere (CTA pairs)
  const bool lean = P.fast && g.rs == 1 && !P.i16 && (P.use_tab == 2 || (P.use_tab == 0 && P.rails_lo));
  const int epi = tune().epi ? (tune().epi == 12 ? 12 : 16) : (lean ? 12 : kDefaultEpi);
  // CTA pairs (M = 256 MMAs, each CTA streams half of the spin columns): the
  // fused run's row split with an even number of parts per column tile and
  // of row tiles; tune key "cta2" 0 turns them off
  bool cta2 = P.run_mode == 1 && g.rs > 1 && g.rs % 2 == 0 && (g.npad / kBM) % 2 == 0 &&
              epi == 16;
  // ... and from 64 row tiles up: below, the MMAs are not what binds and the
  // pair's cross-CTA handshakes cost ~15 % (C3 blocks, scripts/geom_sweep.py);
  // tune key "cta2" 1 pairs whenever the shape allows
  if (tune().cta2 >= 0) cta2 = cta2 && tune().cta2 != 0;
  else cta2 = cta2 && g.npad / kBM >= 64;
  Layout L;
  auto setup = [&](bool pairs) {
    const int b_cols = pairs ? g.tile_cols / 2 : g.tile_cols;
    if (!make_map(&maps[1], Ssrc, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, row_bytes, srows, b_row,
                  uint32_t(b_cols), (pair || i16) ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B))
      return false;
    const int tab_bytes = tab_bytes_of(P);
    L = pick_layout(g.tile_cols, g.tpt, epi / 4, sig_tile_row(P, f4), int(b_row), b_cols, tab_bytes,
                    pair || i16 || g.rs > 1);
    if (tune().stages > 0) {  // experiment overrides
      L = make_layout(g.tile_cols, g.tpt, tune().stages, std::max(1, tune().nps) * (epi / 4),
                      sig_tile_row(P, f4), int(b_row), b_cols, tab_bytes);
    }
    P.stages = L.stages;
    P.nslot = L.nslot;
    return true;
  };
  if (!setup(cta2)) {
    g_tc_err = "cuTensorMapEncodeTiled failed";
    return SSQA_ECUDA;
  }
  int smem = int(L.total);
  const char* trace_path = tune().trace.empty() ? nullptr : tune().trace.c_str();
  long long* dbg = nullptr;
  const int dbg_rts = 4096;
  if (trace_path) {
    pmalloc(&dbg, sizeof(long long) * 4 * dbg_rts * 2);
    cudaMemsetAsync(dbg, 0, sizeof(long long) * 4 * dbg_rts * 2, b->prob->stream);
    P.dbg = dbg;
    P.dbg_rts = dbg_rts;
    P.dbg_skip = tune().tskip;
  }
  cudaError_t e;
  // one persistent CTA per (column tile, row part); every CTA must be
  // resident (the row split synchronises across CTAs): grid <= SM count
  int grid = g.ntiles * g.rs;
  if (cta2) {
    e = f4 ? launch_variant_pair<true, 1>(grid, smem, b->prob->stream, maps, P)
           : launch_variant_pair<false, 1>(grid, smem, b->prob->stream, maps, P);
    if (e == cudaErrorNotSupported) {  // the pairs do not all fit at once: single CTAs
      cudaGetLastError();
      cta2 = false;
      setup(false);
      smem = int(L.total);
    }
  }
  if (!cta2) {
    auto single = [&]() {
      return epi == 16 ? (f4 ? launch_variant<16, true>(grid, smem, b->prob->stream, maps, P)
                             : launch_variant<16, false>(grid, smem, b->prob->stream, maps, P))
                       : (f4 ? launch_variant<12, true>(grid, smem, b->prob->stream, maps, P)
                             : launch_variant<12, false>(grid, smem, b->prob->stream, maps, P));
    };
    e = single();
    if (e == cudaErrorNotSupported && P.g.rs > 1) {
      // the row parts cannot all be resident: every CTA runs all rows of its tile
      cudaGetLastError();
      P.g.rs = 1;
      if (P.use_tab == 2) P.use_tab = 0;  // layout and maps were set up for the split
      grid = g.ntiles;
      e = single();
    }
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_tc_err = std::string("k_sweep_tc launch: ") + cudaGetErrorString(e);
    return SSQA_ECUDA;
  }
  if (dbg) {
    std::vector<long long> h(size_t(4) * dbg_rts * 2);
    cudaStreamSynchronize(b->prob->stream);
    cudaMemcpy(h.data(), dbg, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
    pool_free(dbg);
    if (FILE* f = fopen(trace_path, "wb")) {
      fwrite(h.data(), sizeof(long long), h.size(), f);
      fclose(f);
    }
  }
  b->launches += 1;
  return SSQA_OK;
}

// The fast (table) epilogue is exact when every parameter is finite (so no
// accumulator is ever NaN or -0.0), i0 > 0, n_rnd * 2^p is a small integer,
// the per-quarter int32 energy partials cannot overflow and the table of the
// undecided fields fits (TabConsts): fields X 2^-p >= B = i0 + 2 |jperp| +
// max |acc| + 1 clamp high whatever the rest, X 2^-p <= -B clamp low.
constexpr int kTabMaxW = 255;
bool fast_ok(const ssqa_batch_s* b, TcParams* P) {
  const ssqa_params_c& p = b->p;
  const Quantized& q = b->prob->q;
  for (double v : {p.n_rnd, p.i0, p.alpha, p.jperp_min, p.jperp_max, p.i0 - p.alpha})
    if (!std::isfinite(v)) return false;
  for (double v : b->ssa_levels)
    if (!std::isfinite(v) || !std::isfinite(v - p.alpha)) return false;
  const double x = std::ldexp(p.n_rnd, q.p);
  // the noise joins the integer field through a byte table (noise_lut)
  if (x != std::floor(x) || std::fabs(x) > 127.0) return false;
  const double row_max = double(q.max_abs_j) * q.n + 2.0 * q.max_abs_h;
  if (row_max + std::fabs(x) >= double(1u << 30)) return false;
  if (double(q.npad) / 4.0 * row_max >= 2147483647.0) return false;
  // run-wide bounds: the largest i0, |accumulator| and |jperp| of any cycle
  double i0max = p.i0, accmax = std::max(p.i0, std::fabs(p.i0 - p.alpha)), jpmax = 0.0;
  if (b->ssa) {
    i0max = 0.0;
    for (double v : b->ssa_levels) {
      i0max = std::max(i0max, v);
      accmax = std::max(accmax, std::max(v, std::fabs(v - p.alpha)));
    }
  } else {
    jpmax = std::max(std::fabs(p.jperp_min), std::fabs(p.jperp_max));
  }
  P->nr = int(x);
  // the issue-lean epilogue selects the clamp rails' low word once
  auto lo_word = [](double v) { uint64_t b; std::memcpy(&b, &v, 8); return uint32_t(b); };
  P->rails_lo = 1;
  if (b->ssa) {
    for (double v : b->ssa_levels) P->rails_lo &= lo_word(v - p.alpha) == lo_word(-v);
  } else {
    P->rails_lo = lo_word(p.i0 - p.alpha) == lo_word(-p.i0);
  }
  // table epilogue when i0 > 0 and the undecided band fits (else tab_w = 0)
  P->tab_w = 0;
  bool pos = i0max > 0.0;
  for (double v : b->ssa_levels) pos = pos && v > 0.0;
  const double bound = std::ldexp(i0max + 2.0 * jpmax + accmax + 1.0, q.p);
  if (pos && bound < double(kTabMaxW) && 2 * int(std::ceil(bound)) - 1 <= kTabMaxW) {
    const int thi = int(std::ceil(bound));
    P->tab_hi = thi;
    P->tab_lo1 = 1 - thi;
    P->tab_w = 2 * thi - 1;
  }
  return true;
}

TcParams base_params(ssqa_batch_s* b) {
  TcParams P{};
  P.g = b->g;
  P.H = b->prob->d_H;
  P.multi = b->prob->count > 1 ? 1 : 0;
  P.offsets = b->prob->d_offsets;
  P.scale = b->prob->q.scale;
  P.offset = b->prob->q.offset;
  P.shift_p = b->prob->q.p;
  P.seeds = b->d_seeds;
  P.sig = b->d_sig;
  P.sig_base = reinterpret_cast<uint8_t*>(b->d_sig);
  P.slot_elems = b->slot_elems;
  P.nslots = b->nslots;
  P.d = b->d;
  P.acc = b->d_acc;
  P.jperp_tab = b->d_jperp;
  P.i0_tab = b->d_i0;
  P.i0 = b->p.i0;
  P.n_rnd = b->p.n_rnd;
  P.alpha = b->p.alpha;
  P.bidirectional = b->p.bidirectional;
  P.hi_clamp = b->p.i0 - b->p.alpha;
  P.lo_clamp = -b->p.i0;
  P.fast = fast_ok(b, &P) ? 1 : 0;
  P.i16 = b->prob->q.i16 ? 1 : 0;
  P.exp_flags = tune().exp;
  P.ring_cur = b->cur;
  for (int q = 0; q <= b->d; ++q) P.ring_phys[q] = b->phys[size_t(q)];
  P.best_e = b->d_best_e;
  P.best_k = b->d_best_k;
  P.reached = b->d_reached;
  P.first_hit = b->d_first_hit;
  P.cycles_used = b->d_cycles_used;
  P.active = b->d_active;
  P.best_state = b->d_best_state;
  P.best_packed = b->d_best_packed;
  P.trace = b->d_trace;
  return P;
}

// Host mirror of the kernel's ring evolution over `count` updates.
void advance_ring(ssqa_batch_s* b, long count) {
  for (long s = 0; s < count; ++s) {
    const int dst = ring_free(b->cur, b->phys.data(), b->d, b->nslots);
    b->phys[size_t(b->cycle % (b->d + 1))] = dst;
    b->cur = dst;
    b->cycle += 1;
  }
}

}  // namespace

// FP4 operands when every coupling is e2m1-exact, fields stay below 2^22
// (exact fp32 accumulation and float->int conversion) and the tile leaves
// room for the scale-factor columns; tune key "fp4" 0 forces int8.
void launch_pack_fp4(const int8_t* src, uint8_t* dst, size_t bytes, cudaStream_t st) {
  k_pack_fp4<<<1184, 256, 0, st>>>(src, dst, bytes);
}

bool tc_uses_fp4(const ssqa_batch_s* b) {
  const Quantized& q = b->prob->q;
  return (q.fp4_ok || q.fp4x2_ok) && b->d_sig4 && double(q.max_abs_j) * q.n < double(1 << 22) &&
         2 * b->g.tile_cols <= int(kSfCol) && tune().fp4 != 0;
}

bool tc_supported(int npad, int r, int delay) {
  return npad >= kBM && npad % kBM == 0 && r >= 1 && r <= kMaxCols && delay <= kMaxDelay;
}

int tc_run(ssqa_batch_s* b, const ScanArgs& sa) {
  if (b->d > kMaxDelay) {
    g_tc_err = "tcgen05 engine supports delay <= 30";
    return SSQA_EUNSUP;
  }
  TcParams P = base_params(b);
  P.c_first = 0;
  P.c_last = b->p.sc;
  P.sc = b->p.sc;
  P.run_mode = 1;
  P.has_target = sa.has_target;
  P.stop_at_target = sa.stop_at_target;
  P.record_trace = sa.record_trace;
  P.target_tol = sa.target_tol;
  // FP4 operands when every coupling is e2m1-exact, fields stay below 2^22
  // (exact fp32 accumulation and float->int conversion) and the tile leaves
  // room for the scale-factor columns; tune key "fp4" 0 forces int8.
  const bool f4 = tc_uses_fp4(b);
  if (f4) {
    const size_t bytes = size_t(b->nslots) * b->slot_elems / 2;
    launch_pack_fp4(b->d_sig, b->d_sig4, bytes, b->prob->stream);
    if (cudaGetLastError() != cudaSuccess) {
      g_tc_err = "k_pack_fp4 launch failed";
      return SSQA_ECUDA;
    }
    b->launches += 1;
  }
  int rc = launch(b, P, f4);
  if (rc) return rc;
  advance_ring(b, b->p.sc);
  b->lattice_stale = f4;
  return SSQA_OK;
}

int tc_sweep(ssqa_batch_s* b, double jperp, double i0) {
  if (b->d > kMaxDelay) {
    g_tc_err = "tcgen05 engine supports delay <= 30";
    return SSQA_EUNSUP;
  }
  TcParams P = base_params(b);
  P.c_first = b->cycle;
  P.c_last = b->cycle;
  P.sc = b->cycle + 1;  // exactly one update
  P.run_mode = 0;
  P.fast = 0;  // hand-written lattices may hold any double: exact path only
  P.jperp_fixed = jperp;
  P.i0 = i0;
  P.hi_clamp = i0 - b->p.alpha;
  P.lo_clamp = -i0;
  if (b->lattice_stale) {
    g_tc_err = "lattice state is not kept after a fused run; re-init first";
    return SSQA_EINVAL;
  }
  int rc = launch(b, P, false);
  if (rc) return rc;
  advance_ring(b, 1);
  return SSQA_OK;
}

int tc_shard_pass(ssqa_batch_s* b, int rt0, int nrt, unsigned long long* gE) {
  if (b->d > kMaxDelay) {
    g_tc_err = "tcgen05 engine supports delay <= 30";
    return SSQA_EUNSUP;
  }
  TcParams P = base_params(b);
  P.c_first = b->cycle;
  P.c_last = b->cycle;
  P.sc = b->p.sc;  // cycle sc scans without an update
  P.run_mode = 2;
  P.shard_rt0 = rt0;
  P.shard_nrt = nrt;
  P.gE = gE;
  // row split of the shard's rows over the SMs the column tiles leave free
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, b->prob->device);
  P.g.rs = std::max(1, std::min(nrt, sms / std::max(1, P.g.ntiles)));
  // FP4 / FP4-pair operands when the problem has them (the merge keeps the
  // FP4 slots current, ssqa_batch_shard_begin packs the initial state)
  int rc = launch(b, P, tc_uses_fp4(b));
  if (rc) return rc;
  return SSQA_OK;
}

// The fused exchange needs FP4 operands and the table epilogue (its spin
// words are what goes to the peers).
bool tc_shard_direct_ok(ssqa_batch_s* b) {
  if (!tc_uses_fp4(b)) return false;
  TcParams P = base_params(b);
  return P.fast && P.tab_w > 0 && tune().tab < 0;
}

int tc_shard_pass_direct(ssqa_batch_s* b, int rt0, int nrt, unsigned long long* gE,
                         const long long* peer_delta, unsigned long long* const* peer_E,
                         unsigned* const* peer_flag, int npeer, unsigned epoch,
                         unsigned* push_ctr) {
  if (!tc_shard_direct_ok(b)) {
    g_tc_err = "fused shard exchange needs FP4 operands and the table epilogue";
    return SSQA_EUNSUP;
  }
  TcParams P = base_params(b);
  P.c_first = b->cycle;
  P.c_last = b->cycle;
  P.sc = b->p.sc;
  P.run_mode = 2;
  P.shard_rt0 = rt0;
  P.shard_nrt = nrt;
  P.gE = gE;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, b->prob->device);
  P.g.rs = std::max(1, std::min(nrt, sms / std::max(1, P.g.ntiles)));
  P.npeer = npeer;
  for (int d = 0; d < npeer; ++d) {
    P.peer_delta[d] = peer_delta[d];
    P.peer_E[d] = peer_E[d];
    P.peer_flag[d] = peer_flag[d];
  }
  P.epoch = epoch;
  P.push_ctr = push_ctr;
  return launch(b, P, true);
}

const char* tc_last_error() { return g_tc_err.c_str(); }

std::string tc_watchdog_message() {
  if (!g_host_wd || !reinterpret_cast<volatile WatchdogRec*>(g_host_wd)->fired) return "";
  const volatile WatchdogRec* w = g_host_wd;
  char buf[160];
  std::snprintf(buf, sizeof(buf),
                " [k_sweep_tc watchdog: block %d warp %d lane %d stuck on mbarrier smem 0x%x "
                "parity %u]",
                w->block, w->warp, w->lane, w->addr, w->parity);
  return buf;
}

}  // namespace ssqa_engine
