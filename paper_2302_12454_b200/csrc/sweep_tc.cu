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
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <string>

#include "sweep_tc.h"

namespace ssqa_engine {

namespace {

constexpr int kBM = 128;          // rows (spins i) per MMA tile
constexpr int kBK = 128;          // K bytes per stage (one 128B swizzle row)
constexpr int kEpiWarps = 8;
constexpr int kThreads = 32 * (2 + kEpiWarps);
constexpr int kMaxDelay = 30;
constexpr int kMaxCols = 256;
constexpr int kMaxTrialsPerTile = 256;

thread_local std::string g_tc_err;

struct TcParams {
  Geom g;
  const int32_t* H;
  double scale, offset;
  const uint64_t* seeds;
  int8_t* sig;
  size_t slot_elems;
  int nslots, d;
  double* acc;
  const double* jperp_tab;  // per-cycle jperp (run mode)
  double jperp_fixed;       // sweep mode
  double i0, n_rnd, alpha;
  int bidirectional;
  long c_first, c_last;  // cycles handled: scans/updates for c in [c_first, c_last]
  long sc;               // update iff c < sc
  int run_mode;          // 1: scans + results; 0: plain sweeps (per-step API)
  int has_target, stop_at_target, record_trace;
  double target_tol;
  int ring_cur;
  int ring_phys[kMaxDelay + 1];
  int stages;
  // per-trial results
  double* best_e;
  int* best_k;
  int* reached;
  long* first_hit;
  long* cycles_used;
  int* active;
  int8_t* best_state;
  double* trace;
};

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

// Blocking wait with a watchdog: a pipeline that has not advanced for ~20 s
// traps (kernel error) instead of hanging the device.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try(a, parity)) return;
  const long long t0 = clock64();
  uint32_t n = 0;
  while (!mbar_try(a, parity)) {
    if ((++n & 1023u) == 0 && clock64() - t0 > 40000000000ll) {
      printf("k_sweep_tc: mbarrier wait timed out (block %d thread %d)\n", blockIdx.x,
             threadIdx.x);
      __trap();
    }
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

// Instruction descriptor, kind::i8: D = s32 (c_format 2), A = B = signed
// int8 (format 1), both K-major, N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) |
         (uint32_t(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
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

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void epi_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
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
struct ColTab {
  uint64_t key;   // CounterRng(seed_t, kStreamSweepNoise).key()
  uint64_t base;  // key + spin_counter(cycle, k, 0) * golden, for this cycle
  long long E;    // integer energy sum of this cycle
  int k, tl, up, dn;  // replica, trial-in-tile, neighbour columns (tile-local)
  int live;
};

struct TrialTab {
  double best_e;
  long first_hit, cycles_used;
  int best_k, reached, active, improved;
};

struct SmemCtl {
  uint64_t full[16];
  uint64_t empty[16];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
  int ring_cur, ring_dst, any_active;
  int ring_phys[kMaxDelay + 1];
};

__global__ void __launch_bounds__(kThreads, 1)
    k_sweep_tc(const __grid_constant__ CUtensorMap tmJ, const __grid_constant__ CUtensorMap tmS,
               const TcParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-align the operand area (SWIZZLE_128B atoms)
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const Geom& g = P.g;
  const int NT = g.tile_cols;
  const int stages = P.stages;
  const uint32_t a_bytes = kBM * kBK, b_bytes = uint32_t(NT) * kBK;
  uint8_t* sA = smem;
  uint8_t* sB = smem + size_t(stages) * a_bytes;
  uint8_t* tail = sB + size_t(stages) * b_bytes;
  SmemCtl* ctl = reinterpret_cast<SmemCtl*>(tail);
  ColTab* cols = reinterpret_cast<ColTab*>(tail + ((sizeof(SmemCtl) + 15) / 16) * 16);
  TrialTab* trials = reinterpret_cast<TrialTab*>(cols + NT);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x;
  const int col0 = tile * NT;  // first global column of this tile
  const int ntl = min(g.tpt, g.T - tile * g.tpt);  // live trials in this tile
  const int NRT = g.npad / kBM, NKC = g.npad / kBK;
  const int acc_cols = NT;  // TMEM columns per accumulator buffer

  // ---- one-time setup ----
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&ctl->full[s], 1);
      mbar_init(&ctl->empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ctl->tfull[b], 1);
      mbar_init(&ctl->tempty[b], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    ctl->ring_cur = P.ring_cur;
    for (int q = 0; q <= P.d; ++q) ctl->ring_phys[q] = P.ring_phys[q];
    ctl->any_active = 1;
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmJ);
    prefetch_tmap(&tmS);
  }
  if (warp == 1) {
    const uint32_t ncols = (2 * acc_cols <= 256) ? 256u : 512u;
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&ctl->tmem_base)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int c = threadIdx.x; c < NT; c += blockDim.x) {
    const ColInfo ci = decode_col(g, col0 + c);
    ColTab ct{};
    ct.live = ci.live;
    ct.k = ci.k;
    ct.tl = ci.t - tile * g.tpt;
    ct.key = ci.live ? rng_key(P.seeds[ci.t], kStreamSweepNoise) : 0;
    const int kup = (ci.k + 1 == g.R) ? 0 : ci.k + 1;
    const int kdn = (ci.k == 0) ? g.R - 1 : ci.k - 1;
    ct.up = ct.tl * g.R + kup;
    ct.dn = ct.tl * g.R + kdn;
    ct.E = 0;
    cols[c] = ct;
  }
  for (int t = threadIdx.x; t < ntl; t += blockDim.x) {
    const int tg = tile * g.tpt + t;
    TrialTab tt{};
    tt.active = 1;
    tt.improved = -1;
    if (!P.run_mode) {
      trials[t] = tt;
      continue;
    }
    tt.best_e = P.best_e[tg];
    tt.best_k = P.best_k[tg];
    tt.reached = P.reached[tg];
    tt.first_hit = P.first_hit[tg];
    tt.cycles_used = P.cycles_used[tg];
    tt.active = P.active[tg];
    tt.improved = -1;
    trials[t] = tt;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = ctl->tmem_base;
  const uint32_t idesc = idesc_i8(kBM, NT);

  uint32_t it = 0;      // smem pipeline position (producer and MMA agree)
  uint32_t acc_it = 0;  // accumulator position (MMA and epilogue agree)

  for (long c = P.c_first; c <= P.c_last; ++c) {
    const bool do_update = c < P.sc;
    const int cur = ctl->ring_cur;
    const int src = ctl->ring_phys[c % (P.d + 1)];
    const int dst = do_update ? ring_free(cur, ctl->ring_phys, P.d, P.nslots) : cur;
    if (!ctl->any_active) break;

    if (warp == 0) {
      // ===== TMA producer =====
      if (lane == 0) {
        const int yS = cur * g.ccols + col0;
        for (int rt = 0; rt < NRT; ++rt) {
          for (int kc = 0; kc < NKC; ++kc, ++it) {
            const int s = it % stages;
            const uint32_t ph = (it / stages) & 1;
            mbar_wait(&ctl->empty[s], ph ^ 1);
            mbar_expect_tx(&ctl->full[s], a_bytes + b_bytes);
            tma_load_2d(&tmJ, &ctl->full[s], sA + size_t(s) * a_bytes, kc * kBK, rt * kBM);
            tma_load_2d(&tmS, &ctl->full[s], sB + size_t(s) * b_bytes, kc * kBK, yS);
          }
        }
      }
      __syncwarp();
    } else if (warp == 1) {
      // ===== MMA issuer =====
      if (lane == 0) {
        for (int rt = 0; rt < NRT; ++rt, ++acc_it) {
          const int buf = acc_it & 1;
          const uint32_t aph = (acc_it >> 1) & 1;
          mbar_wait(&ctl->tempty[buf], aph ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + uint32_t(buf * acc_cols);
          for (int kc = 0; kc < NKC; ++kc, ++it) {
            const int s = it % stages;
            const uint32_t ph = (it / stages) & 1;
            mbar_wait(&ctl->full[s], ph);
            tc_fence_after();
            const uint32_t a0 = smem_u32(sA + size_t(s) * a_bytes);
            const uint32_t b0 = smem_u32(sB + size_t(s) * b_bytes);
#pragma unroll
            for (int k = 0; k < kBK / 32; ++k) {
              mma_i8(d_tmem, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc,
                     (kc | k) ? 1u : 0u);
            }
            mma_commit(&ctl->empty[s]);
          }
          mma_commit(&ctl->tfull[buf]);
        }
      }
      __syncwarp();
    } else {
      // ===== epilogue =====
      const int ew = warp - 2;             // 0..7
      const int q = warp & 3;              // TMEM lane quarter this warp may access
      const int half = ew >> 2;            // column half
      const int ncol_half = NT / 2;        // multiple of 8
      // per-cycle RNG bases and energy reset
      for (int cl = ew * 32 + lane; cl < NT; cl += kEpiWarps * 32) {
        cols[cl].base = cols[cl].key + spin_counter(uint64_t(c), uint32_t(cols[cl].k), 0) *
                                           kGolden;
        cols[cl].E = 0;
      }
      epi_bar();
      const double jperp = P.run_mode ? P.jperp_tab[c] : P.jperp_fixed;
      const UpdateConsts uc = make_consts(P.n_rnd, jperp, P.i0, P.alpha);
      const int8_t* sig_cur = P.sig + size_t(cur) * P.slot_elems;
      const int8_t* sig_src = P.sig + size_t(src) * P.slot_elems;
      int8_t* sig_dst = P.sig + size_t(dst) * P.slot_elems;
      for (int rt = 0; rt < NRT; ++rt, ++acc_it) {
        const int buf = acc_it & 1;
        const uint32_t aph = (acc_it >> 1) & 1;
        mbar_wait(&ctl->tfull[buf], aph);
        tc_fence_after();
        const int i = rt * kBM + q * 32 + lane;
        const bool row_live = i < g.n;
        const int h2 = row_live ? 2 * P.H[i] : 0;
        const int h1 = row_live ? P.H[i] : 0;
        const uint64_t iG = uint64_t(i) * kGolden;
        const uint32_t trow = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(buf * acc_cols);
        for (int cb = half * ncol_half; cb < (half + 1) * ncol_half; cb += 16) {
          int32_t v[16];
          tmem_ld16(trow + uint32_t(cb), v);
          const int nc = min(16, (half + 1) * ncol_half - cb);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (j >= nc) continue;
            const int cl = cb + j;
            const ColTab ct = cols[cl];
            int ep = 0;
            if (ct.live && row_live) {
              const size_t gi = size_t(col0 + cl) * g.npad + i;
              const int sgn = sig_cur[gi];
              const int S = v[j];
              ep = sgn * (S + h2);
              if (do_update && trials[ct.tl].active) {
                const double field = scaled(S + h1, P.scale);
                const uint32_t t5 = mix64_top5(ct.base + iG);
                const int up = sig_src[size_t(col0 + ct.up) * g.npad + i];
                const int dn = P.bidirectional ? sig_src[size_t(col0 + ct.dn) * g.npad + i] : 0;
                const double nv = update_one(uc, field, noise_index(t5), up, dn,
                                             P.bidirectional != 0, P.acc[gi]);
                P.acc[gi] = nv;
                sig_dst[gi] = nv >= 0.0 ? 1 : -1;
              }
            }
            const int wsum = __reduce_add_sync(0xffffffffu, ep);
            if (lane == 0 && ct.live) atomicAdd(reinterpret_cast<unsigned long long*>(&cols[cl].E),
                                                (unsigned long long)(long long)wsum);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ctl->tempty[buf]);
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    __syncthreads();

    // ===== scan (annealer.cpp:327-345), one warp per trial =====
    if (P.run_mode && warp >= 2) {
      for (int t = warp - 2; t < ntl; t += kEpiWarps) {
        TrialTab& tt = trials[t];
        if (!tt.active) continue;
        if (lane == 0) {
          double be = tt.best_e;
          int improved = -1;
          const int tg = tile * g.tpt + t;
          for (int k = 0; k < g.R; ++k) {
            const long long ep = cols[t * g.R + k].E;
            const double ek = __dadd_rn(__dmul_rn(-0.5, scaled(ep, P.scale)), P.offset);
            if (ek < be) {
              be = ek;
              improved = k;
              if (P.has_target && !tt.reached && be <= P.target_tol) {
                tt.reached = 1;
                tt.first_hit = c;
              }
            }
            if (P.record_trace) P.trace[(size_t(tg) * (P.sc + 1) + c) * g.R + k] = ek;
          }
          tt.best_e = be;
          if (improved >= 0) tt.best_k = improved;
          tt.improved = improved;
          if (P.stop_at_target && tt.reached && c < P.sc) {
            tt.active = 0;
            tt.cycles_used = c;
          }
        }
        __syncwarp();
        const int improved = tt.improved;
        if (improved >= 0) {
          const int8_t* s = P.sig + size_t(cur) * P.slot_elems +
                            size_t(col0 + t * g.R + improved) * g.npad;
          int8_t* dstp = P.best_state + size_t(tile * g.tpt + t) * g.n;
          for (int i = lane; i < g.n; i += 32) dstp[i] = s[i];
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (do_update) {
        ctl->ring_phys[c % (P.d + 1)] = dst;
        ctl->ring_cur = dst;
      }
      int any = 0;
      for (int t = 0; t < ntl; ++t) any |= trials[t].active;
      ctl->any_active = P.run_mode ? any : 1;
    }
    __syncthreads();
  }

  // ---- write back per-trial results ----
  if (P.run_mode) {
    for (int t = threadIdx.x; t < ntl; t += blockDim.x) {
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
  __syncthreads();
  if (warp == 1) {
    const uint32_t ncols = (2 * acc_cols <= 256) ? 256u : 512u;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(ncols));
  }
}

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

// 2D int8 map: inner dim `inner` bytes (K), `rows` rows, box {128, box_rows}.
bool make_map(CUtensorMap* m, void* base, uint64_t inner, uint64_t rows, uint32_t box_rows) {
  EncodeFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {inner};
  cuuint32_t box[2] = {uint32_t(kBK), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int smem_bytes(int NT, int stages) {
  return 1024 + stages * (kBM * kBK + NT * kBK) + int(((sizeof(SmemCtl) + 15) / 16) * 16) +
         NT * int(sizeof(ColTab)) + kMaxTrialsPerTile * int(sizeof(TrialTab));
}

int pick_stages(int NT) {
  int s = 8;
  while (s > 2 && smem_bytes(NT, s) > 220 * 1024) --s;
  return s;
}

int launch(ssqa_batch_s* b, TcParams& P) {
  const Geom& g = b->g;
  CUtensorMap tmJ, tmS;
  if (!make_map(&tmJ, b->prob->d_J, uint64_t(g.npad), uint64_t(g.npad), kBM) ||
      !make_map(&tmS, b->d_sig, uint64_t(g.npad), uint64_t(b->nslots) * g.ccols,
                uint32_t(g.tile_cols))) {
    g_tc_err = "cuTensorMapEncodeTiled failed";
    return SSQA_ECUDA;
  }
  P.stages = pick_stages(g.tile_cols);
  const int smem = smem_bytes(g.tile_cols, P.stages);
  cudaError_t e = cudaFuncSetAttribute(k_sweep_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem);
  if (e != cudaSuccess) {
    g_tc_err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e);
    return SSQA_ECUDA;
  }
  k_sweep_tc<<<g.ntiles, kThreads, smem, b->prob->stream>>>(tmJ, tmS, P);
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_tc_err = std::string("k_sweep_tc launch: ") + cudaGetErrorString(e);
    return SSQA_ECUDA;
  }
  b->launches += 1;
  return SSQA_OK;
}

TcParams base_params(ssqa_batch_s* b) {
  TcParams P{};
  P.g = b->g;
  P.H = b->prob->d_H;
  P.scale = b->prob->q.scale;
  P.offset = b->prob->q.offset;
  P.seeds = b->d_seeds;
  P.sig = b->d_sig;
  P.slot_elems = b->slot_elems;
  P.nslots = b->nslots;
  P.d = b->d;
  P.acc = b->d_acc;
  P.jperp_tab = b->d_jperp;
  P.i0 = b->p.i0;
  P.n_rnd = b->p.n_rnd;
  P.alpha = b->p.alpha;
  P.bidirectional = b->p.bidirectional;
  P.ring_cur = b->cur;
  for (int q = 0; q <= b->d; ++q) P.ring_phys[q] = b->phys[size_t(q)];
  P.best_e = b->d_best_e;
  P.best_k = b->d_best_k;
  P.reached = b->d_reached;
  P.first_hit = b->d_first_hit;
  P.cycles_used = b->d_cycles_used;
  P.active = b->d_active;
  P.best_state = b->d_best_state;
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
  int rc = launch(b, P);
  if (rc) return rc;
  advance_ring(b, b->p.sc);
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
  P.jperp_fixed = jperp;
  P.i0 = i0;
  int rc = launch(b, P);
  if (rc) return rc;
  advance_ring(b, 1);
  return SSQA_OK;
}

const char* tc_last_error() { return g_tc_err.c_str(); }

}  // namespace ssqa_engine
