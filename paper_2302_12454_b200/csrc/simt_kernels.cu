// simt_kernels.cu -- lattice init, per-trial scan and the CUDA-core sweep
// engine (SSQA_ENGINE_SIMT).  The tcgen05 engine reuses init and scan.
#include "simt_kernels.cuh"

namespace ssqa_engine {

using namespace ssqa_dev;

// init_lattice (annealer.cpp:432-447): sigma = pm1(raw(spin_counter(0,k,i)))
// under key (seed, kStreamSpinInit); acc = 0.  One block per column.
__global__ void k_init(Geom g, const uint64_t* __restrict__ seeds, int8_t* __restrict__ sig,
                       double* __restrict__ acc) {
  const int col = blockIdx.x;
  const ColInfo c = decode_col(g, col);
  const uint64_t key = c.live ? rng_key(seeds[c.t], kStreamSpinInit) : 0;
  int8_t* s = sig + size_t(col) * g.npad;
  double* a = acc + size_t(col) * g.npad;
  for (int i = threadIdx.x; i < g.npad; i += blockDim.x) {
    int8_t v = 0;
    if (c.live && i < g.n) {
      v = (mix64(key + spin_counter(0, c.k, i) * kGolden) >> 63) ? 1 : -1;
    }
    s[i] = v;
    a[i] = 0.0;
  }
}

// Fresh AnnealResult per trial (annealer.cpp:323-324).
__global__ void k_reset_results(int T, long sc, double* best_e, int* best_k, int* reached,
                                long* first_hit, long* cycles_used, int* active) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  best_e[t] = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  best_k[t] = 0;
  reached[t] = 0;
  first_hit[t] = -1;
  cycles_used[t] = sc;
  active[t] = 1;
}

// S[col][i] = sum_j J'[i][j] sigma[col][j]  (int8 x int8 -> int32).
// 64 x 64 output tile per block, 4 x 4 per thread, 64-byte K chunks, dp4a.
__global__ void __launch_bounds__(256) k_field_simt(Geom g, const int8_t* __restrict__ J,
                                                    const int8_t* __restrict__ sig,
                                                    int32_t* __restrict__ S) {
  __shared__ int Js[kFB][kFB / 4 + 1];
  __shared__ int Ss[kFB][kFB / 4 + 1];
  const int i0 = blockIdx.x * kFB, c0 = blockIdx.y * kFB;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  int acc[4][4] = {};
  const int lr = threadIdx.x >> 2, lq = (threadIdx.x & 3) * 4;  // row, word offset
  for (int kk = 0; kk < g.npad; kk += kFB) {
    const int4 jv = *reinterpret_cast<const int4*>(J + size_t(i0 + lr) * g.npad + kk + lq * 4);
    int4 sv = make_int4(0, 0, 0, 0);
    if (c0 + lr < g.ccols)
      sv = *reinterpret_cast<const int4*>(sig + size_t(c0 + lr) * g.npad + kk + lq * 4);
    Js[lr][lq + 0] = jv.x; Js[lr][lq + 1] = jv.y; Js[lr][lq + 2] = jv.z; Js[lr][lq + 3] = jv.w;
    Ss[lr][lq + 0] = sv.x; Ss[lr][lq + 1] = sv.y; Ss[lr][lq + 2] = sv.z; Ss[lr][lq + 3] = sv.w;
    __syncthreads();
#pragma unroll 4
    for (int w = 0; w < kFB / 4; ++w) {
      int a[4], b[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r] = Js[ty * 4 + r][w];
#pragma unroll
      for (int r = 0; r < 4; ++r) b[r] = Ss[tx * 4 + r][w];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[r][q] = __dp4a(a[r], b[q], acc[r][q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int col = c0 + tx * 4 + q;
    if (col < g.ccols) {
      *reinterpret_cast<int4*>(S + size_t(col) * g.npad + i0 + ty * 4) =
          make_int4(acc[0][q], acc[1][q], acc[2][q], acc[3][q]);
    }
  }
}


// energies_from_fields (annealer.cpp:246-256) as an integer sum, fused with
// update_spins (annealer.cpp:258-300).  One block per column.
__global__ void __launch_bounds__(256) k_energy_update_simt(
    Geom g, const int32_t* __restrict__ S, const int32_t* __restrict__ H, double scale,
    const uint64_t* __restrict__ seeds, const int8_t* __restrict__ sig_cur,
    const int8_t* __restrict__ sig_src, int8_t* __restrict__ sig_dst, double* __restrict__ acc,
    long long* __restrict__ E, StepArgs a) {
  const int col = blockIdx.x;
  const ColInfo c = decode_col(g, col);
  const size_t base = size_t(col) * g.npad;
  if (!c.live) {
    if (a.do_update)
      for (int i = threadIdx.x; i < g.npad; i += blockDim.x) sig_dst[base + i] = 0;
    if (threadIdx.x == 0) E[col] = 0;
    return;
  }
  const uint64_t key = rng_key(seeds[c.t], kStreamSweepNoise);
  const UpdateConsts uc = make_consts(a.n_rnd, a.jperp, a.i0, a.alpha);
  const int kup = (c.k + 1 == g.R) ? 0 : c.k + 1;
  const int kdn = (c.k == 0) ? g.R - 1 : c.k - 1;
  const size_t up_base = size_t(col_of(g, c.t, kup)) * g.npad;
  const size_t dn_base = size_t(col_of(g, c.t, kdn)) * g.npad;
  long long e = 0;
  for (int i = threadIdx.x; i < g.npad; i += blockDim.x) {
    if (i >= g.n) {
      if (a.do_update) sig_dst[base + i] = 0;
      continue;
    }
    const int s = S[base + i], h = H[i];
    const int sg = sig_cur[base + i];
    e += (long long)(sg * (s + 2 * h));
    if (a.do_update) {
      const double field = scaled(s + h, scale);
      const uint32_t t5 = mix64_top5(key + spin_counter(uint64_t(a.cycle), c.k, i) * kGolden);
      const int up = sig_src[up_base + i];
      const int dn = a.bidirectional ? sig_src[dn_base + i] : 0;
      const double nv = update_one(uc, field, noise_index(t5), up, dn, a.bidirectional != 0,
                                   acc[base + i]);
      acc[base + i] = nv;
      sig_dst[base + i] = nv >= 0.0 ? 1 : -1;
    }
  }
  // block reduction of the integer energy (exact, order-free)
  __shared__ long long red[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    E[col] = tot;
  }
}


// scan_state (annealer.cpp:327-345) for one trial per warp: energies of all
// replicas in ascending k, strict-< best, first hit, optional trace; then
// the warp snapshots the best column (best_state, annealer.cpp:334-337).
__global__ void k_scan(Geom g, const long long* __restrict__ E, ScanArgs a,
                       const int8_t* __restrict__ sig_cur, double* best_e, int* best_k,
                       int* reached, long* first_hit, long* cycles_used, int* active,
                       int8_t* __restrict__ best_state, double* __restrict__ trace) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int t = warp;
  if (t >= g.T) return;
  if (!active[t]) return;
  int improved = -1;
  if (lane == 0) {
    double be = best_e[t];
    int hit = reached[t];
    for (int k = 0; k < g.R; ++k) {
      const long long ep = E[col_of(g, t, k)];
      const double ek = __dadd_rn(__dmul_rn(-0.5, scaled(ep, a.scale)), a.offset);
      if (ek < be) {
        be = ek;
        improved = k;
        if (a.has_target && !hit && be <= a.target_tol) {
          hit = 1;
          first_hit[t] = a.cycle;
        }
      }
      if (a.record_trace) trace[(size_t(t) * (a.sc + 1) + a.cycle) * g.R + k] = ek;
    }
    best_e[t] = be;
    if (improved >= 0) best_k[t] = improved;
    reached[t] = hit;
    if (a.stop_at_target && hit && a.cycle < a.sc) {
      active[t] = 0;
      cycles_used[t] = a.cycle;
    }
  }
  improved = __shfl_sync(0xffffffffu, improved, 0);
  if (improved >= 0) {
    const int8_t* src = sig_cur + size_t(col_of(g, t, improved)) * g.npad;
    int8_t* dst = best_state + size_t(t) * g.n;
    for (int i = lane; i < g.n; i += 32) dst[i] = src[i];
  }
}


// ---- GPU row shards: exchange chunk of one shard =
// [ccols][nwords] bit-packed spin rows (bit r of word w: row row0 + 32w + r
// is +1) followed by [ccols] int64 energy partials.
// Peer push (ssqa_batch_shard_pass_to): the chunk goes straight into every
// destination -- the shard's slot of each GPU's exchange region, peer memory
// over NVLink -- and the last block to finish raises each destination's flag
// for this shard to `epoch` (system-scope release after every block's
// system-scope fence): the all-gather is the pack kernel's own stores.
__device__ __forceinline__ void push_word(const PeerPush& pp, size_t byte_off, uint32_t v) {
  for (int d = 0; d < pp.n; ++d) *reinterpret_cast<uint32_t*>(pp.dst[d] + byte_off) = v;
}
__device__ __forceinline__ void push_i64(const PeerPush& pp, size_t byte_off, long long v) {
  for (int d = 0; d < pp.n; ++d) *reinterpret_cast<long long*>(pp.dst[d] + byte_off) = v;
}
__device__ __forceinline__ void push_signal(const PeerPush& pp) {
  if (!pp.counter) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned done = atomicAdd(pp.counter, 1u);
    if (done == gridDim.x - 1) {  // every block's stores are fenced: publish
      __threadfence_system();
      for (int d = 0; d < pp.n; ++d)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(pp.flag[d]), "r"(pp.epoch)
                     : "memory");
      *pp.counter = 0u;  // next pass
    }
  }
}

__global__ void k_shard_pack(Geom g, const int8_t* __restrict__ slot, int row0, int nwords,
                             const unsigned long long* __restrict__ E, PeerPush pp) {
  const size_t e_off = size_t(g.ccols) * nwords * 4;
  const size_t total = size_t(g.ccols) * nwords;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < total;
       x += size_t(gridDim.x) * blockDim.x) {
    const int col = int(x / nwords), w = int(x % nwords);
    const int4* src = reinterpret_cast<const int4*>(slot + size_t(col) * g.npad + row0 + 32 * w);
    const int4 a = src[0], b = src[1];
    const uint32_t v[8] = {uint32_t(a.x), uint32_t(a.y), uint32_t(a.z), uint32_t(a.w),
                           uint32_t(b.x), uint32_t(b.y), uint32_t(b.z), uint32_t(b.w)};
    uint32_t word = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int y = 0; y < 4; ++y) word |= uint32_t(int8_t(v[q] >> (8 * y)) > 0) << (4 * q + y);
    push_word(pp, x * 4, word);
  }
  for (int col = blockIdx.x * blockDim.x + threadIdx.x; col < g.ccols; col += gridDim.x * blockDim.x)
    push_i64(pp, e_off + size_t(col) * 8, static_cast<long long>(E[col]));
  push_signal(pp);
}

// FP4 spin slots (two e2m1 nibbles per byte, lower row in the low nibble,
// bit 3 = negative): the same bit-packed chunk from 16 bytes per 32 rows.
__global__ void k_shard_pack_fp4(Geom g, const uint8_t* __restrict__ slot4, int row0, int nwords,
                                 const unsigned long long* __restrict__ E, PeerPush pp) {
  const size_t e_off = size_t(g.ccols) * nwords * 4;
  const size_t total = size_t(g.ccols) * nwords;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < total;
       x += size_t(gridDim.x) * blockDim.x) {
    const int col = int(x / nwords), w = int(x % nwords);
    const int4 a = *reinterpret_cast<const int4*>(slot4 + size_t(col) * (g.npad / 2) +
                                                  (row0 + 32 * w) / 2);
    const uint32_t v[4] = {uint32_t(a.x), uint32_t(a.y), uint32_t(a.z), uint32_t(a.w)};
    uint32_t word = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int y = 0; y < 8; ++y)  // nibble y of word q = row 8q + y; positive when bit 3 clear
        word |= uint32_t(((v[q] >> (4 * y + 3)) & 1u) == 0u) << (8 * q + y);
    push_word(pp, x * 4, word);
  }
  for (int col = blockIdx.x * blockDim.x + threadIdx.x; col < g.ccols; col += gridDim.x * blockDim.x)
    push_i64(pp, e_off + size_t(col) * 8, static_cast<long long>(E[col]));
  push_signal(pp);
}

__global__ void k_shard_unpack(Geom g, int8_t* __restrict__ slot, uint8_t* __restrict__ slot4,
                               const uint8_t* __restrict__ all,
                               size_t chunk_bytes, int nshards, int rows_per_shard,
                               int with_spins, long long* __restrict__ E, PeerWait pw) {
  if (pw.flags) {
    // peer push: every shard's chunk of this epoch has landed once its flag
    // reads `epoch` (system-scope acquire)
    if (threadIdx.x < pw.n) {
      unsigned v;
      do {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(pw.flags + threadIdx.x)
                     : "memory");
      } while (int(v - pw.epoch) < 0);
    }
    __syncthreads();
  }
  const int nwords = rows_per_shard / 32;
  if (with_spins) {
    const size_t total = size_t(nshards) * g.ccols * nwords;
    for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < total;
         x += size_t(gridDim.x) * blockDim.x) {
      const int sh = int(x / (size_t(g.ccols) * nwords));
      const size_t r = x % (size_t(g.ccols) * nwords);
      const int col = int(r / nwords), w = int(r % nwords);
      const uint32_t word = reinterpret_cast<const uint32_t*>(all + size_t(sh) * chunk_bytes)[r];
      uint32_t v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        uint32_t b4 = 0;
#pragma unroll
        for (int y = 0; y < 4; ++y) b4 |= (((word >> (4 * q + y)) & 1u) ? 0x01u : 0xFFu) << (8 * y);
        v[q] = b4;
      }
      int4* dst = reinterpret_cast<int4*>(slot + size_t(col) * g.npad + size_t(sh) * rows_per_shard +
                                          32 * w);
      dst[0] = make_int4(int(v[0]), int(v[1]), int(v[2]), int(v[3]));
      dst[1] = make_int4(int(v[4]), int(v[5]), int(v[6]), int(v[7]));
      if (slot4) {  // the FP4 image for the next pass's MMAs (+1 -> 0x2, -1 -> 0xA)
        uint32_t n4[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t x4 = 0;
#pragma unroll
          for (int y = 0; y < 8; ++y)
            x4 |= (((word >> (8 * q + y)) & 1u) ? 0x2u : 0xAu) << (4 * y);
          n4[q] = x4;
        }
        *reinterpret_cast<int4*>(slot4 + size_t(col) * (g.npad / 2) +
                                 (size_t(sh) * rows_per_shard + 32 * w) / 2) =
            make_int4(int(n4[0]), int(n4[1]), int(n4[2]), int(n4[3]));
      }
    }
  }
  for (int col = blockIdx.x * blockDim.x + threadIdx.x; col < g.ccols; col += gridDim.x * blockDim.x) {
    long long e = 0;
    for (int sh = 0; sh < nshards; ++sh)
      e += reinterpret_cast<const long long*>(all + size_t(sh) * chunk_bytes +
                                              size_t(g.ccols) * nwords * 4)[col];
    E[col] = e;
  }
}

// Fused exchange (tc_shard_pass_direct): the peers' passes already stored
// their spin rows into this GPU's FP4 slot; once every shard's flag reads
// `epoch`, sum the pushed energy partials [nshards][ccols] and refresh the
// int8 slot (scan, best states) from the FP4 slot.
__global__ void k_shard_merge_direct(Geom g, int8_t* __restrict__ slot,
                                     const uint8_t* __restrict__ slot4,
                                     const uint8_t* __restrict__ parts, size_t part_stride,
                                     int nshards, int with_spins, long long* __restrict__ E,
                                     PeerWait pw) {
  if (threadIdx.x < pw.n) {
    unsigned v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(pw.flags + threadIdx.x)
                   : "memory");
    } while (int(v - pw.epoch) < 0);
  }
  __syncthreads();
  if (with_spins) {
    const size_t total = size_t(g.ccols) * (g.npad / 32);  // 32 rows = 16 bytes of nibbles
    for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < total;
         x += size_t(gridDim.x) * blockDim.x) {
      const int4 a = __ldcg(reinterpret_cast<const int4*>(slot4) + x);
      const uint32_t w[4] = {uint32_t(a.x), uint32_t(a.y), uint32_t(a.z), uint32_t(a.w)};
      uint32_t o[8];
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t b4 = 0;
#pragma unroll
          for (int y = 0; y < 4; ++y)  // nibble 4h + y of word q: bit 3 = negative
            b4 |= (((w[q] >> (4 * (4 * h + y) + 3)) & 1u) ? 0xFFu : 0x01u) << (8 * y);
          o[2 * q + h] = b4;
        }
      int4* dst = reinterpret_cast<int4*>(slot) + 2 * x;
      dst[0] = make_int4(int(o[0]), int(o[1]), int(o[2]), int(o[3]));
      dst[1] = make_int4(int(o[4]), int(o[5]), int(o[6]), int(o[7]));
    }
  }
  for (int col = blockIdx.x * blockDim.x + threadIdx.x; col < g.ccols; col += gridDim.x * blockDim.x) {
    long long e = 0;
    for (int sh = 0; sh < nshards; ++sh)
      e += __ldcg(reinterpret_cast<const long long*>(parts + size_t(sh) * part_stride) + col);
    E[col] = e;
  }
}

void launch_shard_merge_direct(const Geom& g, int8_t* slot, const uint8_t* slot4,
                               const void* parts, size_t part_stride, int nshards,
                               bool with_spins, long long* E, const PeerWait& pw,
                               cudaStream_t st) {
  k_shard_merge_direct<<<1184, 256, 0, st>>>(g, slot, slot4, static_cast<const uint8_t*>(parts),
                                             part_stride, nshards, with_spins ? 1 : 0, E, pw);
}

void launch_shard_pack(const Geom& g, const int8_t* slot, int row0, int rows,
                       const unsigned long long* E, const PeerPush& pp, cudaStream_t st) {
  k_shard_pack<<<1184, 256, 0, st>>>(g, slot, row0, rows / 32, E, pp);
}

void launch_shard_pack_fp4(const Geom& g, const uint8_t* slot4, int row0, int rows,
                           const unsigned long long* E, const PeerPush& pp, cudaStream_t st) {
  k_shard_pack_fp4<<<1184, 256, 0, st>>>(g, slot4, row0, rows / 32, E, pp);
}

void launch_shard_unpack(const Geom& g, int8_t* slot, uint8_t* slot4, const void* all,
                         size_t chunk_bytes, int nshards, int rows_per_shard, bool with_spins,
                         long long* E, const PeerWait& pw, cudaStream_t st) {
  k_shard_unpack<<<1184, 256, 0, st>>>(g, slot, slot4, static_cast<const uint8_t*>(all), chunk_bytes,
                                       nshards, rows_per_shard, with_spins ? 1 : 0, E, pw);
}

void launch_init(const Geom& g, const uint64_t* seeds, int8_t* sig, double* acc,
                 cudaStream_t st) {
  k_init<<<g.ccols, 256, 0, st>>>(g, seeds, sig, acc);
}

void launch_reset_results(int T, long sc, double* best_e, int* best_k, int* reached,
                          long* first_hit, long* cycles_used, int* active, cudaStream_t st) {
  k_reset_results<<<(T + 127) / 128, 128, 0, st>>>(T, sc, best_e, best_k, reached, first_hit,
                                                    cycles_used, active);
}

void launch_field_simt(const Geom& g, const int8_t* J, const int8_t* sig, int32_t* S,
                       cudaStream_t st) {
  dim3 grid(g.npad / kFB, (g.ccols + kFB - 1) / kFB);
  k_field_simt<<<grid, 256, 0, st>>>(g, J, sig, S);
}

void launch_energy_update_simt(const Geom& g, const int32_t* S, const int32_t* H, double scale,
                               const uint64_t* seeds, const int8_t* sig_cur,
                               const int8_t* sig_src, int8_t* sig_dst, double* acc,
                               long long* E, const StepArgs& a, cudaStream_t st) {
  k_energy_update_simt<<<g.ccols, 256, 0, st>>>(g, S, H, scale, seeds, sig_cur, sig_src,
                                                sig_dst, acc, E, a);
}

void launch_scan(const Geom& g, const long long* E, const ScanArgs& a, const int8_t* sig_cur,
                 double* best_e, int* best_k, int* reached, long* first_hit, long* cycles_used,
                 int* active, int8_t* best_state, double* trace, cudaStream_t st) {
  const int wpb = 4;
  k_scan<<<(g.T + wpb - 1) / wpb, 32 * wpb, 0, st>>>(g, E, a, sig_cur, best_e, best_k, reached,
                                                     first_hit, cycles_used, active, best_state,
                                                     trace);
}

}  // namespace ssqa_engine
