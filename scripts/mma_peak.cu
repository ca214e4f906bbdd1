// mma_peak.cu -- tcgen05 MMA throughput probe (development tool, not the product).
// One CTA per SM issues back-to-back MMAs on a fixed shared-memory tile (no
// TMA) into one TMEM accumulator and reports MACs per SM clock for
// kind::f16 (bf16), kind::i8 and kind::mxf4 at M = 128 and several N.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_peak scripts/mma_peak.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}
// kind: 0 f16 (bf16 in, f32 acc), 1 i8, 2 mxf4
__host__ __device__ constexpr uint32_t idesc(int kind, int M, int N) {
  return kind == 0 ? ((1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) |
                      (uint32_t(M >> 4) << 24))
       : kind == 1 ? ((2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) |
                      (uint32_t(M >> 4) << 24))
                   : ((1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (1u << 23) |
                      (uint32_t(M >> 4) << 24));
}

template <int KIND>
__global__ void __launch_bounds__(128, 1) k_peak(int N, int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tmem_base;
  if (KIND == 2 && warp < 4) {
    // unit scale factors in TMEM columns 480..511
    const uint32_t v = 0x7F7F7F7Fu, a = tm + (uint32_t(warp * 32) << 16) + 480;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
        "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(a), "r"(v));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    const uint32_t id = idesc(KIND, 128, N);
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 16384);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t ad = desc_sw128(a0 + k * 32), bd = desc_sw128(b0 + k * 32);
        const uint32_t acc = (it | k) ? 1u : 0u;
        if (KIND == 0)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                       "l"(ad), "l"(bd), "r"(id), "r"(acc));
        else if (KIND == 1)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                       "l"(ad), "l"(bd), "r"(id), "r"(acc));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, "
                       "%3, [%5], [%5], p;\n\t}" ::"r"(tm),
                       "l"(ad), "l"(bd), "r"(id), "r"(acc), "r"(tm + 480));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&bar)) : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                   "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
    cycles[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}


__device__ __forceinline__ void bar_wait(uint32_t a, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(a), "r"(ph) : "memory");
}

// Same MMAs behind a full/empty mbarrier ring of S stages, as the sweep
// kernel runs them: warp 1 lane 0 "produces" (waits empty, arrives full, no
// data movement), warp 0 lane 0 waits full, issues 4 MMAs, commits empty.
// mode bits: 1 issuer does not wait on full, 2 no per-stage commit (and no
// producer), 4 one smem address for every stage, 8 no tcgen05 fence, 16 MMAs
// per stage = 8 (two K atoms)
__global__ void __launch_bounds__(128, 1) k_pipe(int N, int iters, int S, int mode,
                                                 long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t full[8], empty[8], done;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < 8; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[s])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tmem_base;
  if (warp < 4) {
    const uint32_t v = 0x7F7F7F7Fu, a = tm + (uint32_t(warp * 32) << 16) + 480;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
        "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(a), "r"(v));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const long long t0 = clock64();
  if (warp == 1 && lane == 0 && !(mode & 2)) {
    for (int it = 0; it < iters; ++it) {
      const int st = it % S;
      bar_wait(smem_u32(&empty[st]), ((it / S) & 1) ^ 1);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[st])) : "memory");
    }
  } else if (warp == 0 && (mode & 32)) {
    // whole warp runs the loop; one elected lane issues inside the asm
    const uint32_t id = idesc(2, 128, N);
    for (int it = 0; it < iters; ++it) {
      const int st = it % S;
      bar_wait(smem_u32(&full[st]), (it / S) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a0 = smem_u32(smem + st * 4096), b0 = smem_u32(smem + 32768 + st * 4096);
      const uint64_t ad0 = desc_sw128(a0), bd0 = desc_sw128(b0);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t acc = (it | k) ? 1u : 0u;
        asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\t"
                     "setp.ne.b32 p, %4, 0;\n\t"
                     "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, "
                     "%3, [%5], [%5], p;\n\t}" ::"r"(tm),
                     "l"(ad0 + uint64_t(k * 2)), "l"(bd0 + uint64_t(k * 2)), "r"(id), "r"(acc),
                     "r"(tm + 480));
      }
      asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                   "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
                   ::"r"(smem_u32(&empty[st])) : "memory");
    }
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
                 ::"r"(smem_u32(&done)) : "memory");
    bar_wait(smem_u32(&done), 0);
    if (lane == 0) cycles[blockIdx.x] = clock64() - t0;
  } else if (warp == 0 && lane == 0) {
    const uint32_t id = idesc(2, 128, N);
    for (int it = 0; it < iters; ++it) {
      const int st = it % S;
      if (!(mode & 3)) bar_wait(smem_u32(&full[st]), (it / S) & 1);
      if (!(mode & 8)) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int so = (mode & 4) ? 0 : st;
      const uint32_t a0 = smem_u32(smem + so * 4096), b0 = smem_u32(smem + 32768 + so * 4096);
      const int nk = (mode & 16) ? 8 : 4;
#pragma unroll
      for (int k = 0; k < nk; ++k) {
        const uint64_t ad = desc_sw128(a0 + (k & 3) * 32 + (k >> 2) * 16384),
                       bd = desc_sw128(b0 + (k & 3) * 32 + (k >> 2) * 16384);
        const uint32_t acc = (it | k) ? 1u : 0u;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, "
                     "%3, [%5], [%5], p;\n\t}" ::"r"(tm),
                     "l"(ad), "l"(bd), "r"(id), "r"(acc), "r"(tm + 480));
      }
      if (!(mode & 2))
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&empty[st])) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&done)) : "memory");
    bar_wait(smem_u32(&done), 0);
    cycles[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

void run_pipe(int N, int S, int sms, int mode = 0) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * sms);
  const int iters = 4096, smem = 100 * 1024;
  cudaFuncSetAttribute(k_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_pipe<<<sms, 128, smem>>>(N, 64, S, mode, d);
  cudaError_t err = cudaDeviceSynchronize();
  k_pipe<<<sms, 128, smem>>>(N, iters, S, mode, d);
  err = cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < sms; ++i) cyc += double(h[i]) / sms;
  const double macs = 128.0 * N * 64 * ((mode & 16) ? 8.0 : 4.0) * iters;
  printf("pipe mxf4 N=%3d stages=%d mode=%2d: %8.1f MAC/clk/SM  %7.1f clk/stage (%s)\n", N, S,
         mode, macs / cyc, cyc / iters, cudaGetErrorString(err));
  cudaFree(d);
}

template <int KIND>
void run(const char* name, int kper, int N, int sms) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * sms);
  const int iters = 4096, smem = 100 * 1024;
  cudaFuncSetAttribute(k_peak<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_peak<KIND><<<sms, 128, smem>>>(N, 64, d);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_peak<KIND><<<sms, 128, smem>>>(N, iters, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[1024];
  cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < sms; ++i) cyc += double(h[i]) / sms;
  const double macs = 128.0 * N * kper * 4.0 * iters;  // per CTA
  printf("%-6s M=128 N=%3d K/instr=%3d: %8.1f MAC/clk/SM  %7.1f clk/instr  chip %.0f TOPS  (%s)\n",
         name, N, kper, macs / cyc, cyc / (4.0 * iters), 2.0 * macs * sms / (ms * 1e-3) / 1e12,
         cudaGetErrorString(err));
  cudaFree(d);
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mode : {0, 32})
    for (int N : {144, 224}) run_pipe(N, 4, sms, mode);
  for (int N : {128, 144, 224, 256}) {
    run<0>("bf16", 16, N, sms);
    run<1>("int8", 32, N, sms);
    run<2>("mxf4", 64, N, sms);
  }
  return 0;
}
