// dadd_probe.cu -- FP64 add throughput per SM, alone and while the tensor
// core runs kind::mxf4 MMAs (development tool, not the product).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(1) << 16) | (uint64_t(64) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

// warps 1..W: DADD chains (8 independent per thread); warp 0: MMAs if mma
__global__ void __launch_bounds__(640, 1) k(int iters, int mma_iters, int op, long long* out,
                                            double* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
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
  const long long t0 = clock64();
  if (warp == 0) {
    if (mma_iters > 0) {
      const uint32_t id = (1u << 7) | (1u << 10) | (uint32_t(224 >> 3) << 17) | (1u << 23) |
                          (uint32_t(128 >> 4) << 24);
      const uint64_t ad = desc_sw128(smem_u32(smem)), bd = desc_sw128(smem_u32(smem + 16384));
      for (int it = 0; it < mma_iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\t"
                       "setp.ne.b32 p, %4, 0;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, "
                       "%3, [%5], [%5], p;\n\t}" ::"r"(tm),
                       "l"(ad + 2 * kk), "l"(bd + 2 * kk), "r"(id), "r"(1u), "r"(tm + 480));
      }
      asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                   "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
                   ::"r"(smem_u32(&bar)) : "memory");
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
      if ((threadIdx.x & 31) == 0) out[blockIdx.x * 2 + 1] = clock64() - t0;
    }
  } else {
    double a[8];
    for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
    const double b = 1.0000001, c = -0.9999999;
    float f[8];
    for (int j = 0; j < 8; ++j) f[j] = threadIdx.x * 1e-3f + j;
    uint32_t u[8];
    for (int j = 0; j < 8; ++j) u[j] = threadIdx.x * 77u + j;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (op == 0) { a[j] = __dadd_rn(a[j], b); a[j] = __dadd_rn(a[j], c); }
        else if (op == 1) { f[j] = __fadd_rn(f[j], 1.0001f); f[j] = __fadd_rn(f[j], -1.0f); }
        else { u[j] = (u[j] ^ (u[j] >> 3)) + 0x9e37u; u[j] = (u[j] << 1) ^ 0x51u; }
      }
    }
    double s = 0;
    for (int j = 0; j < 8; ++j) s += a[j] + f[j] + u[j];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
    __syncwarp();
    if (warp == 1 && (threadIdx.x & 31) == 0) out[blockIdx.x * 2] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d; double* sink;
  cudaMalloc(&d, sizeof(long long) * 2 * sms);
  cudaMalloc(&sink, sizeof(double) * 640 * sms);
  const int smem = 64 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[3] = {"DADD", "FADD", "ALU(shift/xor/add)"};
  for (int op = 0; op < 3; ++op)
    for (int mma : {0, 1}) {
      const int iters = 2000;
      // MMA work sized to outlast the adds
      k<<<sms, 640, smem>>>(iters, mma ? 6000 : 0, op, d, sink);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[2 * 1024];
      cudaMemcpy(h, d, sizeof(long long) * 2 * sms, cudaMemcpyDeviceToHost);
      double cyc = 0;
      for (int i = 0; i < sms; ++i) cyc += double(h[2 * i]) / sms;
      const double ops = 19.0 * 32 * iters * 16;  // 19 warps x 32 lanes x 16 ops/iter
      printf("%-20s %s: %6.1f lane-ops/clk/SM (%s)\n", names[op], mma ? "with MMA   " : "alone      ",
             ops / cyc, cudaGetErrorString(e));
    }
  return 0;
}
