// quantize_kernels.cu -- the quantizer of csrc/quantize.cpp on the device:
// the model's double couplings are uploaded once and scanned, scaled,
// transposed and packed where they will be used (ssqa_problem_create).
// Same rules as the host quantizer: the smallest p >= 0 making every
// coupling and bias an integer, J'[i][j] = J[j][i] * 2^p as int8 (|J'| <=
// 127, else unsupported), and the FP4 (e2m1) image when every J' is one of
// 0, +-1, +-2, +-3, +-4, +-6.
#include <cuda_runtime.h>

#include <cstdint>

#include "quantize_kernels.cuh"

namespace ssqa_engine {

namespace {

// Smallest p with v * 2^p integral (the IEEE bits: v = F * 2^(E-1075)), -1
// for inf / nan, 99 beyond the 62 the engine allows.
__device__ __forceinline__ int dyadic_exp_dev(double v) {
  const uint64_t b = uint64_t(__double_as_longlong(v));
  const int E = int((b >> 52) & 0x7ff);
  if (E == 0x7ff) return -1;
  uint64_t F = b & ((1ull << 52) - 1);
  if (E == 0 && F == 0) return 0;
  if (E != 0) F |= 1ull << 52;
  const int low = (E == 0 ? 1 : E) - 1075 + __ffsll((long long)F) - 1;
  const int p = low >= 0 ? 0 : -low;
  return p <= 62 ? p : 99;
}

__global__ void k_qscan(const double* __restrict__ J, size_t count, int* __restrict__ pmax,
                        unsigned long long* __restrict__ bad) {
  int local = 0;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < count;
       x += size_t(gridDim.x) * blockDim.x) {
    const int e = dyadic_exp_dev(J[x]);
    if (e < 0 || e > 62) atomicMin(bad, static_cast<unsigned long long>(x));
    else local = max(local, e);
  }
  for (int o = 16; o > 0; o >>= 1) local = max(local, __shfl_xor_sync(0xffffffffu, local, o));
  if ((threadIdx.x & 31) == 0 && local > 0) atomicMax(pmax, local);
}

// J'[i][j] = J[j][i] * up through a 32x32 shared tile (coalesced both ways).
__global__ void k_qtranspose(const double* __restrict__ J, int n, int npad, double up,
                             int8_t* __restrict__ Jq, int* __restrict__ maxabs,
                             int* __restrict__ overflow) {
  __shared__ int8_t tile[32][33];
  const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  int local = 0, bad = 0;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int j = j0 + r, i = i0 + threadIdx.x;
    int v = 0;
    if (j < n && i < n) {
      const double x = J[size_t(j) * n + i] * up;  // exact: a power-of-two scale
      if (fabs(x) > 127.0) bad = 1;
      else v = int(x);
    }
    tile[r][threadIdx.x] = int8_t(v);
    local = max(local, abs(v));
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = i0 + r, j = j0 + threadIdx.x;
    if (i < npad && j < npad) Jq[size_t(i) * npad + j] = tile[threadIdx.x][r];
  }
  for (int o = 16; o > 0; o >>= 1) {
    local = max(local, __shfl_xor_sync(0xffffffffu, local, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (local > 0) atomicMax(maxabs, local);
    if (bad) atomicOr(overflow, 1);
  }
}

// e2m1 image, two couplings per byte (lower K index in the low nibble).
__global__ void k_qfp4(const int8_t* __restrict__ Jq, size_t pairs, uint8_t* __restrict__ J4,
                       int* __restrict__ not_fp4) {
  // |v| -> e2m1 magnitude code (0, 1, 2, 3, 4, 6 representable)
  constexpr int kCode[8] = {0, 2, 4, 5, 6, -1, 7, -1};
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < pairs;
       x += size_t(gridDim.x) * blockDim.x) {
    const int a = Jq[2 * x], b = Jq[2 * x + 1];
    const int ma = a < 0 ? -a : a, mb = b < 0 ? -b : b;
    const int ca = ma < 8 ? kCode[ma] : -1, cb = mb < 8 ? kCode[mb] : -1;
    if (ca < 0 || cb < 0) {
      atomicOr(not_fp4, 1);
      continue;
    }
    J4[x] = uint8_t((ca | (a < 0 ? 8 : 0)) | ((cb | (b < 0 ? 8 : 0)) << 4));
  }
}

// FP4 pair image (engine.h Quantized::fp4x2_ok): one thread per output byte
// pair (A1 byte, A2 byte) = two couplings of a row; not_split <- 1 if any
// |J'| has no split (11, or > 12).
__global__ void k_qfp4x2(const int8_t* __restrict__ Jq, int npad, uint8_t* __restrict__ J4,
                         int* __restrict__ not_split) {
  constexpr int kA[13] = {0, 2, 4, 5, 6, 6, 7, 7, 7, 7, 7, 0, 7};
  constexpr int kB[13] = {0, 0, 0, 0, 0, 2, 0, 2, 4, 5, 6, 0, 7};
  const size_t pairs = size_t(npad) * (npad / 2);
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < pairs;
       x += size_t(gridDim.x) * blockDim.x) {
    const size_t i = x / (npad / 2);
    const int j = int(x % (npad / 2)) * 2;  // couplings j, j+1 of row i
    uint32_t a = 0, b = 0;
    for (int u = 0; u < 2; ++u) {
      const int v = Jq[i * npad + j + u];
      int m = v < 0 ? -v : v;
      if (m == 11 || m > 12) {
        atomicOr(not_split, 1);
        m = 0;
      }
      const uint32_t s = v < 0 ? 8u : 0u;
      if (kA[m]) a |= (uint32_t(kA[m]) | s) << (4 * u);
      if (kB[m]) b |= (uint32_t(kB[m]) | s) << (4 * u);
    }
    const size_t o = i * npad + size_t(j >> 7) * 128 + size_t((j & 127) >> 1);
    J4[o] = uint8_t(a);
    J4[o + 64] = uint8_t(b);
  }
}

// int16 variant of k_qtranspose: J16[i][j] = J[j][i] * up; overflow <- 1 if
// any |J * up| > kI16Max (int16 planes, engine.h Quantized::i16).
__global__ void k_qtranspose16(const double* __restrict__ J, int n, int npad, double up,
                               int16_t* __restrict__ Jq, int* __restrict__ maxabs,
                               int* __restrict__ overflow) {
  __shared__ int16_t tile[32][33];
  const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  int local = 0, bad = 0;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int j = j0 + r, i = i0 + threadIdx.x;
    int v = 0;
    if (j < n && i < n) {
      const double x = J[size_t(j) * n + i] * up;  // exact: a power-of-two scale
      if (fabs(x) > 32639.0) bad = 1;
      else v = int(x);
    }
    tile[r][threadIdx.x] = int16_t(v);
    local = max(local, abs(v));
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = i0 + r, j = j0 + threadIdx.x;
    if (i < npad && j < npad) Jq[size_t(i) * npad + j] = tile[threadIdx.x][r];
  }
  for (int o = 16; o > 0; o >>= 1) {
    local = max(local, __shfl_xor_sync(0xffffffffu, local, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (local > 0) atomicMax(maxabs, local);
    if (bad) atomicOr(overflow, 1);
  }
}

// Plane image of int16 J': row i, K chunk kc (64 couplings) -> 64 bytes of
// Alo then 64 bytes of Ahi at byte kc * 128 of a 2 npad-byte row.
__global__ void k_qplanes16(const int16_t* __restrict__ Jq, int npad, uint8_t* __restrict__ out) {
  const size_t total = size_t(npad) * npad;
  for (size_t x = blockIdx.x * size_t(blockDim.x) + threadIdx.x; x < total;
       x += size_t(gridDim.x) * blockDim.x) {
    const size_t i = x / size_t(npad);
    const int j = int(x % size_t(npad));
    const int v = Jq[x];
    const int lo = int(int8_t(uint8_t(v & 0xff)));
    const int hi = (v - lo) / 256;
    const size_t o = i * size_t(2 * npad) + size_t(j >> 6) * 128 + size_t(j & 63);
    out[o] = uint8_t(int8_t(lo));
    out[o + 64] = uint8_t(int8_t(hi));
  }
}

}  // namespace

void launch_qtranspose16(const double* J, int n, int npad, double up, int16_t* Jq, int* maxabs,
                         int* overflow, cudaStream_t st) {
  dim3 grid(npad / 32, npad / 32), block(32, 8);
  k_qtranspose16<<<grid, block, 0, st>>>(J, n, npad, up, Jq, maxabs, overflow);
}

void launch_qplanes16(const int16_t* Jq, int npad, uint8_t* out, cudaStream_t st) {
  k_qplanes16<<<1184, 256, 0, st>>>(Jq, npad, out);
}

void launch_qfp4x2(const int8_t* Jq, int npad, uint8_t* J4, int* not_split, cudaStream_t st) {
  k_qfp4x2<<<1184, 256, 0, st>>>(Jq, npad, J4, not_split);
}

void launch_qscan(const double* J, size_t count, int* pmax, unsigned long long* bad,
                  cudaStream_t st) {
  k_qscan<<<1184, 256, 0, st>>>(J, count, pmax, bad);
}

void launch_qtranspose(const double* J, int n, int npad, double up, int8_t* Jq, int* maxabs,
                       int* overflow, cudaStream_t st) {
  dim3 grid(npad / 32, npad / 32), block(32, 8);
  k_qtranspose<<<grid, block, 0, st>>>(J, n, npad, up, Jq, maxabs, overflow);
}

void launch_qfp4(const int8_t* Jq, size_t elems, uint8_t* J4, int* not_fp4, cudaStream_t st) {
  k_qfp4<<<1184, 256, 0, st>>>(Jq, elems / 2, J4, not_fp4);
}

}  // namespace ssqa_engine
