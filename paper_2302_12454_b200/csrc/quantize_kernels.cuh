// quantize_kernels.cuh -- device quantizer (see quantize_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace ssqa_engine {

// pmax <- max dyadic exponent of J[0..count) (atomicMax, start at 0);
// bad <- smallest index of a non-dyadic / non-finite entry (atomicMin).
void launch_qscan(const double* J, size_t count, int* pmax, unsigned long long* bad,
                  cudaStream_t st);
// Jq[i][j] = J[j][i] * up (int8, npad x npad, rows/cols >= n untouched: zero
// them first); maxabs <- max |Jq|, overflow <- 1 if any |J * up| > 127.
void launch_qtranspose(const double* J, int n, int npad, double up, int8_t* Jq, int* maxabs,
                       int* overflow, cudaStream_t st);
// J4 <- e2m1 image of Jq (elems couplings), not_fp4 <- 1 if any is not exact.
void launch_qfp4(const int8_t* Jq, size_t elems, uint8_t* J4, int* not_fp4, cudaStream_t st);

// J4 <- FP4 pair image of Jq (npad x npad bytes; engine.h Quantized::fp4x2_ok);
// not_split <- 1 if some |Jq| has no split (the image is then unusable).
void launch_qfp4x2(const int8_t* Jq, int npad, uint8_t* J4, int* not_split, cudaStream_t st);

// int16 couplings (127 < max |J'| <= 32639): Jq int16 [npad][npad] (transposed,
// scaled), overflow <- 1 beyond 32639; then the two-plane image (engine.h
// Quantized::i16), rows of 2 npad bytes.
void launch_qtranspose16(const double* J, int n, int npad, double up, int16_t* Jq, int* maxabs,
                         int* overflow, cudaStream_t st);
void launch_qplanes16(const int16_t* Jq, int npad, uint8_t* out, cudaStream_t st);

}  // namespace ssqa_engine
