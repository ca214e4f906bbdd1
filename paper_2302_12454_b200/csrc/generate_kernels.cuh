// generate_kernels.cuh -- problems built on the device (see generate_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace ssqa_engine {

// Dense BASELINE model (kind 0: int[-8,7], kind 1: +-1) straight into J'
// (npad x npad, zero padding) and H' (npad); maxj / maxh <- max |J'| / |H'|.
void launch_gen_dense(int n, int npad, int kind, uint64_t key_j, uint64_t key_h, int8_t* J,
                      int32_t* H, int* maxj, int* maxh, cudaStream_t st);
// GI penalty couplings of `count` instances from their adjacency matrices
// (adj [count][2][nn][nn] bytes) into J' [count][npad][npad]; jo / jm: the
// scaled one-hot and edge-mismatch couplings; maxj <- max |J'|.
void launch_gen_gi(int count, int nn, int npad, int jo, int jm, const uint8_t* adj, int8_t* J,
                   int* maxj, cudaStream_t st);

}  // namespace ssqa_engine
