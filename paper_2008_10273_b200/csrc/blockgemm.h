// Config-2 block fit + reconstruct kernels (blockgemm.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace hivc {

// 64x64 fit-and-rebuild operator of one shared mask layout (float64).
void shared_block_operator(uint64_t mask, std::vector<double>& R);

// (a) rec = R f for every 8x8 block of a float32 plane, 3xTF32 tcgen05 GEMM.
// r_kl (nullable): the two halves pre-laid in the K-major UMMA layout for the
// TMA-fed kernel (planes of whole 8x8 blocks); else the generic kernel runs.
void launch_block_operator_tc(const float* plane, float* out, int h, int w, const float* r_hi, const float* r_lo,
                              int num_sms, cudaStream_t s, const float* r_kl = nullptr);

// (b) per-block masks (device uint64 per block), float64 shared-memory solves.
// status[0]: 1 empty mask, 2 singular, 4 a block needs the wide kernel;
// status[1] != 0: blocks with more than 8 points await the second pass.
void launch_block_perblock(const float* plane, float* out, int h, int w, const uint64_t* masks, int* status,
                           cudaStream_t s, bool wide = false, bool second_pass = false);

}  // namespace hivc
