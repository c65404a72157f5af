// alex.h -- memory-bound kernels of the AlexNet workload (alex.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/pooch.h"

namespace pooch {

// local response normalisation (Krizhevsky et al.; Chainer's defaults): n = 5, k = 2,
// alpha = 1e-4, beta = 0.75 -- the oracle's layers.LRN_* constants
constexpr int kLrnN = 5;
constexpr float kLrnK = 2.f, kLrnAlpha = 1e-4f, kLrnBeta = 0.75f;

// y = LRN(x) over the C channels of every pixel; gx = its adjoint applied to gy (C <= 1024).
pooch_status lrn_fwd(const float* x, float* y, int64_t pixels, int C, cudaStream_t st);
pooch_status lrn_bwd(const float* x, const float* gy, float* gx, int64_t pixels, int C, cudaStream_t st);

// g (rows x C, in place) = y > 0 ? g * scale : 0; db[c] = sum over rows of the result (fixed order);
// ws: relu_mask_sum_ws_bytes(C) bytes
size_t relu_mask_sum_ws_bytes(int C);
pooch_status relu_mask_sum(float* g, const float* y, int64_t rows, int C, float scale, float* db, float* ws,
                           cudaStream_t st);

// inverted dropout in place (counter-based mask keyed by rng = {seed, step} in device memory)
pooch_status dropout_fwd(float* y, int64_t n, const uint32_t* rng, int task, float ratio, cudaStream_t st);
// rng[1] += 1 (the step counter, after the update)
pooch_status rng_advance(uint32_t* rng, cudaStream_t st);

}  // namespace pooch
