// eltwise.h -- memory-bound kernels of the training step (BN, ReLU, residual add, pooling,
// softmax cross-entropy, SGD). NHWC fp32, 128-bit vectorised, deterministic reductions.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/pooch.h"

namespace pooch {

// ---- BN statistics from the conv epilogue's per-tile partial sums (fixed-order reduction).
// ws: >= bn_finalize_ws_bytes(C) bytes. Writes mean, invstd, scale = gamma*invstd,
// shift = beta - mean*scale (each [C]).
size_t bn_finalize_ws_bytes(int C);
pooch_status bn_finalize(const float* tile_sum, const float* tile_sq, int tiles, int C, int64_t count,
                         const float* gamma, const float* beta, float* mean, float* invstd, float* scale, float* shift,
                         double* ws, cudaStream_t st);

// ---- y = relu(a*sa + ta + [b*sb + tb | b | 0])   (BN-apply + residual + ReLU), rows x C
// mode: 0 = no residual, 1 = residual is BN(b) (projection), 2 = residual is b (identity)
pooch_status bn_apply_relu(const float* a, const float* sa, const float* ta, const float* b, const float* sb,
                           const float* tb, int mode, float* y, int64_t rows, int C, cudaStream_t st);

// ---- BN(+add)+ReLU backward. dz = gy * [y > 0] with y recomputed from (a, b) exactly as in
// the forward kernel. Pass 1 reduces per channel sum(dz) and sum(dz * xhat) for BN(a) (and
// BN(b) when mode == 1) into per-block partials; pass 2 (finalize) writes dgamma/dbeta and
// the apply coefficients; pass 3 writes ga = gamma*invstd*(dz - mean(dz) - xhat*mean(dz*xhat))
// (and gb likewise for mode 1; gb (=|+=) dz for mode 2).
struct BnBwdArgs {
  const float* a; const float* b; const float* gy;
  const float* sa; const float* ta; const float* sb; const float* tb;   // forward scale/shift
  const float* mean_a; const float* invstd_a; const float* gamma_a;
  const float* mean_b; const float* invstd_b; const float* gamma_b;
  float* dgamma_a; float* dbeta_a; float* dgamma_b; float* dbeta_b;
  float* ga; float* gb;
  int mode;            // 0, 1, 2 as above
  int gb_accumulate;   // mode 2: gb += dz
  int64_t rows;
  int C;
};
size_t bn_bwd_ws_bytes(int C);
pooch_status bn_bwd(const BnBwdArgs& a, float* ws, cudaStream_t st);
// BN(-ReLU) in pieces for the divided layers (divide.cu): partial sums of a chunk (mode 0)
// accumulated into acc[2][C] (fp64, chunk order); finalize dbeta / dgamma / coef (3C floats) from
// acc over total_rows; apply on a chunk. Forward: tile partials of a chunk's conv epilogue into
// acc[2][C], then mean / invstd / scale / shift from acc (bn_finalize's formula).
size_t bn_relu_bwd_partial_ws_bytes(int64_t rows, int C);   // ws of bn_relu_bwd_partial for `rows` rows
pooch_status bn_relu_bwd_partial(const BnBwdArgs& a, float* ws, double* acc, cudaStream_t st);
pooch_status bn_relu_bwd_finalize(const BnBwdArgs& a, const double* acc, int64_t total_rows, float* coef,
                                  cudaStream_t st);
pooch_status bn_relu_bwd_apply(const BnBwdArgs& a, const float* coef, cudaStream_t st);
pooch_status bn_acc_tiles(const float* ts, const float* tq, int tiles, int C, double* acc, cudaStream_t st);
pooch_status bn_finalize_sums(const double* acc, int C, int64_t count, const float* gamma, const float* beta,
                              float* mean, float* invstd, float* scale, float* shift, cudaStream_t st);

// ---- pooling (NHWC)
pooch_status maxpool_fwd(const float* x, float* y, int N, int H, int W, int C, int k, int s, int p, int Ho, int Wo,
                         cudaStream_t st);
// gx = gradient routed to the first maximum of every window (argmax recomputed from x)
// arg_ws: N*Ho*Wo*C bytes of scratch for the window argmax indices
// 3D max-pool k2 s2 p0 over x [D][H][W][C] (batch 1); bwd re-derives the first-max argmax from x
// 3D max-pool over x [D][H][W][C] (batch 1): k2 s2 p0 (the U-Net's, windows tile the input) or
// any k / s / p with -inf padding (ResNeXt-101 (3D)'s k3 s2 p1; bwd then takes arg_ws of
// Do*Ho*Wo*C bytes: the first-maximum index per output, gathered from the input side).
pooch_status maxpool3d_fwd(const float* x, float* y, int D, int H, int W, int C, cudaStream_t st, int k = 2,
                           int s = 2, int p = 0);
pooch_status maxpool3d_bwd(const float* x, const float* gy, float* gx, int D, int H, int W, int C, bool accumulate,
                           cudaStream_t st, int k = 2, int s = 2, int p = 0, uint8_t* arg_ws = nullptr);
pooch_status maxpool_bwd(const float* x, const float* gy, float* gx, uint8_t* arg_ws, int N, int H, int W, int C,
                         int k, int s, int p, int Ho, int Wo, cudaStream_t st);
pooch_status avgpool_fwd(const float* x, float* y, int N, int HW, int C, cudaStream_t st);
pooch_status avgpool_bwd(const float* gy, float* gx, int N, int HW, int C, cudaStream_t st);

// ---- softmax cross-entropy over the first `classes` of `ld` logits per row.
// fwd: loss_rows[n], loss = mean (single-block fixed order). bwd: dz = (softmax - onehot) / B
// (padded columns get 0) and db[c] = sum_n dz[n][c].
// ws (nullable): ce_ws_bytes() of device scratch for the two-stage reductions of narrow heads
pooch_status ce_fwd(const float* z, const int32_t* labels, int B, int classes, int ld, float* loss_rows, float* loss,
                    cudaStream_t st, double* ws = nullptr);
pooch_status ce_bwd(const float* z, const int32_t* labels, int B, int classes, int ld, float* dz, float* db,
                    cudaStream_t st, double* ws = nullptr);
size_t ce_ws_bytes();

// ---- momentum SGD over n floats: v = mu*v + scale*g; w -= lr*v
pooch_status sgd_momentum(float* w, float* v, const float* g, int64_t n, float lr, float mu, float scale,
                          cudaStream_t st);

// ---- weight transpose for dgrad: wt[c][r][s][k] = w[k][r][s][c]
// Depth-folded 3D stem (ResNeXt-101 (3D), executor TaskRt::fold): xs[od][h][w][j] =
// x[od + u - p][h][w][c] for j = u*C + c < k*C (zero outside the volume and for j >= k*C), 32
// channels; the weight to / from the 2D layout W2[o][v][t][u*C + c] <-> W[o][u][v][t][c].
pooch_status depth_im2col(const float* x, float* xs, int D, int H, int W, int C, int k, int p, int Do,
                          cudaStream_t st);
pooch_status fold_weight(const float* w, float* w2, int K, int k, int C, cudaStream_t st);
pooch_status unfold_weight(const float* w2, float* w, int K, int k, int C, cudaStream_t st);
pooch_status transpose_krsc(const float* w, float* wt, int K, int RS, int C, cudaStream_t st);

}  // namespace pooch
