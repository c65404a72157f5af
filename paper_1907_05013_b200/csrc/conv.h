// conv.h -- host launchers of the tensor-core implicit-GEMM kernels (igemm.cuh).
#pragma once
#include <cuda_runtime.h>

#include "../../include/pooch.h"

namespace pooch {

struct ConvGeom {
  int N, H, W, C, K, R, S, stride, pad, Ho, Wo;
  int prec = 0;  // 0: TF32 (one MMA per k-step), 1: 3xTF32 split (fp32-faithful)
};
ConvGeom conv_geom(const pooch_conv_desc& d);
bool conv_shape_ok(const ConvGeom& g);

// y = conv(x, w); bias (nullable) per output channel; stat_sum/sq nullable.
pooch_status launch_conv_fwd(const ConvGeom& g, const float* x, const float* w, float* y, float* stat_sum,
                             float* stat_sq, const float* bias, cudaStream_t st);
pooch_status launch_conv_dgrad(const ConvGeom& g, const float* dy, const float* wt, float* dx, bool accumulate,
                               cudaStream_t st);
size_t conv_wgrad_ws_bytes(const ConvGeom& g);
pooch_status launch_conv_wgrad(const ConvGeom& g, const float* x, const float* dy, float* dw, float* ws,
                               size_t ws_bytes, cudaStream_t st);
// number of M-tiles of the forward pass = rows of its BN partial-sum arrays
int conv_stat_tiles(const ConvGeom& g);
inline int conv_mtiles(const ConvGeom& g) { return conv_stat_tiles(g); }

}  // namespace pooch
