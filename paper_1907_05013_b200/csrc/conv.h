// conv.h -- host launchers of the tensor-core implicit-GEMM kernels (igemm.cuh).
#pragma once
#include <cuda_runtime.h>

#include "../../include/pooch.h"

namespace pooch {

struct ConvGeom {
  int N, H, W, C, K, R, S, stride, pad, Ho, Wo;
  int prec = 0;  // 0: TF32 (one MMA per k-step), 1: 3xTF32 split (fp32-faithful)
  // 3D (D > 0): NDHWC with N = 1, cubic kernel (T = R taps along depth); Do = output depth
  int D = 0, Do = 0;
  // two-source input: x = concat_c(x0 [.., C1], x1 [.., C - C1]); 0 = one source
  int C1 = 0;
  // grouped convolution (ResNeXt; gconv.cu): groups > 1, C == K, C / groups in {4, 8, 16, 32}
  int groups = 1;
  // 3D: stride along depth (0 = stride); ResNeXt-101 (3D)'s stem strides (1, 2, 2)
  int stride_d = 0;
  bool is3d() const { return D > 0; }
  int sd() const { return D > 0 ? (stride_d > 0 ? stride_d : stride) : 1; }
  // 3D: padding along depth (-1 = pad); the divided layers (divide.cu) run depth slabs whose halo
  // rows are real or zero-filled rows, so their sub-convolutions pad only H and W
  int pad_d = -1;
  int pd() const { return D > 0 ? (pad_d >= 0 ? pad_d : pad) : 0; }
  int T() const { return D > 0 ? R : 1; }
};
ConvGeom conv_geom(const pooch_conv_desc& d);
bool conv_shape_ok(const ConvGeom& g);

// y = conv(x, w); bias (nullable) per output channel; stat_sum/sq nullable.
// xf_scale / xf_shift (nullable): the operand is relu(scale[c] * x + shift[c]) (BN-ReLU on load)
// relu: the epilogue applies max(v, 0) after the bias (y = relu(conv(x, w) + b)).
pooch_status launch_conv_fwd(const ConvGeom& g, const float* x, const float* w, float* y, float* stat_sum,
                             float* stat_sq, const float* bias, cudaStream_t st, const float* x1 = nullptr,
                             const float* xf_scale = nullptr, const float* xf_shift = nullptr, bool relu = false);
// dx (and, two-source, dx1 for channels [C1, C)); accumulate / accumulate1 per destination
pooch_status launch_conv_dgrad(const ConvGeom& g, const float* dy, const float* wt, float* dx, bool accumulate,
                               cudaStream_t st, float* dx1 = nullptr, bool accumulate1 = false);
size_t conv_wgrad_ws_bytes(const ConvGeom& g);
pooch_status launch_conv_wgrad(const ConvGeom& g, const float* x, const float* dy, float* dw, float* ws,
                               size_t ws_bytes, cudaStream_t st, const float* x1 = nullptr,
                               const float* xf_scale = nullptr, const float* xf_shift = nullptr);
// number of M-tiles of the forward pass = rows of its BN partial-sum arrays
int conv_stat_tiles(const ConvGeom& g);
inline int conv_mtiles(const ConvGeom& g) { return conv_stat_tiles(g); }

// grouped 3D convolution on the CUDA cores (gconv.cu); the launch_conv_* entry points dispatch
// to these when g.groups > 1. dgrad reads the weights in their own [K][taps][C/groups] layout.
bool gconv_shape_ok(const ConvGeom& g);
int gconv_stat_tiles(const ConvGeom& g);
size_t gconv_wgrad_ws_bytes(const ConvGeom& g);
pooch_status gconv_fwd(const ConvGeom& g, const float* x, const float* w, float* y, float* stat_sum,
                       float* stat_sq, cudaStream_t st);
pooch_status gconv_dgrad(const ConvGeom& g, const float* dy, const float* w, float* dx, bool accumulate,
                         cudaStream_t st);
pooch_status gconv_wgrad(const ConvGeom& g, const float* x, const float* dy, float* dw, float* ws, size_t ws_bytes,
                         cudaStream_t st);

}  // namespace pooch
