// eltwise.cu -- memory-bound kernels (see eltwise.h). HBM-bound: 128-bit loads/stores,
// grid-stride loops sized to the 148 SMs, fixed-order (deterministic) reductions so that any
// keep / swap / recompute plan reproduces the in-core run bit for bit.
#include <algorithm>
#include <cmath>

#include "common.h"
#include "eltwise.h"

namespace pooch {

namespace {

constexpr int kSMs = 148;

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float f4get(const float4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

int grid_for(int64_t n, int per_block, int max_blocks = kSMs * 8) {
  int64_t b = (n + per_block - 1) / per_block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, max_blocks));
}

// ------------------------------------------------------------------ BN finalize
constexpr int kFinRows = 256;  // row-chunks of the tile partials

__global__ void bn_fin_partial_kernel(const float* __restrict__ ts, const float* __restrict__ tq, int tiles, int C,
                                      double* __restrict__ part) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  int chunk = blockIdx.y;
  if (c >= C) return;
  int per = (tiles + kFinRows - 1) / kFinRows;
  int t0 = chunk * per, t1 = min(tiles, t0 + per);
  double s = 0, q = 0;
  for (int t = t0; t < t1; ++t) {
    s += (double)ts[(size_t)t * C + c];
    q += (double)tq[(size_t)t * C + c];
  }
  part[(size_t)chunk * C + c] = s;
  part[(size_t)(kFinRows + chunk) * C + c] = q;
}

// 32 channels per block, kFinWarps warps stride the rows; fixed-order combine (deterministic)
constexpr int kFinWarps = 32;
__global__ void __launch_bounds__(kFinWarps * 32) bn_fin_final_kernel(const double* __restrict__ part, int C, double count, const float* gamma,
                                    const float* beta, float* mean, float* invstd, float* scale, float* shift) {
  __shared__ double sh[2][kFinWarps][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  double s = 0, q = 0;
  if (c < C) {
#pragma unroll 4
    for (int r = w; r < kFinRows; r += kFinWarps) {
      s += part[(size_t)r * C + c];
      q += part[(size_t)(kFinRows + r) * C + c];
    }
  }
  sh[0][w][lane] = s;
  sh[1][w][lane] = q;
  __syncthreads();
  if (w == 0 && c < C) {
    s = 0;
    q = 0;
    for (int k = 0; k < kFinWarps; ++k) {
      s += sh[0][k][lane];
      q += sh[1][k][lane];
    }
    double mu = s / count;
    double var = q / count - mu * mu;
    if (var < 0) var = 0;
    float is = (float)(1.0 / sqrt(var + 1e-5));
    float m = (float)mu;
    mean[c] = m;
    invstd[c] = is;
    float sc = gamma[c] * is;
    scale[c] = sc;
    shift[c] = __fsub_rn(beta[c], __fmul_rn(m, sc));
  }
}

// ------------------------------------------------------------------ BN apply (+add) + ReLU
template <int MODE>
__device__ __forceinline__ float pre_act(float a, float sa, float ta, float b, float sb, float tb) {
  float v = __fmaf_rn(a, sa, ta);
  if (MODE == 1) v = __fadd_rn(v, __fmaf_rn(b, sb, tb));
  if (MODE == 2) v = __fadd_rn(v, b);
  return v;
}

template <int MODE>
__global__ void bn_apply_kernel(const float* __restrict__ a, const float* __restrict__ sa, const float* __restrict__ ta,
                                const float* __restrict__ b, const float* __restrict__ sb,
                                const float* __restrict__ tb, float* __restrict__ y, int64_t n4, int C4) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int cstep = (int)(stride % C4);
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int cg = (int)(i % C4);  // channel group, advanced incrementally (no 64-bit modulo per element)
  auto one = [&](int64_t k, int c, const float4& av, const float4& bv) {
    const float4 s1 = ld4(sa + c), t1 = ld4(ta + c);
    float4 s2 = make_float4(0, 0, 0, 0), t2 = s2;
    if (MODE == 1) {
      s2 = ld4(sb + c);
      t2 = ld4(tb + c);
    }
    float4 o;
    o.x = fmaxf(pre_act<MODE>(av.x, s1.x, t1.x, bv.x, s2.x, t2.x), 0.f);
    o.y = fmaxf(pre_act<MODE>(av.y, s1.y, t1.y, bv.y, s2.y, t2.y), 0.f);
    o.z = fmaxf(pre_act<MODE>(av.z, s1.z, t1.z, bv.z, s2.z, t2.z), 0.f);
    o.w = fmaxf(pre_act<MODE>(av.w, s1.w, t1.w, bv.w, s2.w, t2.w), 0.f);
    st4(y + 4 * k, o);
  };
  // two elements of the grid-stride loop per iteration, both loads issued before either store
  for (; i + stride < n4; i += 2 * stride) {
    const int c0 = cg * 4;
    cg += cstep;
    if (cg >= C4) cg -= C4;
    const int c1 = cg * 4;
    cg += cstep;
    if (cg >= C4) cg -= C4;
    const float4 a0 = ld4(a + 4 * i), a1 = ld4(a + 4 * (i + stride));
    float4 b0 = make_float4(0, 0, 0, 0), b1 = b0;
    if (MODE != 0) {
      b0 = ld4(b + 4 * i);
      b1 = ld4(b + 4 * (i + stride));
    }
    one(i, c0, a0, b0);
    one(i + stride, c1, a1, b1);
  }
  for (; i < n4; i += stride) {
    const int c = cg * 4;
    cg += cstep;
    if (cg >= C4) cg -= C4;
    float4 bv = make_float4(0, 0, 0, 0);
    if (MODE != 0) bv = ld4(b + 4 * i);
    one(i, c, ld4(a + 4 * i), bv);
  }
}

// ------------------------------------------------------------------ BN backward
constexpr int kBwdThreads = 256;
constexpr int kBwdMaxBlocks = 592;

int bwd_blocks(int64_t rows) { return (int)std::max<int64_t>(1, std::min<int64_t>((rows + 63) / 64, kBwdMaxBlocks)); }

// partial layout in ws: [q][block][C] for q in {sum dz, sum dz*xa, sum dz*xb}
template <int MODE, int CGPT>
__global__ void __launch_bounds__(kBwdThreads) bn_bwd_reduce_kernel(BnBwdArgs p, float* __restrict__ part) {
  extern __shared__ float red[];  // [nq][rpi][C]
  const int C = p.C, C4 = C / 4;
  const int tpr = C4 / CGPT;  // threads per row
  const int rpi = kBwdThreads / tpr;
  const int tid = threadIdx.x;
  const int roff = tid / tpr, cg0 = tid % tpr;
  const int64_t per = (p.rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per, r1 = min(p.rows, r0 + per);
  constexpr int NQ = MODE == 1 ? 3 : 2;
  float acc[NQ][CGPT][4];
#pragma unroll
  for (int q = 0; q < NQ; ++q)
#pragma unroll
    for (int j = 0; j < CGPT; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[q][j][e] = 0.f;
  if (roff < rpi) {
#pragma unroll
    for (int j = 0; j < CGPT; ++j) {
      // per-channel parameters: loop-invariant, loaded once
      const int c = 4 * (cg0 + j * tpr);
      const float4 s1 = ld4(p.sa + c), t1 = ld4(p.ta + c), m1 = ld4(p.mean_a + c), i1 = ld4(p.invstd_a + c);
      float4 s2 = make_float4(0, 0, 0, 0), t2 = s2, m2 = s2, i2 = s2;
      if (MODE == 1) {
        s2 = ld4(p.sb + c); t2 = ld4(p.tb + c); m2 = ld4(p.mean_b + c); i2 = ld4(p.invstd_b + c);
      }
      auto row = [&](const float4& av, const float4& g, const float4& bv) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float v = pre_act<MODE>(f4get(av, e), f4get(s1, e), f4get(t1, e), f4get(bv, e), f4get(s2, e), f4get(t2, e));
          float dz = v > 0.f ? f4get(g, e) : 0.f;
          acc[0][j][e] += dz;
          acc[1][j][e] += dz * ((f4get(av, e) - f4get(m1, e)) * f4get(i1, e));
          if (MODE == 1) acc[2 % NQ][j][e] += dz * ((f4get(bv, e) - f4get(m2, e)) * f4get(i2, e));
        }
      };
      int64_t r = r0 + roff;
      // two rows per iteration: all loads first (more bytes in flight), then the same
      // accumulation order as one row at a time
      for (; r + rpi < r1; r += 2 * rpi) {
        const size_t o0 = (size_t)r * C + c, o1 = o0 + (size_t)rpi * C;
        const float4 a0 = ld4(p.a + o0), g0 = ld4(p.gy + o0), a1 = ld4(p.a + o1), g1 = ld4(p.gy + o1);
        float4 b0 = make_float4(0, 0, 0, 0), b1 = b0;
        if (MODE != 0) {
          b0 = ld4(p.b + o0);
          b1 = ld4(p.b + o1);
        }
        row(a0, g0, b0);
        row(a1, g1, b1);
      }
      for (; r < r1; r += rpi) {
        const size_t o0 = (size_t)r * C + c;
        float4 b0 = make_float4(0, 0, 0, 0);
        if (MODE != 0) b0 = ld4(p.b + o0);
        row(ld4(p.a + o0), ld4(p.gy + o0), b0);
      }
    }
  }
  if (roff < rpi) {
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int j = 0; j < CGPT; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) red[((size_t)q * rpi + roff) * C + 4 * (cg0 + j * tpr) + e] = acc[q][j][e];
  }
  __syncthreads();
  for (int c = tid; c < C; c += kBwdThreads) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      float s = 0.f;
      for (int r = 0; r < rpi; ++r) s += red[((size_t)q * rpi + r) * C + c];
      part[((size_t)q * gridDim.x + blockIdx.x) * C + c] = s;
    }
  }
}

// coef layout after the partials: [ka, kb, kc] for BN(a) then BN(b), each [C]
template <int MODE>
__global__ void __launch_bounds__(kFinWarps * 32) bn_bwd_finalize_kernel(BnBwdArgs p, const float* __restrict__ part, int blocks, float* coef) {
  constexpr int NQ = MODE == 1 ? 3 : 2;
  __shared__ double sh[NQ][kFinWarps][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0;
  if (c < p.C) {
    for (int b = w; b < blocks; b += kFinWarps) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) acc[q] += (double)part[((size_t)q * blocks + b) * p.C + c];
    }
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q) sh[q][w][lane] = acc[q];
  __syncthreads();
  if (w != 0 || c >= p.C) return;
  double s[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    double t = 0;
    for (int k = 0; k < kFinWarps; ++k) t += sh[q][k][lane];
    s[q] = t;
  }
  double M = (double)p.rows;
  p.dbeta_a[c] = (float)s[0];
  p.dgamma_a[c] = (float)s[1];
  coef[c] = p.gamma_a[c] * p.invstd_a[c];
  coef[p.C + c] = (float)(s[0] / M);
  coef[2 * p.C + c] = (float)(s[1] / M);
  if (MODE == 1) {
    p.dbeta_b[c] = (float)s[0];
    p.dgamma_b[c] = (float)s[2 % NQ];
    coef[3 * p.C + c] = p.gamma_b[c] * p.invstd_b[c];
    coef[4 * p.C + c] = (float)(s[0] / M);
    coef[5 * p.C + c] = (float)(s[2 % NQ] / M);
  }
}

template <int MODE>
__global__ void bn_bwd_apply_kernel(BnBwdArgs p, const float* __restrict__ coef, int64_t n4) {
  const int C = p.C, C4 = C / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int cstep = (int)(stride % C4);
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int cg = (int)(i % C4);
  for (; i < n4; i += stride) {
    int c = cg * 4;
    cg += cstep;
    if (cg >= C4) cg -= C4;
    size_t off = 4 * (size_t)i;
    float4 av = ld4(p.a + off), g = ld4(p.gy + off);
    float4 s1 = ld4(p.sa + c), t1 = ld4(p.ta + c), m1 = ld4(p.mean_a + c), i1 = ld4(p.invstd_a + c);
    float4 ka = ld4(coef + c), kb = ld4(coef + C + c), kc = ld4(coef + 2 * C + c);
    float4 bv = make_float4(0, 0, 0, 0), s2 = bv, t2 = bv, m2 = bv, i2 = bv, la = bv, lb = bv, lc = bv;
    if (MODE != 0) bv = ld4(p.b + off);
    if (MODE == 1) {
      s2 = ld4(p.sb + c); t2 = ld4(p.tb + c); m2 = ld4(p.mean_b + c); i2 = ld4(p.invstd_b + c);
      la = ld4(coef + 3 * C + c); lb = ld4(coef + 4 * C + c); lc = ld4(coef + 5 * C + c);
    }
    float oa[4], ob[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float v = pre_act<MODE>(f4get(av, e), f4get(s1, e), f4get(t1, e), f4get(bv, e), f4get(s2, e), f4get(t2, e));
      float dz = v > 0.f ? f4get(g, e) : 0.f;
      float xa = (f4get(av, e) - f4get(m1, e)) * f4get(i1, e);
      oa[e] = f4get(ka, e) * (dz - f4get(kb, e) - xa * f4get(kc, e));
      if (MODE == 1) {
        float xb = (f4get(bv, e) - f4get(m2, e)) * f4get(i2, e);
        ob[e] = f4get(la, e) * (dz - f4get(lb, e) - xb * f4get(lc, e));
      } else {
        ob[e] = dz;
      }
    }
    st4(p.ga + off, make_float4(oa[0], oa[1], oa[2], oa[3]));
    if (MODE == 1) st4(p.gb + off, make_float4(ob[0], ob[1], ob[2], ob[3]));
    if (MODE == 2) {
      float4 o = make_float4(ob[0], ob[1], ob[2], ob[3]);
      if (p.gb_accumulate) {
        float4 q = ld4(p.gb + off);
        o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
      }
      st4(p.gb + off, o);
    }
  }
}

// ------------------------------------------------------------------ pooling
// 2D max-pool. One block per output row (n, ho) (backward: per input row (n, h)); threads
// stride the row's (w, 4-channel group) pairs, so all index math is 32-bit and division-free
// except one per element by C4 (a power of two in every network here).
// K, S > 0: window / stride fixed at compile time (ResNet's 3x3 / 2; the loops unroll and the
// divisions by the stride become shifts); 0: runtime k, s. cs >= 0: C4 = 1 << cs (j / C4 and
// j % C4 are a shift and a mask), else a division.
__device__ __forceinline__ void split_j(int j, int C4, int cs, int& c4, int& q) {
  if (cs >= 0) {
    c4 = j & (C4 - 1);
    q = j >> cs;
  } else {
    c4 = j % C4;
    q = j / C4;
  }
}

template <int K, int S>
__global__ void maxpool_fwd_kernel(const float* __restrict__ x, float* __restrict__ y, int N, int H, int W, int C4,
                                   int cs, int k_, int s_, int p, int Ho, int Wo) {
  const int k = K ? K : k_, s = S ? S : s_;
  const int ho = blockIdx.x % Ho, n = blockIdx.x / Ho;
  const float4* xn = reinterpret_cast<const float4*>(x) + (size_t)n * H * W * C4;
  float4* yr = reinterpret_cast<float4*>(y) + ((size_t)n * Ho + ho) * Wo * C4;
  const int h0 = ho * s - p;
  for (int j = threadIdx.x; j < Wo * C4; j += blockDim.x) {
    int c4, wo;
    split_j(j, C4, cs, c4, wo);
    const int w0 = wo * s - p;
    float4 m = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
#pragma unroll
    for (int u = 0; u < (K ? K : 8); ++u) {
      if (!K && u >= k) break;
      const int h = h0 + u;
      if (h < 0 || h >= H) continue;
#pragma unroll
      for (int v = 0; v < (K ? K : 8); ++v) {
        if (!K && v >= k) break;
        const int w = w0 + v;
        if (w < 0 || w >= W) continue;
        float4 q = __ldg(xn + (h * W + w) * C4 + c4);
        m.x = fmaxf(m.x, q.x); m.y = fmaxf(m.y, q.y); m.z = fmaxf(m.z, q.z); m.w = fmaxf(m.w, q.w);
      }
    }
    yr[j] = m;
  }
}

// window argmax (first maximum in row-major order; -inf padding never wins) -> u*k+v per channel
template <int K, int S>
__global__ void maxpool_arg_kernel(const float* __restrict__ x, uint8_t* __restrict__ arg, int N, int H, int W,
                                   int C4, int cs, int k_, int s_, int p, int Ho, int Wo) {
  const int k = K ? K : k_, s = S ? S : s_;
  const int ho = blockIdx.x % Ho, n = blockIdx.x / Ho;
  const float4* xn = reinterpret_cast<const float4*>(x) + (size_t)n * H * W * C4;
  uchar4* ar = reinterpret_cast<uchar4*>(arg) + ((size_t)n * Ho + ho) * Wo * C4;
  const int h0 = ho * s - p;
  for (int j = threadIdx.x; j < Wo * C4; j += blockDim.x) {
    int c4, wo;
    split_j(j, C4, cs, c4, wo);
    const int w0 = wo * s - p;
    float best[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    uint8_t a[4] = {255, 255, 255, 255};
#pragma unroll
    for (int u = 0; u < (K ? K : 8); ++u) {
      if (!K && u >= k) break;
      const int h = h0 + u;
      if (h < 0 || h >= H) continue;
#pragma unroll
      for (int v = 0; v < (K ? K : 8); ++v) {
        if (!K && v >= k) break;
        const int w = w0 + v;
        if (w < 0 || w >= W) continue;
        float4 q = __ldg(xn + (h * W + w) * C4 + c4);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float val = f4get(q, e);
          if (a[e] == 255 || val > best[e]) {
            best[e] = val;
            a[e] = (uint8_t)(u * k + v);
          }
        }
      }
    }
    ar[j] = make_uchar4(a[0], a[1], a[2], a[3]);
  }
}

template <int K, int S>
__global__ void maxpool_bwd_kernel(const uint8_t* __restrict__ arg, const float* __restrict__ gy,
                                   float* __restrict__ gx, int N, int H, int W, int C4, int cs, int k_, int s_, int p,
                                   int Ho, int Wo) {
  const int k = K ? K : k_, s = S ? S : s_;
  const int h = blockIdx.x % H, n = blockIdx.x / H;
  const uchar4* an = reinterpret_cast<const uchar4*>(arg) + (size_t)n * Ho * Wo * C4;
  const float4* gn = reinterpret_cast<const float4*>(gy) + (size_t)n * Ho * Wo * C4;
  float4* gr = reinterpret_cast<float4*>(gx) + ((size_t)n * H + h) * W * C4;
  const int ho_lo = max(0, (h + p - k + s) / s), ho_hi = min(Ho - 1, (h + p) / s);
  for (int j = threadIdx.x; j < W * C4; j += blockDim.x) {
    int c4, w;
    split_j(j, C4, cs, c4, w);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    const int wo_lo = max(0, (w + p - k + s) / s), wo_hi = min(Wo - 1, (w + p) / s);
    for (int ho = ho_lo; ho <= ho_hi; ++ho) {
      const int u = h - (ho * s - p);
      if (u < 0 || u >= k) continue;
      for (int wo = wo_lo; wo <= wo_hi; ++wo) {
        const int v = w - (wo * s - p);
        if (v < 0 || v >= k) continue;
        const int o = (ho * Wo + wo) * C4 + c4;
        uchar4 a = an[o];
        float4 g = __ldg(gn + o);
        const int me = u * k + v;
        if (a.x == me) acc[0] += g.x;
        if (a.y == me) acc[1] += g.y;
        if (a.z == me) acc[2] += g.z;
        if (a.w == me) acc[3] += g.w;
      }
    }
    gr[j] = make_float4(acc[0], acc[1], acc[2], acc[3]);
  }
}

// 3D max-pool, k2 s2 p0 (the U-Net's down-sampling): the 2x2x2 windows tile the input, so the
// backward pass is a gather -- each thread owns one output voxel x 4 channels, re-reads its
// window and routes the gradient to the FIRST maximum in (u, v, t) row-major order.
__global__ void maxpool3d_fwd_kernel(const float* __restrict__ x, float* __restrict__ y, int D, int H, int W, int C4) {
  const int Do = D / 2, Ho = H / 2, Wo = W / 2;
  const int64_t total = (int64_t)Do * Ho * Wo * C4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c4 = (int)(i % C4);
    int64_t t = i / C4;
    const int wo = (int)(t % Wo);
    t /= Wo;
    const int ho = (int)(t % Ho);
    const int dz = (int)(t / Ho);
    float4 m = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    for (int u = 0; u < 2; ++u)
      for (int v = 0; v < 2; ++v)
        for (int w = 0; w < 2; ++w) {
          const float4 q = ld4(x + ((((size_t)(2 * dz + u) * H + 2 * ho + v) * W + 2 * wo + w) * C4 + c4) * 4);
          m.x = fmaxf(m.x, q.x); m.y = fmaxf(m.y, q.y); m.z = fmaxf(m.z, q.z); m.w = fmaxf(m.w, q.w);
        }
    st4(y + 4 * i, m);
  }
}

__global__ void maxpool3d_bwd_kernel(const float* __restrict__ x, const float* __restrict__ gy, float* __restrict__ gx,
                                     int D, int H, int W, int C4, int accumulate) {
  const int Do = D / 2, Ho = H / 2, Wo = W / 2;
  const int64_t total = (int64_t)Do * Ho * Wo * C4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c4 = (int)(i % C4);
    int64_t t = i / C4;
    const int wo = (int)(t % Wo);
    t /= Wo;
    const int ho = (int)(t % Ho);
    const int dz = (int)(t / Ho);
    float best[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    int arg[4] = {-1, -1, -1, -1};
    for (int e = 0; e < 8; ++e) {
      const int u = e >> 2, v = (e >> 1) & 1, w = e & 1;
      const float4 q = ld4(x + ((((size_t)(2 * dz + u) * H + 2 * ho + v) * W + 2 * wo + w) * C4 + c4) * 4);
      const float qa[4] = {q.x, q.y, q.z, q.w};
      for (int j = 0; j < 4; ++j)
        if (qa[j] > best[j]) {  // strict: the first maximum wins
          best[j] = qa[j];
          arg[j] = e;
        }
    }
    const float4 g = ld4(gy + 4 * i);
    const float ga[4] = {g.x, g.y, g.z, g.w};
    for (int e = 0; e < 8; ++e) {
      const int u = e >> 2, v = (e >> 1) & 1, w = e & 1;
      float o[4];
      for (int j = 0; j < 4; ++j) o[j] = arg[j] == e ? ga[j] : 0.f;
      float* dst = gx + ((((size_t)(2 * dz + u) * H + 2 * ho + v) * W + 2 * wo + w) * C4 + c4) * 4;
      if (accumulate) {  // windows do not overlap: this thread is the only writer of these elements
        const float4 q = ld4(dst);
        o[0] += q.x; o[1] += q.y; o[2] += q.z; o[3] += q.w;
      }
      st4(dst, make_float4(o[0], o[1], o[2], o[3]));
    }
  }
}

__global__ void avgpool_fwd_kernel(const float* __restrict__ x, float* __restrict__ y, int HW, int C4) {
  int n = blockIdx.y;
  int c4 = blockIdx.x * blockDim.x + threadIdx.x;
  if (c4 >= C4) return;
  float4 s = make_float4(0, 0, 0, 0);
  for (int i = 0; i < HW; ++i) {
    float4 q = ld4(x + ((size_t)n * HW + i) * C4 * 4 + 4 * c4);
    s.x += q.x; s.y += q.y; s.z += q.z; s.w += q.w;
  }
  float inv = 1.0f / (float)HW;
  st4(y + ((size_t)n * C4 + c4) * 4, make_float4(s.x * inv, s.y * inv, s.z * inv, s.w * inv));
}

__global__ void avgpool_bwd_kernel(const float* __restrict__ gy, float* __restrict__ gx, int64_t n4, int HW, int C4) {
  float inv = 1.0f / (float)HW;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    int c4 = (int)(i % C4);
    int64_t n = i / C4 / HW;
    float4 g = ld4(gy + (n * C4 + c4) * 4);
    st4(gx + 4 * i, make_float4(g.x * inv, g.y * inv, g.z * inv, g.w * inv));
  }
}

// ------------------------------------------------------------------ softmax cross-entropy
__device__ __forceinline__ float warp_max(float v) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void ce_rows_kernel(const float* __restrict__ z, const int32_t* __restrict__ lab, int B, int classes,
                               int ld, float* __restrict__ loss_rows, float* __restrict__ dz, int write_dz) {
  int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x & 31;
  if (row >= B) return;
  const float* zr = z + (size_t)row * ld;
  float m = -INFINITY;
  for (int c = lane; c < classes; c += 32) m = fmaxf(m, zr[c]);
  m = warp_max(m);
  float s = 0.f;
  for (int c = lane; c < classes; c += 32) s += expf(zr[c] - m);
  s = warp_sum(s);
  int t = lab[row];
  if (!write_dz) {
    if (lane == 0) loss_rows[row] = logf(s) + m - zr[t];
    return;
  }
  float invB = 1.0f / (float)B;
  for (int c = lane; c < ld; c += 32) {
    float v = 0.f;
    if (c < classes) v = (expf(zr[c] - m) / s - (c == t ? 1.f : 0.f)) * invB;
    dz[(size_t)row * ld + c] = v;
  }
}

__global__ void mean_kernel(const float* __restrict__ v, int n, float* __restrict__ out) {
  __shared__ double sh[256];
  double s = 0;
  for (int i = threadIdx.x; i < n; i += 256) s += (double)v[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = (float)(sh[0] / n);
}

// Per-row softmax-CE for narrow rows (the voxel head: ld <= 8): one thread per row.
__global__ void ce_rows_narrow_kernel(const float* __restrict__ z, const int32_t* __restrict__ lab, int64_t rows,
                                      int classes, int ld, float* __restrict__ loss_rows, float* __restrict__ dz,
                                      int write_dz) {
  for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < rows;
       row += (int64_t)gridDim.x * blockDim.x) {
    const float* zr = z + (size_t)row * ld;
    float m = -INFINITY;
    for (int c = 0; c < classes; ++c) m = fmaxf(m, zr[c]);
    float s = 0.f;
    for (int c = 0; c < classes; ++c) s += expf(zr[c] - m);
    const int t = lab[row];
    if (!write_dz) {
      loss_rows[row] = logf(s) + m - zr[t];
      continue;
    }
    const float inv = 1.0f / (float)rows;
    for (int c = 0; c < ld; ++c)
      dz[(size_t)row * ld + c] = c < classes ? (expf(zr[c] - m) / s - (c == t ? 1.f : 0.f)) * inv : 0.f;
  }
}

// Deterministic column sums of a tall, narrow matrix m [rows][ld] (ld <= 8): block b sums its
// row range in a fixed thread / warp order (fp64), then one block adds the partials in order.
constexpr int kColsumBlocks = 592;
__global__ void colsum_partial_kernel(const float* __restrict__ m, int64_t rows, int ld, double* __restrict__ part) {
  __shared__ double sh[8][8];
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
  for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x)
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c < ld) acc[c] += (double)m[(size_t)r * ld + c];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < 8; ++c)
    for (int o = 16; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
  if (lane == 0)
    for (int c = 0; c < 8; ++c) sh[w][c] = acc[c];
  __syncthreads();
  if (threadIdx.x < ld) {
    double s = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += sh[k][threadIdx.x];
    part[(size_t)blockIdx.x * ld + threadIdx.x] = s;
  }
}

// out[c] = sum_b part[b][c] * scale, in block order
__global__ void colsum_final_kernel(const double* __restrict__ part, int blocks, int ld, double scale,
                                    float* __restrict__ out) {
  const int c = threadIdx.x;
  if (c >= ld) return;
  double s = 0;
  for (int b = 0; b < blocks; ++b) s += part[(size_t)b * ld + c];
  out[c] = (float)(s * scale);
}

__global__ void colsum_kernel(const float* __restrict__ m, int rows, int ld, float* __restrict__ out) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ld) return;
  float s = 0.f;
  for (int r = 0; r < rows; ++r) s += m[(size_t)r * ld + c];
  out[c] = s;
}

// ------------------------------------------------------------------ SGD, transpose
__global__ void sgd_kernel(float* __restrict__ w, float* __restrict__ v, const float* __restrict__ g, int64_t n4,
                           float lr, float mu, float scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 wv = ld4(w + 4 * i), vv = ld4(v + 4 * i), gv = ld4(g + 4 * i);
    vv.x = mu * vv.x + scale * gv.x; vv.y = mu * vv.y + scale * gv.y;
    vv.z = mu * vv.z + scale * gv.z; vv.w = mu * vv.w + scale * gv.w;
    wv.x -= lr * vv.x; wv.y -= lr * vv.y; wv.z -= lr * vv.z; wv.w -= lr * vv.w;
    st4(v + 4 * i, vv);
    st4(w + 4 * i, wv);
  }
}

__global__ void sgd_tail_kernel(float* w, float* v, const float* g, int64_t start, int64_t n, float lr, float mu,
                                float scale) {
  int64_t i = start + threadIdx.x;
  if (i < n) {
    v[i] = mu * v[i] + scale * g[i];
    w[i] -= lr * v[i];
  }
}

__global__ void transpose_kernel(const float* __restrict__ w, float* __restrict__ wt, int K, int RS, int C) {
  __shared__ float tile[32][33];
  int rs = blockIdx.z;
  int c0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int k = k0 + i, c = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (k < K && c < C) ? w[((size_t)k * RS + rs) * C + c] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int c = c0 + i, k = k0 + threadIdx.x;
    if (c < C && k < K) wt[((size_t)c * RS + rs) * K + k] = tile[threadIdx.x][i];
  }
}

}  // namespace

// ======================================================================== launchers
size_t bn_finalize_ws_bytes(int C) { return (size_t)2 * kFinRows * C * sizeof(double); }

pooch_status bn_finalize(const float* ts, const float* tq, int tiles, int C, int64_t count, const float* gamma,
                         const float* beta, float* mean, float* invstd, float* scale, float* shift, double* ws,
                         cudaStream_t st) {
  dim3 g1((C + 127) / 128, kFinRows);
  count_launch();
  bn_fin_partial_kernel<<<g1, 128, 0, st>>>(ts, tq, tiles, C, ws);
  count_launch();
  bn_fin_final_kernel<<<(C + 31) / 32, kFinWarps * 32, 0, st>>>(ws, C, (double)count, gamma, beta, mean, invstd, scale, shift);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

pooch_status bn_apply_relu(const float* a, const float* sa, const float* ta, const float* b, const float* sb,
                           const float* tb, int mode, float* y, int64_t rows, int C, cudaStream_t st) {
  int64_t n4 = rows * C / 4;
  int grid = grid_for(n4, 256);
  if (mode == 0) { count_launch(); bn_apply_kernel<0><<<grid, 256, 0, st>>>(a, sa, ta, b, sb, tb, y, n4, C / 4); }
  else if (mode == 1) { count_launch(); bn_apply_kernel<1><<<grid, 256, 0, st>>>(a, sa, ta, b, sb, tb, y, n4, C / 4); }
  else { count_launch(); bn_apply_kernel<2><<<grid, 256, 0, st>>>(a, sa, ta, b, sb, tb, y, n4, C / 4); }
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

size_t bn_bwd_ws_bytes(int C) { return ((size_t)3 * kBwdMaxBlocks * C + 6 * (size_t)C) * sizeof(float); }

template <int MODE>
static pooch_status bn_bwd_mode(const BnBwdArgs& a, float* ws, cudaStream_t st) {
  const int C = a.C, C4 = C / 4;
  int blocks = bwd_blocks(a.rows);
  int cgpt = C4 > kBwdThreads ? C4 / kBwdThreads : 1;
  constexpr int NQ = MODE == 1 ? 3 : 2;
  int tpr = C4 / cgpt;
  int rpi = kBwdThreads / tpr;
  size_t smem = (size_t)NQ * rpi * C * sizeof(float);
  float* coef = ws + (size_t)3 * kBwdMaxBlocks * C;
  if (cgpt == 1) {
    if (smem > 48 * 1024) POOCH_CUDA(cudaFuncSetAttribute(bn_bwd_reduce_kernel<MODE, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    count_launch();
    bn_bwd_reduce_kernel<MODE, 1><<<blocks, kBwdThreads, smem, st>>>(a, ws);
  } else if (cgpt == 2) {
    if (smem > 48 * 1024) POOCH_CUDA(cudaFuncSetAttribute(bn_bwd_reduce_kernel<MODE, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    count_launch();
    bn_bwd_reduce_kernel<MODE, 2><<<blocks, kBwdThreads, smem, st>>>(a, ws);
  } else {
    return fail(POOCH_EUSAGE, "BN backward supports C <= 2048 (C = %d)", C);
  }
  count_launch();
  bn_bwd_finalize_kernel<MODE><<<(C + 31) / 32, kFinWarps * 32, 0, st>>>(a, ws, blocks, coef);
  int64_t n4 = a.rows * C / 4;
  count_launch();
  bn_bwd_apply_kernel<MODE><<<grid_for(n4, 256), 256, 0, st>>>(a, coef, n4);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

// ---- BN-ReLU backward in pieces (divided layers, divide.cu): per-chunk partial sums accumulated
// in fp64 across chunks in order, one finalize, per-chunk apply
namespace {
__global__ void acc_partials_kernel(const float* __restrict__ part, int blocks, int C, int nq, double* __restrict__ acc) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  for (int q = 0; q < nq; ++q) {
    double s = 0;
    for (int b = 0; b < blocks; ++b) s += (double)part[((size_t)q * blocks + b) * C + c];
    acc[(size_t)q * C + c] += s;
  }
}

__global__ void bn_bwd_finalize_sums_kernel(BnBwdArgs p, const double* __restrict__ acc, double M, float* coef) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= p.C) return;
  p.dbeta_a[c] = (float)acc[c];
  p.dgamma_a[c] = (float)acc[p.C + c];
  coef[c] = p.gamma_a[c] * p.invstd_a[c];
  coef[p.C + c] = (float)(acc[c] / M);
  coef[2 * p.C + c] = (float)(acc[p.C + c] / M);
}

__global__ void acc_tiles_kernel(const float* __restrict__ ts, const float* __restrict__ tq, int tiles, int C,
                                 double* __restrict__ acc) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double s = 0, q = 0;
  for (int t = 0; t < tiles; ++t) {
    s += (double)ts[(size_t)t * C + c];
    q += (double)tq[(size_t)t * C + c];
  }
  acc[c] += s;
  acc[C + c] += q;
}

__global__ void bn_finalize_sums_kernel(const double* __restrict__ acc, int C, double count, const float* gamma,
                                        const float* beta, float* mean, float* invstd, float* scale, float* shift) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double mu = acc[c] / count;
  double var = acc[C + c] / count - mu * mu;
  if (var < 0) var = 0;
  const float is = (float)(1.0 / sqrt(var + 1e-5));
  const float m = (float)mu;
  mean[c] = m;
  invstd[c] = is;
  const float sc = gamma[c] * is;
  scale[c] = sc;
  shift[c] = __fsub_rn(beta[c], __fmul_rn(m, sc));
}
}  // namespace

size_t bn_relu_bwd_partial_ws_bytes(int64_t rows, int C) { return (size_t)2 * bwd_blocks(rows) * C * sizeof(float); }

pooch_status bn_relu_bwd_partial(const BnBwdArgs& a, float* ws, double* acc, cudaStream_t st) {
  const int C = a.C, C4 = C / 4;
  if (a.mode != 0 || C % 4 || C > 2048) return fail(POOCH_EUSAGE, "divided BN-ReLU backward: mode 0, C %% 4 == 0, C <= 2048");
  const int blocks = bwd_blocks(a.rows);
  const int cgpt = C4 > kBwdThreads ? C4 / kBwdThreads : 1;
  const int rpi = kBwdThreads / (C4 / cgpt);
  const size_t smem = (size_t)2 * rpi * C * sizeof(float);
  count_launch();
  if (cgpt == 1) {
    if (smem > 48 * 1024) POOCH_CUDA(cudaFuncSetAttribute(bn_bwd_reduce_kernel<0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    bn_bwd_reduce_kernel<0, 1><<<blocks, kBwdThreads, smem, st>>>(a, ws);
  } else {
    if (smem > 48 * 1024) POOCH_CUDA(cudaFuncSetAttribute(bn_bwd_reduce_kernel<0, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    bn_bwd_reduce_kernel<0, 2><<<blocks, kBwdThreads, smem, st>>>(a, ws);
  }
  count_launch();
  acc_partials_kernel<<<(C + 127) / 128, 128, 0, st>>>(ws, blocks, C, 2, acc);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

pooch_status bn_relu_bwd_finalize(const BnBwdArgs& a, const double* acc, int64_t total_rows, float* coef,
                                  cudaStream_t st) {
  count_launch();
  bn_bwd_finalize_sums_kernel<<<(a.C + 127) / 128, 128, 0, st>>>(a, acc, (double)total_rows, coef);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

pooch_status bn_relu_bwd_apply(const BnBwdArgs& a, const float* coef, cudaStream_t st) {
  const int64_t n4 = a.rows * a.C / 4;
  count_launch();
  bn_bwd_apply_kernel<0><<<grid_for(n4, 256), 256, 0, st>>>(a, coef, n4);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

pooch_status bn_acc_tiles(const float* ts, const float* tq, int tiles, int C, double* acc, cudaStream_t st) {
  count_launch();
  acc_tiles_kernel<<<(C + 127) / 128, 128, 0, st>>>(ts, tq, tiles, C, acc);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

pooch_status bn_finalize_sums(const double* acc, int C, int64_t count, const float* gamma, const float* beta,
                              float* mean, float* invstd, float* scale, float* shift, cudaStream_t st) {
  count_launch();
  bn_finalize_sums_kernel<<<(C + 127) / 128, 128, 0, st>>>(acc, C, (double)count, gamma, beta, mean, invstd, scale,
                                                           shift);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

pooch_status bn_bwd(const BnBwdArgs& a, float* ws, cudaStream_t st) {
  if (a.C % 4 != 0 || a.C > 2048 || a.C < 4) return fail(POOCH_EUSAGE, "BN backward: bad C %d", a.C);
  if (a.mode == 0) return bn_bwd_mode<0>(a, ws, st);
  if (a.mode == 1) return bn_bwd_mode<1>(a, ws, st);
  return bn_bwd_mode<2>(a, ws, st);
}

pooch_status maxpool_fwd(const float* x, float* y, int N, int H, int W, int C, int k, int s, int p, int Ho, int Wo,
                         cudaStream_t st) {
  if (C % 4 || (int64_t)H * W * C >= (1LL << 31)) return fail(POOCH_EUSAGE, "max-pool: C %% 4 != 0 or image too large");
  if (k > 8) return fail(POOCH_EUSAGE, "max-pool window > 8");
  const int C4 = C / 4, cs = (C4 & (C4 - 1)) == 0 ? __builtin_ctz(C4) : -1;
  count_launch();
  if (k == 3 && s == 2) maxpool_fwd_kernel<3, 2><<<N * Ho, 256, 0, st>>>(x, y, N, H, W, C4, cs, k, s, p, Ho, Wo);
  else if (k == 2 && s == 2) maxpool_fwd_kernel<2, 2><<<N * Ho, 256, 0, st>>>(x, y, N, H, W, C4, cs, k, s, p, Ho, Wo);
  else maxpool_fwd_kernel<0, 0><<<N * Ho, 256, 0, st>>>(x, y, N, H, W, C4, cs, k, s, p, Ho, Wo);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

pooch_status maxpool_bwd(const float* x, const float* gy, float* gx, uint8_t* arg_ws, int N, int H, int W, int C,
                         int k, int s, int p, int Ho, int Wo, cudaStream_t st) {
  if (C % 4 || (int64_t)H * W * C >= (1LL << 31)) return fail(POOCH_EUSAGE, "max-pool: C %% 4 != 0 or image too large");
  if (k > 8) return fail(POOCH_EUSAGE, "max-pool window > 8");
  const int C4 = C / 4, cs = (C4 & (C4 - 1)) == 0 ? __builtin_ctz(C4) : -1;
  count_launch();
  count_launch();
  if (k == 3 && s == 2) {
    maxpool_arg_kernel<3, 2><<<N * Ho, 256, 0, st>>>(x, arg_ws, N, H, W, C4, cs, k, s, p, Ho, Wo);
    maxpool_bwd_kernel<3, 2><<<N * H, 256, 0, st>>>(arg_ws, gy, gx, N, H, W, C4, cs, k, s, p, Ho, Wo);
  } else if (k == 2 && s == 2) {
    maxpool_arg_kernel<2, 2><<<N * Ho, 256, 0, st>>>(x, arg_ws, N, H, W, C4, cs, k, s, p, Ho, Wo);
    maxpool_bwd_kernel<2, 2><<<N * H, 256, 0, st>>>(arg_ws, gy, gx, N, H, W, C4, cs, k, s, p, Ho, Wo);
  } else {
    maxpool_arg_kernel<0, 0><<<N * Ho, 256, 0, st>>>(x, arg_ws, N, H, W, C4, cs, k, s, p, Ho, Wo);
    maxpool_bwd_kernel<0, 0><<<N * H, 256, 0, st>>>(arg_ws, gy, gx, N, H, W, C4, cs, k, s, p, Ho, Wo);
  }
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

// General 3D max-pool (k, s, p; -inf padding): ResNeXt-101 (3D)'s 3^3 / 2 pad 1. Windows overlap,
// so the backward pass records each output's first-maximum window index (uint8, (u*k+v)*k+t)
// and then gathers on the INPUT side: every input voxel sums, in (od, oh, ow) order, the dy of
// the windows that cover it and chose it -- one writer per element, deterministic.
namespace {

struct Pool3 {
  int D, H, W, C4, Do, Ho, Wo, k, s, p;
};

__global__ void maxpool3d_gen_fwd_kernel(const float* __restrict__ x, float* __restrict__ y,  // y / arg nullable
                                         uchar4* __restrict__ arg, Pool3 q) {
  const int64_t total = (int64_t)q.Do * q.Ho * q.Wo * q.C4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c4 = (int)(i % q.C4);
    int64_t t = i / q.C4;
    const int wo = (int)(t % q.Wo);
    t /= q.Wo;
    const int ho = (int)(t % q.Ho);
    const int dz = (int)(t / q.Ho);
    float best[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    int a[4] = {0, 0, 0, 0};
    for (int u = 0; u < q.k; ++u) {
      const int zi = dz * q.s - q.p + u;
      if (zi < 0 || zi >= q.D) continue;
      for (int v = 0; v < q.k; ++v) {
        const int hi = ho * q.s - q.p + v;
        if (hi < 0 || hi >= q.H) continue;
        for (int w = 0; w < q.k; ++w) {
          const int wi = wo * q.s - q.p + w;
          if (wi < 0 || wi >= q.W) continue;
          const float4 v4 = ld4(x + ((((int64_t)zi * q.H + hi) * q.W + wi) * q.C4 + c4) * 4);
          const float va[4] = {v4.x, v4.y, v4.z, v4.w};
          const int e = (u * q.k + v) * q.k + w;
          for (int j = 0; j < 4; ++j)
            if (va[j] > best[j]) {  // strict: the first maximum wins
              best[j] = va[j];
              a[j] = e;
            }
        }
      }
    }
    if (y) st4(y + 4 * i, make_float4(best[0], best[1], best[2], best[3]));
    if (arg) arg[i] = make_uchar4((unsigned char)a[0], (unsigned char)a[1], (unsigned char)a[2], (unsigned char)a[3]);
  }
}

__global__ void maxpool3d_gen_bwd_kernel(const uchar4* __restrict__ arg, const float* __restrict__ gy,
                                         float* __restrict__ gx, Pool3 q, int accumulate) {
  const int64_t total = (int64_t)q.D * q.H * q.W * q.C4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c4 = (int)(i % q.C4);
    int64_t t = i / q.C4;
    const int wi = (int)(t % q.W);
    t /= q.W;
    const int hi = (int)(t % q.H);
    const int zi = (int)(t / q.H);
    float o[4] = {0.f, 0.f, 0.f, 0.f};
    // outputs whose window covers this voxel: od*s - p <= zi <= od*s - p + k - 1
    const int d0 = max(0, (zi + q.p - q.k + q.s) / q.s), d1 = min(q.Do - 1, (zi + q.p) / q.s);
    const int h0 = max(0, (hi + q.p - q.k + q.s) / q.s), h1 = min(q.Ho - 1, (hi + q.p) / q.s);
    const int w0 = max(0, (wi + q.p - q.k + q.s) / q.s), w1 = min(q.Wo - 1, (wi + q.p) / q.s);
    for (int od = d0; od <= d1; ++od)
      for (int oh = h0; oh <= h1; ++oh)
        for (int ow = w0; ow <= w1; ++ow) {
          const int e = ((zi - (od * q.s - q.p)) * q.k + (hi - (oh * q.s - q.p))) * q.k + (wi - (ow * q.s - q.p));
          const int64_t oi = (((int64_t)od * q.Ho + oh) * q.Wo + ow) * q.C4 + c4;
          const uchar4 a = arg[oi];
          const float4 g = ld4(gy + 4 * oi);
          if (a.x == e) o[0] += g.x;
          if (a.y == e) o[1] += g.y;
          if (a.z == e) o[2] += g.z;
          if (a.w == e) o[3] += g.w;
        }
    float* dst = gx + 4 * i;
    if (accumulate) {
      const float4 q4 = ld4(dst);
      o[0] += q4.x; o[1] += q4.y; o[2] += q4.z; o[3] += q4.w;
    }
    st4(dst, make_float4(o[0], o[1], o[2], o[3]));
  }
}

}  // namespace

static Pool3 pool3(int D, int H, int W, int C, int k, int s, int p) {
  Pool3 q{D, H, W, C / 4, (D + 2 * p - k) / s + 1, (H + 2 * p - k) / s + 1, (W + 2 * p - k) / s + 1, k, s, p};
  return q;
}

pooch_status maxpool3d_fwd(const float* x, float* y, int D, int H, int W, int C, cudaStream_t st, int k, int s,
                           int p) {
  if (!(k == 2 && s == 2 && p == 0)) {
    if (C % 4 || k < 1 || k > 6 || s < 1 || p < 0 || p >= k || D + 2 * p < k || H + 2 * p < k || W + 2 * p < k)
      return fail(POOCH_EUSAGE, "3D max-pool: bad k / s / p or C %% 4 != 0");
    const Pool3 q = pool3(D, H, W, C, k, s, p);
    const int64_t total = (int64_t)q.Do * q.Ho * q.Wo * q.C4;
    count_launch();
    maxpool3d_gen_fwd_kernel<<<grid_for(total, 256), 256, 0, st>>>(x, y, nullptr, q);
    POOCH_CUDA(cudaGetLastError());
    return POOCH_OK;
  }
  if (D % 2 || H % 2 || W % 2 || C % 4) return fail(POOCH_EUSAGE, "3D max-pool needs even extents, C % 4 == 0");
  int64_t total = (int64_t)(D / 2) * (H / 2) * (W / 2) * C / 4;
  count_launch();
  maxpool3d_fwd_kernel<<<grid_for(total, 256), 256, 0, st>>>(x, y, D, H, W, C / 4);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

pooch_status maxpool3d_bwd(const float* x, const float* gy, float* gx, int D, int H, int W, int C, bool accumulate,
                           cudaStream_t st, int k, int s, int p, uint8_t* arg_ws) {
  if (!(k == 2 && s == 2 && p == 0)) {
    if (C % 4 || k < 1 || k > 6 || s < 1 || p < 0 || p >= k || !arg_ws)
      return fail(POOCH_EUSAGE, "3D max-pool bwd: bad k / s / p, C %% 4 != 0 or no argmax workspace");
    const Pool3 q = pool3(D, H, W, C, k, s, p);
    const int64_t nout = (int64_t)q.Do * q.Ho * q.Wo * q.C4, nin = (int64_t)D * H * W * q.C4;
    // the window winners, recomputed from x (the forward kernel storing only arg)
    count_launch();
    maxpool3d_gen_fwd_kernel<<<grid_for(nout, 256), 256, 0, st>>>(x, nullptr, reinterpret_cast<uchar4*>(arg_ws), q);
    POOCH_CUDA(cudaGetLastError());
    count_launch();
    maxpool3d_gen_bwd_kernel<<<grid_for(nin, 256), 256, 0, st>>>(reinterpret_cast<const uchar4*>(arg_ws), gy, gx, q,
                                                                  accumulate ? 1 : 0);
    POOCH_CUDA(cudaGetLastError());
    return POOCH_OK;
  }
  if (D % 2 || H % 2 || W % 2 || C % 4) return fail(POOCH_EUSAGE, "3D max-pool needs even extents, C % 4 == 0");
  int64_t total = (int64_t)(D / 2) * (H / 2) * (W / 2) * C / 4;
  count_launch();
  maxpool3d_bwd_kernel<<<grid_for(total, 256), 256, 0, st>>>(x, gy, gx, D, H, W, C / 4, accumulate ? 1 : 0);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

pooch_status avgpool_fwd(const float* x, float* y, int N, int HW, int C, cudaStream_t st) {
  dim3 g((C / 4 + 127) / 128, N);
  count_launch();
  avgpool_fwd_kernel<<<g, 128, 0, st>>>(x, y, HW, C / 4);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

pooch_status avgpool_bwd(const float* gy, float* gx, int N, int HW, int C, cudaStream_t st) {
  int64_t n4 = (int64_t)N * HW * C / 4;
  count_launch();
  avgpool_bwd_kernel<<<grid_for(n4, 256), 256, 0, st>>>(gy, gx, n4, HW, C / 4);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

// Narrow heads with many rows (the per-voxel CE): thread-per-row CE and two-stage reductions.
static bool ce_narrow(int B, int ld) { return ld <= 8 && B >= 2048; }

pooch_status ce_fwd(const float* z, const int32_t* labels, int B, int classes, int ld, float* loss_rows, float* loss,
                    cudaStream_t st, double* ws) {
  if (ce_narrow(B, ld) && ws) {
    count_launch();
    ce_rows_narrow_kernel<<<grid_for(B, 256), 256, 0, st>>>(z, labels, B, classes, ld, loss_rows, nullptr, 0);
    count_launch();
    colsum_partial_kernel<<<kColsumBlocks, 256, 0, st>>>(loss_rows, B, 1, ws);
    count_launch();
    colsum_final_kernel<<<1, 32, 0, st>>>(ws, kColsumBlocks, 1, 1.0 / B, loss);
    POOCH_CUDA(cudaGetLastError());
    return POOCH_OK;
  }
  count_launch();
  ce_rows_kernel<<<(B + 7) / 8, 256, 0, st>>>(z, labels, B, classes, ld, loss_rows, nullptr, 0);
  count_launch();
  mean_kernel<<<1, 256, 0, st>>>(loss_rows, B, loss);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

pooch_status ce_bwd(const float* z, const int32_t* labels, int B, int classes, int ld, float* dz, float* db,
                    cudaStream_t st, double* ws) {
  if (ce_narrow(B, ld) && ws) {
    count_launch();
    ce_rows_narrow_kernel<<<grid_for(B, 256), 256, 0, st>>>(z, labels, B, classes, ld, nullptr, dz, 1);
    count_launch();
    colsum_partial_kernel<<<kColsumBlocks, 256, 0, st>>>(dz, B, ld, ws);
    count_launch();
    colsum_final_kernel<<<1, 32, 0, st>>>(ws, kColsumBlocks, ld, 1.0, db);
    POOCH_CUDA(cudaGetLastError());
    return POOCH_OK;
  }
  count_launch();
  ce_rows_kernel<<<(B + 7) / 8, 256, 0, st>>>(z, labels, B, classes, ld, nullptr, dz, 1);
  count_launch();
  colsum_kernel<<<(ld + 127) / 128, 128, 0, st>>>(dz, B, ld, db);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

size_t ce_ws_bytes() { return (size_t)kColsumBlocks * 8 * sizeof(double); }

pooch_status sgd_momentum(float* w, float* v, const float* g, int64_t n, float lr, float mu, float scale,
                          cudaStream_t st) {
  int64_t n4 = n / 4;
  if (n4 > 0) { count_launch(); sgd_kernel<<<grid_for(n4, 256), 256, 0, st>>>(w, v, g, n4, lr, mu, scale); }
  if (n % 4) { count_launch(); sgd_tail_kernel<<<1, 32, 0, st>>>(w, v, g, n4 * 4, n, lr, mu, scale); }
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

namespace {
// one thread per (output slice voxel, float4 of the 32 channels); C % 4 == 0
__global__ void depth_im2col_kernel(const float* __restrict__ x, float* __restrict__ xs, int D, int H, int W, int C4,
                                    int k, int p, int Do) {
  const int64_t total = (int64_t)Do * H * W * 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int j4 = (int)(i & 7);
    const int64_t vox = i >> 3;
    const int64_t hw = vox % ((int64_t)H * W);
    const int od = (int)(vox / ((int64_t)H * W));
    const int u = j4 / C4, c4 = j4 % C4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    const int d = od + u - p;
    if (u < k && d >= 0 && d < D) v = ld4(x + (((int64_t)d * H * W + hw) * C4 + c4) * 4);
    st4(xs + 4 * i, v);
  }
}

__global__ void fold_weight_kernel(float* w, float* w2, int K, int k, int C, int back) {
  const int64_t total = (int64_t)K * k * k * 32;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(i % 32);
    const int64_t r = i / 32;                 // (o, v, t)
    const int t = (int)(r % k), v = (int)((r / k) % k), o = (int)(r / ((int64_t)k * k));
    const int u = j / C, c = j % C;
    if (back) {
      if (u < k) w[((((int64_t)o * k + u) * k + v) * k + t) * C + c] = w2[i];
    } else {
      w2[i] = u < k ? w[((((int64_t)o * k + u) * k + v) * k + t) * C + c] : 0.f;
    }
  }
}
}  // namespace

pooch_status depth_im2col(const float* x, float* xs, int D, int H, int W, int C, int k, int p, int Do,
                          cudaStream_t st) {
  if (C % 4 || k * C > 32) return fail(POOCH_EUSAGE, "depth_im2col: k * C must be <= 32, C %% 4 == 0");
  const int64_t total = (int64_t)Do * H * W * 8;
  count_launch();
  depth_im2col_kernel<<<grid_for(total, 256), 256, 0, st>>>(x, xs, D, H, W, C / 4, k, p, Do);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

pooch_status fold_weight(const float* w, float* w2, int K, int k, int C, cudaStream_t st) {
  count_launch();
  fold_weight_kernel<<<grid_for((int64_t)K * k * k * 32, 256), 256, 0, st>>>(const_cast<float*>(w), w2, K, k, C, 0);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

pooch_status unfold_weight(const float* w2, float* w, int K, int k, int C, cudaStream_t st) {
  count_launch();
  fold_weight_kernel<<<grid_for((int64_t)K * k * k * 32, 256), 256, 0, st>>>(w, const_cast<float*>(w2), K, k, C, 1);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

pooch_status transpose_krsc(const float* w, float* wt, int K, int RS, int C, cudaStream_t st) {
  dim3 g((C + 31) / 32, (K + 31) / 32, RS);
  count_launch();
  transpose_kernel<<<g, dim3(32, 8), 0, st>>>(w, wt, K, RS, C);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

}  // namespace pooch

extern "C" pooch_status pooch_op_maxpool2d_fwd(const float* x, float* y, int32_t N, int32_t H, int32_t W, int32_t C,
                                               int32_t k, int32_t s, int32_t p, void* stream) {
  if (!x || !y || N <= 0 || H <= 0 || W <= 0 || k <= 0 || s <= 0 || p < 0 || H + 2 * p < k || W + 2 * p < k)
    return pooch::fail(POOCH_EUSAGE, "maxpool2d: bad arguments");
  const int Ho = (H + 2 * p - k) / s + 1, Wo = (W + 2 * p - k) / s + 1;
  return pooch::maxpool_fwd(x, y, N, H, W, C, k, s, p, Ho, Wo, (cudaStream_t)stream);
}

extern "C" pooch_status pooch_op_maxpool2d_bwd(const float* x, const float* gy, float* gx, void* arg_ws, int32_t N,
                                               int32_t H, int32_t W, int32_t C, int32_t k, int32_t s, int32_t p,
                                               void* stream) {
  if (!x || !gy || !gx || !arg_ws || N <= 0 || H <= 0 || W <= 0 || k <= 0 || s <= 0 || p < 0 || H + 2 * p < k ||
      W + 2 * p < k || k * k > 255)
    return pooch::fail(POOCH_EUSAGE, "maxpool2d: bad arguments");
  const int Ho = (H + 2 * p - k) / s + 1, Wo = (W + 2 * p - k) / s + 1;
  return pooch::maxpool_bwd(x, gy, gx, reinterpret_cast<uint8_t*>(arg_ws), N, H, W, C, k, s, p, Ho, Wo, (cudaStream_t)stream);
}

// ---- kernel-level entry points of the BN(-ReLU) and 3D max-pool kernels (parity tests; the
// executor calls the same launchers)
extern "C" size_t pooch_op_bn_ws_bytes(int32_t C) {
  return std::max(pooch::bn_finalize_ws_bytes(C), pooch::bn_bwd_ws_bytes(C));
}

extern "C" pooch_status pooch_op_bn_finalize(const float* tile_sum, const float* tile_sq, int32_t tiles, int32_t C,
                                             int64_t count, const float* gamma, const float* beta, float* mean,
                                             float* invstd, float* scale, float* shift, void* ws, void* stream) {
  if (!tile_sum || !tile_sq || !gamma || !beta || !mean || !invstd || !scale || !shift || !ws || tiles <= 0 || C <= 0 ||
      C % 4 || count <= 0)
    return pooch::fail(POOCH_EUSAGE, "bn_finalize: bad arguments");
  return pooch::bn_finalize(tile_sum, tile_sq, tiles, C, count, gamma, beta, mean, invstd, scale, shift,
                            reinterpret_cast<double*>(ws), (cudaStream_t)stream);
}

extern "C" pooch_status pooch_op_bn_relu_fwd(const float* x, const float* scale, const float* shift, float* y,
                                             int64_t rows, int32_t C, void* stream) {
  if (!x || !scale || !shift || !y || rows <= 0 || C <= 0 || C % 4)
    return pooch::fail(POOCH_EUSAGE, "bn_relu_fwd: bad arguments");
  return pooch::bn_apply_relu(x, scale, shift, nullptr, nullptr, nullptr, 0, y, rows, C, (cudaStream_t)stream);
}

extern "C" pooch_status pooch_op_bn_relu_bwd(const float* x, const float* gy, const float* scale, const float* shift,
                                             const float* mean, const float* invstd, const float* gamma, float* dgamma,
                                             float* dbeta, float* gx, int64_t rows, int32_t C, void* ws,
                                             void* stream) {
  if (!x || !gy || !scale || !shift || !mean || !invstd || !gamma || !dgamma || !dbeta || !gx || !ws || rows <= 0 ||
      C <= 0 || C % 4)
    return pooch::fail(POOCH_EUSAGE, "bn_relu_bwd: bad arguments");
  pooch::BnBwdArgs a{};
  a.a = x;
  a.gy = gy;
  a.sa = scale;
  a.ta = shift;
  a.mean_a = mean;
  a.invstd_a = invstd;
  a.gamma_a = gamma;
  a.dgamma_a = dgamma;
  a.dbeta_a = dbeta;
  a.ga = gx;
  a.mode = 0;
  a.rows = rows;
  a.C = C;
  return pooch::bn_bwd(a, reinterpret_cast<float*>(ws), (cudaStream_t)stream);
}

extern "C" pooch_status pooch_op_maxpool3d_fwd(const float* x, float* y, int32_t D, int32_t H, int32_t W, int32_t C,
                                               void* stream) {
  if (!x || !y || D < 2 || H < 2 || W < 2 || C <= 0 || C % 4) return pooch::fail(POOCH_EUSAGE, "maxpool3d: bad arguments");
  return pooch::maxpool3d_fwd(x, y, D, H, W, C, (cudaStream_t)stream);
}

extern "C" pooch_status pooch_op_maxpool3d_fwd_k(const float* x, float* y, int32_t D, int32_t H, int32_t W,
                                                 int32_t C, int32_t k, int32_t s, int32_t p, void* stream) {
  if (!x || !y || D < 1 || H < 1 || W < 1 || C <= 0) return pooch::fail(POOCH_EUSAGE, "maxpool3d: bad arguments");
  return pooch::maxpool3d_fwd(x, y, D, H, W, C, (cudaStream_t)stream, k, s, p);
}

extern "C" pooch_status pooch_op_maxpool3d_bwd_k(const float* x, const float* gy, float* gx, void* arg_ws, int32_t D,
                                                 int32_t H, int32_t W, int32_t C, int32_t k, int32_t s, int32_t p,
                                                 int32_t accumulate, void* stream) {
  if (!x || !gy || !gx || D < 1 || H < 1 || W < 1 || C <= 0) return pooch::fail(POOCH_EUSAGE, "maxpool3d: bad arguments");
  return pooch::maxpool3d_bwd(x, gy, gx, D, H, W, C, accumulate != 0, (cudaStream_t)stream, k, s, p,
                              static_cast<uint8_t*>(arg_ws));
}

extern "C" pooch_status pooch_op_maxpool3d_bwd(const float* x, const float* gy, float* gx, int32_t D, int32_t H,
                                               int32_t W, int32_t C, int32_t accumulate, void* stream) {
  if (!x || !gy || !gx || D < 2 || H < 2 || W < 2 || C <= 0 || C % 4)
    return pooch::fail(POOCH_EUSAGE, "maxpool3d: bad arguments");
  return pooch::maxpool3d_bwd(x, gy, gx, D, H, W, C, accumulate != 0, (cudaStream_t)stream);
}
