// gconv.cu -- grouped 3D convolution on the CUDA cores (ResNeXt-101 (3D)'s 3^3 bottleneck conv,
// SURVEY 8(f) f4; Sec. 5.2): fwd (+ BN partial sums), dgrad, wgrad.
//
// Definition (oracle layers.gconv3d_fwd): with Cg = C / G input and Kg = K / G output channels
// per group, y[z,h,w, g*Kg+o] = sum_{c < Cg, taps (u,v,t)} x[sd*z+u-p, s*h+v-p, s*w+t-p, g*Cg+c]
// * w[g*Kg+o, u, v, t, c]. NDHWC, batch 1, weights [K][k][k][k][Cg].
//
// Why not the tensor cores: ResNeXt's groups hold 4 / 8 / 16 / 32 channels, so each group is a
// GEMM with N = K_g <= 32 and K-dim 27 * C_g <= 864 -- far below a tcgen05 tile (N >= 64 to
// keep the pipe busy; block-diagonal packing would multiply the work by the groups per tile).
// At 27 taps x C_g MACs per output element the pass is ALU-bound on FP32 FMA:
// every kernel here register-blocks 32 accumulators per thread so one shared-memory or global
// load feeds 4-32 FMAs, and all reductions run in a fixed order (plans stay bit-exact).
//
// fwd  : one thread = one output voxel x 32 output channels (NG = 32 / Kg groups); a block = 128
//        voxels x one 32-channel group block; weights of those groups transposed into shared
//        memory [group][tap][c][o]; BN partial sums per block in a fixed order.
// dgrad: one thread = one input voxel x 32 input channels; the taps whose output position is an
//        integer (stride 2: one or two per axis) gather dy; weights in smem [group][tap][o][c].
// wgrad: a block = a chunk of output voxels x a group block x a slice of taps; 32-voxel tiles of
//        dy and of the tap-shifted x are staged in smem; every thread owns 4 x 4 (o, c) blocks of
//        dw; per-chunk partials are summed over the chunks in order by a second kernel.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.h"
#include "conv.h"

namespace pooch {

namespace {

constexpr int kFwdThreads = 128;
constexpr int kWgV = 32;          // voxels per wgrad smem tile
constexpr int kWgThreads = 256;

struct GArgs {
  const float* x;    // [D][H][W][C]
  const float* w;    // [K][taps][Cg]
  const float* dy;   // [Do][Ho][Wo][K]
  float* out;
  float* stat_sum;
  float* stat_sq;
  int D, H, W, C, Do, Ho, Wo, K, k, sd, s, pad;
  int64_t M;         // output voxels
  int accumulate;
  int tap0, ntap;    // wgrad: tap slice of this launch's z index (ntap per z)
  int64_t chunk;     // wgrad: voxels per chunk
};

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// ------------------------------------------------------------------------------ forward
template <int CG>  // channels per group (in == out); NG = 32 / CG groups per block
__global__ void __launch_bounds__(kFwdThreads) gconv_fwd_kernel(GArgs a) {
  constexpr int NG = 32 / CG;
  extern __shared__ float ws[];  // [NG][taps][CG (c)][CG (o)]
  const int taps = a.k * a.k * a.k;
  const int gb = blockIdx.y;     // 32-channel block: groups gb*NG .. gb*NG+NG-1
  for (int i = threadIdx.x; i < NG * taps * CG * CG; i += blockDim.x) {
    // i -> (j, tap, c, o) in smem order; the global weight is [K][taps][CG]
    const int o = i % CG, c = (i / CG) % CG, tap = (i / (CG * CG)) % taps, j = i / (CG * CG * taps);
    ws[i] = a.w[((int64_t)(gb * 32 + j * CG + o) * taps + tap) * CG + c];
  }
  __syncthreads();
  const int64_t m = (int64_t)blockIdx.x * kFwdThreads + threadIdx.x;
  float acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = 0.f;
  const bool valid = m < a.M;
  if (valid) {
    const int ow = (int)(m % a.Wo);
    const int oh = (int)((m / a.Wo) % a.Ho);
    const int od = (int)(m / ((int64_t)a.Wo * a.Ho));
    int tap = 0;
    for (int u = 0; u < a.k; ++u) {
      const int zi = od * a.sd - a.pad + u;
      for (int v = 0; v < a.k; ++v) {
        const int hi = oh * a.s - a.pad + v;
        for (int t = 0; t < a.k; ++t, ++tap) {
          const int wi = ow * a.s - a.pad + t;
          if (zi < 0 || zi >= a.D || hi < 0 || hi >= a.H || wi < 0 || wi >= a.W) continue;
          const float* xp = a.x + (((int64_t)zi * a.H + hi) * a.W + wi) * a.C + gb * 32;
#pragma unroll
          for (int j = 0; j < NG; ++j) {
            float xv[CG];
#pragma unroll
            for (int c4 = 0; c4 < CG / 4; ++c4) {
              const float4 q = ldg4(xp + j * CG + 4 * c4);
              xv[4 * c4] = q.x; xv[4 * c4 + 1] = q.y; xv[4 * c4 + 2] = q.z; xv[4 * c4 + 3] = q.w;
            }
            const float* wr = ws + ((j * taps + tap) * CG) * CG;
#pragma unroll
            for (int c = 0; c < CG; ++c) {
#pragma unroll
              for (int o4 = 0; o4 < CG / 4; ++o4) {
                const float4 wv = *reinterpret_cast<const float4*>(wr + c * CG + 4 * o4);
                float* ac = acc + j * CG + 4 * o4;
                ac[0] = fmaf(xv[c], wv.x, ac[0]);
                ac[1] = fmaf(xv[c], wv.y, ac[1]);
                ac[2] = fmaf(xv[c], wv.z, ac[2]);
                ac[3] = fmaf(xv[c], wv.w, ac[3]);
              }
            }
          }
        }
      }
    }
    float* yp = a.out + m * a.K + gb * 32;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      *reinterpret_cast<float4*>(yp + 4 * i) = make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
  }
  if (!a.stat_sum) return;
  // BN partial sums of this block's 128 voxels x 32 channels: warp shuffles, then the four
  // warps in order (invalid voxels contribute zeros)
  __shared__ float red[2][kFwdThreads / 32][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    float sv = acc[i], qv = acc[i] * acc[i];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      sv += __shfl_xor_sync(0xffffffffu, sv, off);
      qv += __shfl_xor_sync(0xffffffffu, qv, off);
    }
    if (lane == i) {
      red[0][warp][i] = sv;
      red[1][warp][i] = qv;
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    float sv = 0.f, qv = 0.f;
    for (int w = 0; w < kFwdThreads / 32; ++w) {
      sv += red[0][w][threadIdx.x];
      qv += red[1][w][threadIdx.x];
    }
    a.stat_sum[(int64_t)blockIdx.x * a.K + gb * 32 + threadIdx.x] = sv;
    a.stat_sq[(int64_t)blockIdx.x * a.K + gb * 32 + threadIdx.x] = qv;
  }
}

// ------------------------------------------------------------------------------ dgrad
// first tap index u (0 <= u < k) with (i + pad - u) % s == 0, and the output position
__device__ __forceinline__ bool tap_ok(int i, int u, int pad, int s, int n_out, int& o) {
  const int q = i + pad - u;
  if (q < 0 || q % s) return false;
  o = q / s;
  return o < n_out;
}

template <int CG>
__global__ void __launch_bounds__(kFwdThreads) gconv_dgrad_kernel(GArgs a) {
  constexpr int NG = 32 / CG;
  extern __shared__ float ws[];  // [NG][taps][CG (o)][CG (c)]: the global layout per group
  const int taps = a.k * a.k * a.k;
  const int gb = blockIdx.y;
  for (int i = threadIdx.x; i < NG * taps * CG * CG; i += blockDim.x) {
    const int c = i % CG, o = (i / CG) % CG, tap = (i / (CG * CG)) % taps, j = i / (CG * CG * taps);
    ws[i] = a.w[((int64_t)(gb * 32 + j * CG + o) * taps + tap) * CG + c];
  }
  __syncthreads();
  const int64_t n_in = (int64_t)a.D * a.H * a.W;
  const int64_t m = (int64_t)blockIdx.x * kFwdThreads + threadIdx.x;
  if (m >= n_in) return;
  const int wi = (int)(m % a.W);
  const int hi = (int)((m / a.W) % a.H);
  const int zi = (int)(m / ((int64_t)a.W * a.H));
  float acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = 0.f;
  for (int u = 0; u < a.k; ++u) {
    int od;
    if (!tap_ok(zi, u, a.pad, a.sd, a.Do, od)) continue;
    for (int v = 0; v < a.k; ++v) {
      int oh;
      if (!tap_ok(hi, v, a.pad, a.s, a.Ho, oh)) continue;
      for (int t = 0; t < a.k; ++t) {
        int ow;
        if (!tap_ok(wi, t, a.pad, a.s, a.Wo, ow)) continue;
        const int tap = (u * a.k + v) * a.k + t;
        const float* gp = a.dy + (((int64_t)od * a.Ho + oh) * a.Wo + ow) * a.K + gb * 32;
#pragma unroll
        for (int j = 0; j < NG; ++j) {
          float gv[CG];
#pragma unroll
          for (int o4 = 0; o4 < CG / 4; ++o4) {
            const float4 q = ldg4(gp + j * CG + 4 * o4);
            gv[4 * o4] = q.x; gv[4 * o4 + 1] = q.y; gv[4 * o4 + 2] = q.z; gv[4 * o4 + 3] = q.w;
          }
          const float* wr = ws + ((j * taps + tap) * CG) * CG;
#pragma unroll
          for (int o = 0; o < CG; ++o) {
#pragma unroll
            for (int c4 = 0; c4 < CG / 4; ++c4) {
              const float4 wv = *reinterpret_cast<const float4*>(wr + o * CG + 4 * c4);
              float* ac = acc + j * CG + 4 * c4;
              ac[0] = fmaf(gv[o], wv.x, ac[0]);
              ac[1] = fmaf(gv[o], wv.y, ac[1]);
              ac[2] = fmaf(gv[o], wv.z, ac[2]);
              ac[3] = fmaf(gv[o], wv.w, ac[3]);
            }
          }
        }
      }
    }
  }
  float* xp = a.out + m * a.C + gb * 32;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float4 r = make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
    if (a.accumulate) {
      const float4 q = *reinterpret_cast<const float4*>(xp + 4 * i);
      r.x += q.x; r.y += q.y; r.z += q.z; r.w += q.w;
    }
    *reinterpret_cast<float4*>(xp + 4 * i) = r;
  }
}

// ------------------------------------------------------------------------------ wgrad
// grid (chunks, K / 32, tap slices); ws[chunk][K][taps][CG] partials (or dw itself, one chunk)
template <int CG, int TZ>  // TZ taps per slice
__global__ void __launch_bounds__(kWgThreads) gconv_wgrad_kernel(GArgs a) {
  constexpr int NG = 32 / CG;
  constexpr int NB4 = NG * TZ * (CG / 4) * (CG / 4);   // 4x4 (o, c) blocks of this CTA
  constexpr int PER = (NB4 + kWgThreads - 1) / kWgThreads;
  extern __shared__ __align__(16) float wsm[];   // dy tile [V][32], then x tiles [TZ][V][32]
  float(*dys)[32] = reinterpret_cast<float(*)[32]>(wsm);
  float(*xs)[kWgV][32] = reinterpret_cast<float(*)[kWgV][32]>(wsm + kWgV * 32);
  const int taps = a.k * a.k * a.k;
  const int gb = blockIdx.y;
  const int tap0 = blockIdx.z * TZ;
  const int64_t m0 = (int64_t)blockIdx.x * a.chunk, m1 = min(a.M, m0 + a.chunk);
  float acc[PER][16];
#pragma unroll
  for (int p = 0; p < PER; ++p)
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[p][i] = 0.f;
  for (int64_t mt = m0; mt < m1; mt += kWgV) {
    // stage dy [V][32] and x [TZ][V][32] (zero outside the tile / the padding)
    for (int i = threadIdx.x; i < kWgV * 8; i += kWgThreads) {
      const int v = i >> 3, c4 = i & 7;
      const int64_t m = mt + v;
      float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
      if (m < m1) q = ldg4(a.dy + m * a.K + gb * 32 + 4 * c4);
      *reinterpret_cast<float4*>(&dys[v][4 * c4]) = q;
    }
    for (int i = threadIdx.x; i < TZ * kWgV * 8; i += kWgThreads) {
      const int c4 = i & 7, v = (i >> 3) % kWgV, tz = i / (8 * kWgV);
      const int tap = tap0 + tz;
      const int64_t m = mt + v;
      float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
      if (m < m1 && tap < taps) {
        const int ow = (int)(m % a.Wo), oh = (int)((m / a.Wo) % a.Ho), od = (int)(m / ((int64_t)a.Wo * a.Ho));
        const int u = tap / (a.k * a.k), vv = (tap / a.k) % a.k, t = tap % a.k;
        const int zi = od * a.sd - a.pad + u, hi = oh * a.s - a.pad + vv, wi = ow * a.s - a.pad + t;
        if (zi >= 0 && zi < a.D && hi >= 0 && hi < a.H && wi >= 0 && wi < a.W)
          q = ldg4(a.x + (((int64_t)zi * a.H + hi) * a.W + wi) * a.C + gb * 32 + 4 * c4);
      }
      *reinterpret_cast<float4*>(&xs[tz][v][4 * c4]) = q;
    }
    __syncthreads();
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      const int b = threadIdx.x + p * kWgThreads;
      if (b < NB4) {
        // b -> (j, tz, o4, c4)
        const int c4 = b % (CG / 4), o4 = (b / (CG / 4)) % (CG / 4), tz = (b / ((CG / 4) * (CG / 4))) % TZ,
                  j = b / ((CG / 4) * (CG / 4) * TZ);
        const int oc = j * CG + 4 * o4, xc = j * CG + 4 * c4;
#pragma unroll 8
        for (int v = 0; v < kWgV; ++v) {
          const float4 g = *reinterpret_cast<const float4*>(&dys[v][oc]);
          const float4 xv = *reinterpret_cast<const float4*>(&xs[tz][v][xc]);
          const float ga[4] = {g.x, g.y, g.z, g.w}, xa[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
          for (int oo = 0; oo < 4; ++oo)
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) acc[p][oo * 4 + cc] = fmaf(ga[oo], xa[cc], acc[p][oo * 4 + cc]);
        }
      }
    }
    __syncthreads();
  }
  float* dst = a.out + (int64_t)blockIdx.x * a.K * taps * CG;
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    const int b = threadIdx.x + p * kWgThreads;
    if (b >= NB4) continue;
    const int c4 = b % (CG / 4), o4 = (b / (CG / 4)) % (CG / 4), tz = (b / ((CG / 4) * (CG / 4))) % TZ,
              j = b / ((CG / 4) * (CG / 4) * TZ);
    const int tap = tap0 + tz;
    if (tap >= taps) continue;
#pragma unroll
    for (int oo = 0; oo < 4; ++oo) {
      const int o = gb * 32 + j * CG + 4 * o4 + oo;
      *reinterpret_cast<float4*>(dst + ((int64_t)o * taps + tap) * CG + 4 * c4) =
          make_float4(acc[p][oo * 4], acc[p][oo * 4 + 1], acc[p][oo * 4 + 2], acc[p][oo * 4 + 3]);
    }
  }
}

__global__ void gconv_chunk_reduce_kernel(const float4* __restrict__ ws, float4* __restrict__ dw, int64_t n4,
                                          int chunks) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 s = ws[i];
    for (int c = 1; c < chunks; ++c) {
      const float4 q = ws[(int64_t)c * n4 + i];
      s.x += q.x; s.y += q.y; s.z += q.z; s.w += q.w;
    }
    dw[i] = s;
  }
}

GArgs gargs(const ConvGeom& g) {
  GArgs a{};
  a.D = g.D; a.H = g.H; a.W = g.W; a.C = g.C;
  a.Do = g.Do; a.Ho = g.Ho; a.Wo = g.Wo; a.K = g.K;
  a.k = g.R; a.sd = g.sd(); a.s = g.stride; a.pad = g.pad;
  a.M = (int64_t)g.Do * g.Ho * g.Wo;
  return a;
}

int cg_of(const ConvGeom& g) { return g.C / g.groups; }

// taps per wgrad slice: the CTA's 4x4 blocks (NG * TZ * (CG/4)^2) fit two per thread
int wgrad_tz(int cg) { return cg == 32 ? 3 : (cg == 16 ? 9 : 27); }

int wgrad_chunks(const ConvGeom& g) {
  const int taps = g.R * g.R * g.R;
  const int tz = wgrad_tz(cg_of(g));
  const int per_chunk = (g.K / 32) * ((taps + tz - 1) / tz);
  const int64_t M = (int64_t)g.Do * g.Ho * g.Wo;
  // ~2 waves of 148 SMs, at least 4 tiles of 32 voxels per chunk
  int64_t ch = std::max<int64_t>(1, (2 * 148 + per_chunk - 1) / per_chunk);
  ch = std::min<int64_t>(ch, std::max<int64_t>(1, M / (4 * kWgV)));
  return (int)std::min<int64_t>(ch, 256);
}

template <typename Kern>
pooch_status set_smem(Kern k, int bytes) {
  if (bytes > 48 * 1024) POOCH_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  return POOCH_OK;
}

}  // namespace

bool gconv_shape_ok(const ConvGeom& g) {
  const int cg = g.groups > 0 ? g.C / g.groups : 0;
  return g.is3d() && g.groups > 1 && g.C == g.K && g.C % g.groups == 0 &&
         (cg == 4 || cg == 8 || cg == 16 || cg == 32) && g.K % 32 == 0 && (g.R == 1 || g.R == 3) && g.R == g.S &&
         g.stride >= 1 && g.stride <= 2 && g.sd() >= 1 && g.sd() <= 2 && g.N == 1;
}

int gconv_stat_tiles(const ConvGeom& g) {
  return (int)(((int64_t)g.Do * g.Ho * g.Wo + kFwdThreads - 1) / kFwdThreads);
}

size_t gconv_wgrad_ws_bytes(const ConvGeom& g) {
  const int ch = wgrad_chunks(g);
  return ch > 1 ? (size_t)ch * g.K * g.R * g.R * g.R * cg_of(g) * sizeof(float) : 0;
}

pooch_status gconv_fwd(const ConvGeom& g, const float* x, const float* w, float* y, float* stat_sum,
                       float* stat_sq, cudaStream_t st) {
  if (!gconv_shape_ok(g)) return fail(POOCH_EUSAGE, "grouped conv: unsupported shape");
  GArgs a = gargs(g);
  a.x = x; a.w = w; a.out = y; a.stat_sum = stat_sum; a.stat_sq = stat_sq;
  if ((stat_sum == nullptr) != (stat_sq == nullptr)) return fail(POOCH_EUSAGE, "stat_sum / stat_sq: both or none");
  const int taps = g.R * g.R * g.R, cg = cg_of(g);
  const int smem = 32 * taps * cg * (int)sizeof(float);
  dim3 grid((unsigned)gconv_stat_tiles(g), g.K / 32);
  if (a.M == 0) return POOCH_OK;
  count_launch();
  switch (cg) {
    case 4: POOCH_CHECK(set_smem(gconv_fwd_kernel<4>, smem)); gconv_fwd_kernel<4><<<grid, kFwdThreads, smem, st>>>(a); break;
    case 8: POOCH_CHECK(set_smem(gconv_fwd_kernel<8>, smem)); gconv_fwd_kernel<8><<<grid, kFwdThreads, smem, st>>>(a); break;
    case 16: POOCH_CHECK(set_smem(gconv_fwd_kernel<16>, smem)); gconv_fwd_kernel<16><<<grid, kFwdThreads, smem, st>>>(a); break;
    case 32: POOCH_CHECK(set_smem(gconv_fwd_kernel<32>, smem)); gconv_fwd_kernel<32><<<grid, kFwdThreads, smem, st>>>(a); break;
  }
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

pooch_status gconv_dgrad(const ConvGeom& g, const float* dy, const float* w, float* dx, bool accumulate,
                         cudaStream_t st) {
  if (!gconv_shape_ok(g)) return fail(POOCH_EUSAGE, "grouped conv: unsupported shape");
  GArgs a = gargs(g);
  a.dy = dy; a.w = w; a.out = dx; a.accumulate = accumulate ? 1 : 0;
  const int taps = g.R * g.R * g.R, cg = cg_of(g);
  const int smem = 32 * taps * cg * (int)sizeof(float);
  const int64_t n_in = (int64_t)g.D * g.H * g.W;
  dim3 grid((unsigned)((n_in + kFwdThreads - 1) / kFwdThreads), g.C / 32);
  if (n_in == 0) return POOCH_OK;
  count_launch();
  switch (cg) {
    case 4: POOCH_CHECK(set_smem(gconv_dgrad_kernel<4>, smem)); gconv_dgrad_kernel<4><<<grid, kFwdThreads, smem, st>>>(a); break;
    case 8: POOCH_CHECK(set_smem(gconv_dgrad_kernel<8>, smem)); gconv_dgrad_kernel<8><<<grid, kFwdThreads, smem, st>>>(a); break;
    case 16: POOCH_CHECK(set_smem(gconv_dgrad_kernel<16>, smem)); gconv_dgrad_kernel<16><<<grid, kFwdThreads, smem, st>>>(a); break;
    case 32: POOCH_CHECK(set_smem(gconv_dgrad_kernel<32>, smem)); gconv_dgrad_kernel<32><<<grid, kFwdThreads, smem, st>>>(a); break;
  }
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

pooch_status gconv_wgrad(const ConvGeom& g, const float* x, const float* dy, float* dw, float* ws, size_t ws_bytes,
                         cudaStream_t st) {
  if (!gconv_shape_ok(g)) return fail(POOCH_EUSAGE, "grouped conv: unsupported shape");
  const int chunks = wgrad_chunks(g);
  if (chunks > 1 && ws_bytes < gconv_wgrad_ws_bytes(g))
    return fail(POOCH_EUSAGE, "grouped wgrad workspace too small: %zu < %zu", ws_bytes, gconv_wgrad_ws_bytes(g));
  GArgs a = gargs(g);
  a.x = x; a.dy = dy; a.out = chunks > 1 ? ws : dw;
  a.chunk = (a.M + chunks - 1) / chunks;
  const int taps = g.R * g.R * g.R, cg = cg_of(g), tz = wgrad_tz(cg);
  dim3 grid(chunks, g.K / 32, (taps + tz - 1) / tz);
  const int smem = (1 + tz) * kWgV * 32 * (int)sizeof(float);
  count_launch();
  switch (cg) {
    case 4: POOCH_CHECK(set_smem(gconv_wgrad_kernel<4, 27>, smem)); gconv_wgrad_kernel<4, 27><<<grid, kWgThreads, smem, st>>>(a); break;
    case 8: POOCH_CHECK(set_smem(gconv_wgrad_kernel<8, 27>, smem)); gconv_wgrad_kernel<8, 27><<<grid, kWgThreads, smem, st>>>(a); break;
    case 16: POOCH_CHECK(set_smem(gconv_wgrad_kernel<16, 9>, smem)); gconv_wgrad_kernel<16, 9><<<grid, kWgThreads, smem, st>>>(a); break;
    case 32: POOCH_CHECK(set_smem(gconv_wgrad_kernel<32, 3>, smem)); gconv_wgrad_kernel<32, 3><<<grid, kWgThreads, smem, st>>>(a); break;
  }
  POOCH_CUDA(cudaGetLastError());
  if (chunks > 1) {
    const int64_t n4 = (int64_t)g.K * taps * cg / 4;
    count_launch();
    gconv_chunk_reduce_kernel<<<(int)std::min<int64_t>((n4 + 255) / 256, 148 * 8), 256, 0, st>>>(
        reinterpret_cast<const float4*>(ws), reinterpret_cast<float4*>(dw), n4, chunks);
    POOCH_CUDA(cudaGetLastError());
  }
  return POOCH_OK;
}

}  // namespace pooch
