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
// fwd  : a block = 128 output voxels x one 32-channel block (32 / Cg groups); a thread = 4 voxels
//        x one channel quad, so a warp-wide 128-bit load covers 4 voxels' 128 contiguous bytes and
//        one shared-memory weight quad feeds 16 FMAs; weights staged [tap][c][o]; BN partial sums
//        per block in a fixed order.
// dgrad: the same layout over input voxels; the taps whose output position is an integer gather
//        dy (stride 2: each warp owns one W parity, so its lanes skip the same taps).
// wgrad: a block = a chunk of output voxels x a 32-channel block x a slice of taps; 16 / 32-voxel
//        tiles of dy and of the tap-shifted x are staged in smem; every thread owns 4 x 4 (o, c)
//        blocks of dw; per-chunk partials are summed over the chunks in order by a second kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>

#include "common.h"
#include "conv.h"

namespace pooch {

namespace {

constexpr int kThreads = 256;     // every kernel: 8 warps
constexpr int kVoxBlk = 128;      // fwd / dgrad: voxels per block (8 warps x 4 voxel lanes x kV)

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

// the output position o of input coordinate i through tap u (stride S, padding pad), if integral
template <int S>
__device__ __forceinline__ bool tap_ok(int i, int u, int pad, int n_out, int& o) {
  const int q = i + pad - u;
  if (q < 0 || (S == 2 && (q & 1))) return false;
  o = S == 2 ? q >> 1 : q;
  return o < n_out;
}

// ------------------------------------------------------------------------------ forward
// Thread layout shared by fwd and dgrad: lane = (vs, q) with q = lane & 7 the channel quad (4
// channels of the block's 32) and vs = lane >> 3; a thread owns kV voxels, so one warp-wide
// 128-bit access covers 4 voxels x 128 contiguous bytes, and one shared-memory weight quad
// (broadcast to the lanes of equal q, conflict-free across q) feeds 4 x kV FMAs.
constexpr int kV = 4;

__device__ __forceinline__ float f4c(const float4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}
__device__ __forceinline__ void fma4(float4& acc, float s, const float4& w) {
  acc.x = fmaf(s, w.x, acc.x);
  acc.y = fmaf(s, w.y, acc.y);
  acc.z = fmaf(s, w.z, acc.z);
  acc.w = fmaf(s, w.w, acc.w);
}

template <int CG>  // channels per group (in == out)
__global__ void __launch_bounds__(kThreads) gconv_fwd_kernel(GArgs a) {
  extern __shared__ float4 smem4[];
  float* ws = reinterpret_cast<float*>(smem4);  // [taps][CG (c)][32 (o of the block)]
  const int taps = a.k * a.k * a.k;
  const int gb = blockIdx.y;
  for (int i = threadIdx.x; i < taps * CG * 32; i += kThreads) {
    const int o = i & 31, c = (i >> 5) % CG, tap = i / (32 * CG);
    ws[i] = a.w[((int64_t)(gb * 32 + o) * taps + tap) * CG + c];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane & 7, vs = lane >> 3;
  const int cin0 = gb * 32 + ((4 * q) / CG) * CG;  // first input channel of this thread's group
  int64_t m[kV];
  int od[kV], oh[kV], ow[kV];
  bool ok[kV];
#pragma unroll
  for (int i = 0; i < kV; ++i) {
    m[i] = (int64_t)blockIdx.x * kVoxBlk + warp * 16 + vs + 4 * i;
    ok[i] = m[i] < a.M;
    // voxel counts < 2^31 (gconv_shape_ok): 32-bit divisions
    const unsigned mu = (unsigned)m[i], q1 = mu / (unsigned)a.Wo;
    ow[i] = (int)(mu - q1 * (unsigned)a.Wo);
    oh[i] = (int)(q1 % (unsigned)a.Ho);
    od[i] = (int)(q1 / (unsigned)a.Ho);
  }
  float4 acc[kV];
#pragma unroll
  for (int i = 0; i < kV; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int u = 0; u < a.k; ++u) {
    for (int v = 0; v < a.k; ++v) {
      const float* rp[kV];
      bool rv[kV];
#pragma unroll
      for (int i = 0; i < kV; ++i) {
        const int zi = od[i] * a.sd - a.pad + u, hi = oh[i] * a.s - a.pad + v;
        rv[i] = ok[i] && zi >= 0 && zi < a.D && hi >= 0 && hi < a.H;
        rp[i] = a.x + ((int64_t)(rv[i] ? zi : 0) * a.H + (rv[i] ? hi : 0)) * a.W * a.C + cin0;
      }
      for (int t = 0; t < a.k; ++t) {
        const float* wt = ws + ((u * a.k + v) * a.k + t) * CG * 32 + 4 * q;
        const float* xp[kV];
        bool xv_ok[kV];
#pragma unroll
        for (int i = 0; i < kV; ++i) {
          const int wi = ow[i] * a.s - a.pad + t;
          xv_ok[i] = rv[i] && wi >= 0 && wi < a.W;
          xp[i] = rp[i] + (int64_t)(xv_ok[i] ? wi : 0) * a.C;
        }
#pragma unroll
        for (int c4 = 0; c4 < CG / 4; ++c4) {
          float4 xv[kV];
#pragma unroll
          for (int i = 0; i < kV; ++i) xv[i] = xv_ok[i] ? ldg4(xp[i] + 4 * c4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const float4 w4 = *reinterpret_cast<const float4*>(wt + (4 * c4 + cc) * 32);
#pragma unroll
            for (int i = 0; i < kV; ++i) fma4(acc[i], f4c(xv[i], cc), w4);
          }
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kV; ++i)
    if (ok[i]) *reinterpret_cast<float4*>(a.out + m[i] * a.K + gb * 32 + 4 * q) = acc[i];
  if (!a.stat_sum) return;
  // BN partial sums of the block's 128 voxels: the thread's kV voxels, the four voxel lanes of
  // its quad (shuffles), then the eight warps in order (invalid voxels hold zeros)
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f), sq = s;
#pragma unroll
  for (int i = 0; i < kV; ++i) {
    s.x += acc[i].x; s.y += acc[i].y; s.z += acc[i].z; s.w += acc[i].w;
    sq.x = fmaf(acc[i].x, acc[i].x, sq.x); sq.y = fmaf(acc[i].y, acc[i].y, sq.y);
    sq.z = fmaf(acc[i].z, acc[i].z, sq.z); sq.w = fmaf(acc[i].w, acc[i].w, sq.w);
  }
#pragma unroll
  for (int off = 8; off < 32; off <<= 1) {
    s.x += __shfl_xor_sync(0xffffffffu, s.x, off); s.y += __shfl_xor_sync(0xffffffffu, s.y, off);
    s.z += __shfl_xor_sync(0xffffffffu, s.z, off); s.w += __shfl_xor_sync(0xffffffffu, s.w, off);
    sq.x += __shfl_xor_sync(0xffffffffu, sq.x, off); sq.y += __shfl_xor_sync(0xffffffffu, sq.y, off);
    sq.z += __shfl_xor_sync(0xffffffffu, sq.z, off); sq.w += __shfl_xor_sync(0xffffffffu, sq.w, off);
  }
  __shared__ float4 red[2][kThreads / 32][8];
  if (vs == 0) {
    red[0][warp][q] = s;
    red[1][warp][q] = sq;
  }
  __syncthreads();
  if (threadIdx.x < 16) {
    const int which = threadIdx.x >> 3, qq = threadIdx.x & 7;
    float4 r = red[which][0][qq];
    for (int w = 1; w < kThreads / 32; ++w) {
      const float4 e = red[which][w][qq];
      r.x += e.x; r.y += e.y; r.z += e.z; r.w += e.w;
    }
    float* dst = (which ? a.stat_sq : a.stat_sum) + (int64_t)blockIdx.x * a.K + gb * 32 + 4 * qq;
    *reinterpret_cast<float4*>(dst) = r;
  }
}

// ------------------------------------------------------------------------------ dgrad
// dx[in voxel][c] = sum over taps whose output position is an integer, sum_o dy[out][o] w[o][tap][c].
// Strides are uniform (1 or 2, S2). Stride 2: a warp owns 16 input voxels of one parity along W
// (every other voxel of 32), so its lanes skip the same taps.
template <int CG, bool S2>
__global__ void __launch_bounds__(kThreads) gconv_dgrad_kernel(GArgs a) {
  extern __shared__ float4 smem4[];
  float* wd = reinterpret_cast<float*>(smem4);  // [taps][CG (o)][32 (c of the block)]
  const int taps = a.k * a.k * a.k;
  const int gb = blockIdx.y;
  for (int i = threadIdx.x; i < taps * CG * 32; i += kThreads) {
    const int c32 = i & 31, o = (i >> 5) % CG, tap = i / (32 * CG);
    wd[i] = a.w[((int64_t)(gb * 32 + (c32 / CG) * CG + o) * taps + tap) * CG + (c32 % CG)];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane & 7, vs = lane >> 3;
  const int o0 = gb * 32 + ((4 * q) / CG) * CG;  // first dy channel of this thread's group
  const int64_t n_in = (int64_t)a.D * a.H * a.W;
  int64_t m[kV];
  int zi[kV], hi[kV], wi[kV];
  bool ok[kV];
#pragma unroll
  for (int i = 0; i < kV; ++i) {
    m[i] = S2 ? (int64_t)blockIdx.x * kVoxBlk + (warp >> 1) * 32 + (warp & 1) + 2 * (vs + 4 * i)
              : (int64_t)blockIdx.x * kVoxBlk + warp * 16 + vs + 4 * i;
    ok[i] = m[i] < n_in;
    const unsigned mu = (unsigned)m[i], q1 = mu / (unsigned)a.W;
    wi[i] = (int)(mu - q1 * (unsigned)a.W);
    hi[i] = (int)(q1 % (unsigned)a.H);
    zi[i] = (int)(q1 / (unsigned)a.H);
  }
  float4 acc[kV];
#pragma unroll
  for (int i = 0; i < kV; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int u = 0; u < a.k; ++u) {
    int odv[kV];
    bool zv[kV], any_z = false;
#pragma unroll
    for (int i = 0; i < kV; ++i) {
      zv[i] = ok[i] && tap_ok<(S2 ? 2 : 1)>(zi[i], u, a.pad, a.Do, odv[i]);
      any_z |= zv[i];
    }
    if (!any_z) continue;
    for (int v = 0; v < a.k; ++v) {
      int ohv[kV];
      bool hv[kV], any_h = false;
#pragma unroll
      for (int i = 0; i < kV; ++i) {
        hv[i] = zv[i] && tap_ok<(S2 ? 2 : 1)>(hi[i], v, a.pad, a.Ho, ohv[i]);
        any_h |= hv[i];
      }
      if (!any_h) continue;
      for (int t = 0; t < a.k; ++t) {
        const float* gp[kV];
        bool gv_ok[kV], any_w = false;
#pragma unroll
        for (int i = 0; i < kV; ++i) {
          int owv = 0;
          gv_ok[i] = hv[i] && tap_ok<(S2 ? 2 : 1)>(wi[i], t, a.pad, a.Wo, owv);
          any_w |= gv_ok[i];
          gp[i] = a.dy + (gv_ok[i] ? (((int64_t)odv[i] * a.Ho + ohv[i]) * a.Wo + owv) * a.K : 0) + o0;
        }
        if (!any_w) continue;
        const float* wt = wd + ((u * a.k + v) * a.k + t) * CG * 32 + 4 * q;
#pragma unroll
        for (int o4 = 0; o4 < CG / 4; ++o4) {
          float4 gv[kV];
#pragma unroll
          for (int i = 0; i < kV; ++i) gv[i] = gv_ok[i] ? ldg4(gp[i] + 4 * o4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int oo = 0; oo < 4; ++oo) {
            const float4 w4 = *reinterpret_cast<const float4*>(wt + (4 * o4 + oo) * 32);
#pragma unroll
            for (int i = 0; i < kV; ++i) fma4(acc[i], f4c(gv[i], oo), w4);
          }
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kV; ++i) {
    if (!ok[i]) continue;
    float* xp = a.out + m[i] * a.C + gb * 32 + 4 * q;
    float4 r = acc[i];
    if (a.accumulate) {
      const float4 e = *reinterpret_cast<const float4*>(xp);
      r.x += e.x; r.y += e.y; r.z += e.z; r.w += e.w;
    }
    *reinterpret_cast<float4*>(xp) = r;
  }
}

// ------------------------------------------------------------------------------ wgrad
// grid (chunks, K / 32, tap slices); out = ws[chunk][K][taps][CG] partials (or dw, one chunk).
// Per V-voxel tile: dy [V][32] and the TZ tap-shifted x tiles [TZ][V][32] are staged in
// shared memory (one thread per (voxel, quad), coordinates decoded once per tile, the taps from
// a table); then every thread accumulates its 4 x 4 (o, c) blocks over the tile's voxels. The
// block index puts the input-channel quad fastest, so a warp's x reads are whole 128-byte rows.
template <int CG, int TZ>
__global__ void __launch_bounds__(kThreads) gconv_wgrad_kernel(GArgs a) {
  constexpr int NG = 32 / CG;
  constexpr int Q = CG / 4;
  constexpr int NB4 = NG * TZ * Q * Q;
  constexpr int PER = (NB4 + kThreads - 1) / kThreads;
  constexpr int V = TZ > 9 ? 16 : 32;   // voxels per tile (smem: (1 + TZ) x V x 128 B)
  extern __shared__ float4 smem4[];
  float(*dys)[32] = reinterpret_cast<float(*)[32]>(smem4);
  float(*xs)[V][32] = reinterpret_cast<float(*)[V][32]>(reinterpret_cast<float*>(smem4) + V * 32);
  __shared__ int tap_uvt[TZ][3];
  __shared__ int vox_c[V][3];
  const int taps = a.k * a.k * a.k;
  const int gb = blockIdx.y;
  const int tap0 = blockIdx.z * TZ;
  if (threadIdx.x < TZ) {
    const int tap = tap0 + threadIdx.x;
    tap_uvt[threadIdx.x][0] = tap < taps ? tap / (a.k * a.k) : -1;
    tap_uvt[threadIdx.x][1] = (tap / a.k) % a.k;
    tap_uvt[threadIdx.x][2] = tap % a.k;
  }
  const int64_t m0 = (int64_t)blockIdx.x * a.chunk, m1 = min(a.M, m0 + a.chunk);
  float acc[PER][16];
#pragma unroll
  for (int p = 0; p < PER; ++p)
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[p][i] = 0.f;
  for (int64_t mt = m0; mt < m1; mt += V) {
    if (threadIdx.x < V) {
      const int64_t m = mt + threadIdx.x;
      const unsigned mu = (unsigned)m, q1 = mu / (unsigned)a.Wo;
      vox_c[threadIdx.x][0] = m < m1 ? (int)(q1 / (unsigned)a.Ho) * a.sd - a.pad : INT_MIN / 2;
      vox_c[threadIdx.x][1] = (int)(q1 % (unsigned)a.Ho) * a.s - a.pad;
      vox_c[threadIdx.x][2] = (int)(mu - q1 * (unsigned)a.Wo) * a.s - a.pad;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < V * 8; i += kThreads) {
      const int v = i >> 3, c4 = i & 7;
      const int64_t m = mt + v;
      float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
      if (m < m1) g = ldg4(a.dy + m * a.K + gb * 32 + 4 * c4);
      *reinterpret_cast<float4*>(&dys[v][4 * c4]) = g;
    }
    for (int i = threadIdx.x; i < TZ * V * 8; i += kThreads) {
      const int c4 = i & 7, v = (i >> 3) % V, tz = i / (8 * V);
      float4 xv = make_float4(0.f, 0.f, 0.f, 0.f);
      const int u = tap_uvt[tz][0];
      if (u >= 0) {
        const int zi = vox_c[v][0] + u, hi = vox_c[v][1] + tap_uvt[tz][1], wi = vox_c[v][2] + tap_uvt[tz][2];
        if (zi >= 0 && zi < a.D && hi >= 0 && hi < a.H && wi >= 0 && wi < a.W)
          xv = ldg4(a.x + (((int64_t)zi * a.H + hi) * a.W + wi) * a.C + gb * 32 + 4 * c4);
      }
      *reinterpret_cast<float4*>(&xs[tz][v][4 * c4]) = xv;
    }
    __syncthreads();
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      const int b = threadIdx.x + p * kThreads;
      if (b < NB4) {
        const int c4 = b % Q, o4 = (b / Q) % Q, j = (b / (Q * Q)) % NG, tz = b / (Q * Q * NG);
        const int oc = j * CG + 4 * o4, xc = j * CG + 4 * c4;
#pragma unroll 4
        for (int v = 0; v < V; ++v) {
          const float4 g = *reinterpret_cast<const float4*>(&dys[v][oc]);
          const float4 xv = *reinterpret_cast<const float4*>(&xs[tz][v][xc]);
#pragma unroll
          for (int oo = 0; oo < 4; ++oo)
#pragma unroll
            for (int cc = 0; cc < 4; ++cc)
              acc[p][oo * 4 + cc] = fmaf(f4c(g, oo), f4c(xv, cc), acc[p][oo * 4 + cc]);
        }
      }
    }
    __syncthreads();
  }
  float* dst = a.out + (int64_t)blockIdx.x * a.K * taps * CG;
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    const int b = threadIdx.x + p * kThreads;
    if (b >= NB4) continue;
    const int c4 = b % Q, o4 = (b / Q) % Q, j = (b / (Q * Q)) % NG, tz = b / (Q * Q * NG);
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

// wgrad for narrow groups (Cg = 4, 8; 3^3 taps): a staged x tile would be consumed by exactly one
// (or two) threads, so each thread -- one (tap, group, o quad, c quad) 4 x 4 block of dw -- streams
// its own tap-shifted x rows and the dy rows straight from L1 / L2 over the block's voxel chunk:
// a warp (4 taps x 8 channel quads, Cg = 4) reads one 128-byte dy row and four 128-byte x rows per
// voxel for 16 FMAs each, with no shared memory and no barriers.
template <int CG>
__global__ void __launch_bounds__(CG == 4 ? 224 : 448) gconv_wgrad_direct_kernel(GArgs a) {
  constexpr int NG = 32 / CG, Q = CG / 4, NB = NG * 27 * Q * Q;
  const int b = threadIdx.x;
  if (b >= NB) return;
  const int c4 = b % Q, o4 = (b / Q) % Q, j = (b / (Q * Q)) % NG, tap = b / (Q * Q * NG);
  const int u = tap / 9, v = (tap / 3) % 3, t = tap % 3;
  const int gb = blockIdx.y;
  const int oc = gb * 32 + j * CG + 4 * o4, xc = gb * 32 + j * CG + 4 * c4;
  // this block's output rows (od, oh) [r0, r1): a.chunk rows each
  const int64_t rows = (int64_t)a.Do * a.Ho;
  const int64_t r0 = (int64_t)blockIdx.x * a.chunk, r1 = min(rows, r0 + a.chunk);
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.f;
  for (int64_t r = r0; r < r1; ++r) {
    const int od = (int)(r / a.Ho), oh = (int)(r - (int64_t)od * a.Ho);
    const int zi = od * a.sd - a.pad + u, hi = oh * a.s - a.pad + v;
    if (zi < 0 || zi >= a.D || hi < 0 || hi >= a.H) continue;   // this tap reads padding: no term
    const float* xrow = a.x + ((int64_t)zi * a.H + hi) * a.W * a.C + xc;
    const float* gp = a.dy + r * a.Wo * a.K + oc;
#pragma unroll 4
    for (int ow = 0; ow < a.Wo; ++ow) {
      const int wi = ow * a.s - a.pad + t;
      const bool ok = wi >= 0 && wi < a.W;
      const float4 g = ldg4(gp + (int64_t)ow * a.K);
      const float4 xr = ldg4(xrow + (int64_t)(ok ? wi : 0) * a.C);
      const float4 xv = ok ? xr : make_float4(0.f, 0.f, 0.f, 0.f);
      const float ga[4] = {g.x, g.y, g.z, g.w}, xa[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
      for (int oo = 0; oo < 4; ++oo)
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) acc[oo * 4 + cc] = fmaf(ga[oo], xa[cc], acc[oo * 4 + cc]);
    }
  }
  float* dst = a.out + (int64_t)blockIdx.x * a.K * 27 * CG;
#pragma unroll
  for (int oo = 0; oo < 4; ++oo) {
    const int o = gb * 32 + j * CG + 4 * o4 + oo;
    *reinterpret_cast<float4*>(dst + ((int64_t)o * 27 + tap) * CG + 4 * c4) =
        make_float4(acc[oo * 4], acc[oo * 4 + 1], acc[oo * 4 + 2], acc[oo * 4 + 3]);
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

int wgrad_v(int cg) { return wgrad_tz(cg) > 9 ? 16 : 32; }

bool wgrad_direct(const ConvGeom& g) { return g.R == 3 && cg_of(g) == 4; }   // Cg = 8: the staged tile (measured faster)

int wgrad_chunks(const ConvGeom& g) {
  const int taps = g.R * g.R * g.R;
  const int tz = wgrad_tz(cg_of(g));
  const int per_chunk = (g.K / 32) * (wgrad_direct(g) ? 1 : (taps + tz - 1) / tz);
  const int64_t M = (int64_t)g.Do * g.Ho * g.Wo;
  // ~4 waves of 148 SMs, at least 8 tiles per chunk
  int64_t ch = std::max<int64_t>(1, (4 * 148 + per_chunk - 1) / per_chunk);
  ch = std::min<int64_t>(ch, std::max<int64_t>(1, M / (8 * wgrad_v(cg_of(g)))));
  if (wgrad_direct(g)) ch = std::min<int64_t>(ch, (int64_t)g.Do * g.Ho);   // whole rows per chunk
  return (int)std::min<int64_t>(ch, 512);
}

template <typename Kern>
pooch_status set_smem(Kern k, int bytes) {
  if (bytes > 48 * 1024) POOCH_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  return POOCH_OK;
}

template <int CG>
pooch_status launch_dgrad(dim3 grid, int smem, cudaStream_t st, const GArgs& a, bool s2) {
  if (s2) {
    POOCH_CHECK(set_smem(gconv_dgrad_kernel<CG, true>, smem));
    gconv_dgrad_kernel<CG, true><<<grid, kThreads, smem, st>>>(a);
  } else {
    POOCH_CHECK(set_smem(gconv_dgrad_kernel<CG, false>, smem));
    gconv_dgrad_kernel<CG, false><<<grid, kThreads, smem, st>>>(a);
  }
  return POOCH_OK;
}

}  // namespace

bool gconv_shape_ok(const ConvGeom& g) {
  const int cg = g.groups > 0 ? g.C / g.groups : 0;
  return g.is3d() && g.groups > 1 && g.C == g.K && g.C % g.groups == 0 &&
         (int64_t)g.D * g.H * g.W < (1ll << 31) && (int64_t)g.Do * g.Ho * g.Wo < (1ll << 31) &&
         (cg == 4 || cg == 8 || cg == 16 || cg == 32) && g.K % 32 == 0 && (g.R == 1 || g.R == 3) && g.R == g.S &&
         g.stride >= 1 && g.stride <= 2 && g.sd() == g.stride && g.N == 1;
}

int gconv_stat_tiles(const ConvGeom& g) {
  return (int)(((int64_t)g.Do * g.Ho * g.Wo + kVoxBlk - 1) / kVoxBlk);
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
    case 4: POOCH_CHECK(set_smem(gconv_fwd_kernel<4>, smem)); gconv_fwd_kernel<4><<<grid, kThreads, smem, st>>>(a); break;
    case 8: POOCH_CHECK(set_smem(gconv_fwd_kernel<8>, smem)); gconv_fwd_kernel<8><<<grid, kThreads, smem, st>>>(a); break;
    case 16: POOCH_CHECK(set_smem(gconv_fwd_kernel<16>, smem)); gconv_fwd_kernel<16><<<grid, kThreads, smem, st>>>(a); break;
    case 32: POOCH_CHECK(set_smem(gconv_fwd_kernel<32>, smem)); gconv_fwd_kernel<32><<<grid, kThreads, smem, st>>>(a); break;
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
  dim3 grid((unsigned)((n_in + kVoxBlk - 1) / kVoxBlk), g.C / 32);
  const bool s2 = g.stride == 2;
  if (n_in == 0) return POOCH_OK;
  count_launch();
  switch (cg) {
    case 4: POOCH_CHECK(launch_dgrad<4>(grid, smem, st, a, s2)); break;
    case 8: POOCH_CHECK(launch_dgrad<8>(grid, smem, st, a, s2)); break;
    case 16: POOCH_CHECK(launch_dgrad<16>(grid, smem, st, a, s2)); break;
    case 32: POOCH_CHECK(launch_dgrad<32>(grid, smem, st, a, s2)); break;
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
  // voxels per chunk; the direct kernel takes whole output rows (od, oh) per chunk
  a.chunk = wgrad_direct(g) ? ((int64_t)g.Do * g.Ho + chunks - 1) / chunks : (a.M + chunks - 1) / chunks;
  const int taps = g.R * g.R * g.R, cg = cg_of(g), tz = wgrad_tz(cg);
  dim3 grid(chunks, g.K / 32, (taps + tz - 1) / tz);
  const int smem = (1 + tz) * wgrad_v(cg) * 32 * (int)sizeof(float);
  count_launch();
  if (wgrad_direct(g)) {
    grid.z = 1;
    if (cg == 4)
      gconv_wgrad_direct_kernel<4><<<grid, 224, 0, st>>>(a);
    else
      gconv_wgrad_direct_kernel<8><<<grid, 448, 0, st>>>(a);
  } else switch (cg) {
    case 4: POOCH_CHECK(set_smem(gconv_wgrad_kernel<4, 27>, smem)); gconv_wgrad_kernel<4, 27><<<grid, kThreads, smem, st>>>(a); break;
    case 8: POOCH_CHECK(set_smem(gconv_wgrad_kernel<8, 27>, smem)); gconv_wgrad_kernel<8, 27><<<grid, kThreads, smem, st>>>(a); break;
    case 16: POOCH_CHECK(set_smem(gconv_wgrad_kernel<16, 9>, smem)); gconv_wgrad_kernel<16, 9><<<grid, kThreads, smem, st>>>(a); break;
    case 32: POOCH_CHECK(set_smem(gconv_wgrad_kernel<32, 3>, smem)); gconv_wgrad_kernel<32, 3><<<grid, kThreads, smem, st>>>(a); break;
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
