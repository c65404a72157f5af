// alex.cu -- the memory-bound kernels of the AlexNet workload:
// local response normalisation across channels, the ReLU-mask + bias-gradient pass of the
// conv / FC layers, counter-based inverted dropout, and the dropout step counter. NHWC fp32.
//
// Conv / FC forward with bias + ReLU runs in the tensor-core kernels' epilogue (igemm.cuh,
// GemmParams::relu); these kernels do the rest. All reductions are deterministic: per-block
// partial sums over fixed row ranges in a fixed order, then an fp64 sum over blocks in order.
#include <algorithm>

#include "alex.h"
#include "common.h"

namespace pooch {

namespace {

constexpr int kLrnPix = 16;       // pixels per LRN block (their C channels staged in shared memory)
constexpr int kSumBlocks = 592;   // 4 x 148 SMs: blocks of the per-channel reductions

__device__ __forceinline__ float lrn_pow(float s, float e) { return exp2f(e * log2f(s)); }

// y[p][c] = x[p][c] * s^(-beta), s = k + alpha / n * sum_{|c' - c| <= n/2} x[p][c']^2
__global__ void lrn_fwd_kernel(const float* __restrict__ x, float* __restrict__ y, int64_t pixels, int C, int half,
                               float k, float an, float beta) {
  extern __shared__ float sm[];   // [kLrnPix][C] of x^2
  const int64_t p0 = (int64_t)blockIdx.x * kLrnPix;
  const int np = (int)(pixels - p0 < kLrnPix ? pixels - p0 : kLrnPix);
  const int total = np * C;
  const float* xb = x + p0 * C;
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    const float v = xb[i];
    sm[i] = v * v;
  }
  __syncthreads();
  float* yb = y + p0 * C;
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    const int c = i % C, row = i - c;
    float s = 0.f;
    for (int j = max(0, c - half); j <= min(C - 1, c + half); ++j) s += sm[row + j];  // fixed order
    yb[i] = xb[i] * lrn_pow(k + an * s, -beta);
  }
}

// gx[c] = gy[c] s_c^(-beta) - (2 alpha beta / n) x[c] sum_{|j - c| <= n/2} gy[j] x[j] s_j^(-beta - 1)
__global__ void lrn_bwd_kernel(const float* __restrict__ x, const float* __restrict__ gy, float* __restrict__ gx,
                               int64_t pixels, int C, int half, float k, float an, float beta, float coef) {
  extern __shared__ float sm[];   // [2][kLrnPix][C]: x^2, then s; t
  const int64_t p0 = (int64_t)blockIdx.x * kLrnPix;
  const int np = (int)(pixels - p0 < kLrnPix ? pixels - p0 : kLrnPix);
  const int total = np * C;
  float* sq = sm;
  float* tt = sm + kLrnPix * C;
  const float* xb = x + p0 * C;
  const float* gb = gy + p0 * C;
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    const float v = xb[i];
    sq[i] = v * v;
  }
  __syncthreads();
  float sv[8];   // this thread's s values (i = threadIdx.x + r * blockDim.x), reused below
  int r = 0;
  for (int i = threadIdx.x; i < total; i += blockDim.x, ++r) {
    const int c = i % C, row = i - c;
    float s = 0.f;
    for (int j = max(0, c - half); j <= min(C - 1, c + half); ++j) s += sq[row + j];
    s = k + an * s;
    if (r < 8) sv[r] = s;
    tt[i] = gb[i] * xb[i] * lrn_pow(s, -beta - 1.f);
  }
  __syncthreads();
  float* ob = gx + p0 * C;
  r = 0;
  for (int i = threadIdx.x; i < total; i += blockDim.x, ++r) {
    const int c = i % C, row = i - c;
    float s;
    if (r < 8) {
      s = sv[r];
    } else {
      float q = 0.f;
      for (int j = max(0, c - half); j <= min(C - 1, c + half); ++j) q += sq[row + j];
      s = k + an * q;
    }
    float a = 0.f;
    for (int j = max(0, c - half); j <= min(C - 1, c + half); ++j) a += tt[row + j];
    ob[i] = gb[i] * lrn_pow(s, -beta) - coef * xb[i] * a;
  }
}

// g = y > 0 ? g * scale : 0 (in place), and per-block partial column sums of the result:
// part[block][c]. Block b owns rows [b * per, (b + 1) * per); threads cover columns in float4
// groups, rows strided by rows-per-iteration; the block's sums are combined in row-group order.
__global__ void relu_mask_sum_kernel(float* __restrict__ g, const float* __restrict__ y, int64_t rows, int C,
                                     float scale, float* __restrict__ part) {
  extern __shared__ float red[];   // [rpi][C]
  const int C4 = C / 4;
  const int tpr = min(C4, (int)blockDim.x);        // threads per row
  const int rpi = blockDim.x / tpr;                // rows per iteration
  const int tid = threadIdx.x;
  const int ro = tid / tpr, cg0 = tid % tpr;
  const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(rows, r0 + per);
  for (int cg = cg0; cg < C4; cg += tpr) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (ro < rpi) {
      for (int64_t r = r0 + ro; r < r1; r += rpi) {
        const size_t o = (size_t)r * C + 4 * cg;
        float4 gv = *reinterpret_cast<const float4*>(g + o);
        const float4 yv = *reinterpret_cast<const float4*>(y + o);
        gv.x = yv.x > 0.f ? gv.x * scale : 0.f;
        gv.y = yv.y > 0.f ? gv.y * scale : 0.f;
        gv.z = yv.z > 0.f ? gv.z * scale : 0.f;
        gv.w = yv.w > 0.f ? gv.w * scale : 0.f;
        *reinterpret_cast<float4*>(g + o) = gv;
        acc.x += gv.x; acc.y += gv.y; acc.z += gv.z; acc.w += gv.w;
      }
      *reinterpret_cast<float4*>(red + (size_t)ro * C + 4 * cg) = acc;
    }
  }
  __syncthreads();
  for (int c = tid; c < C; c += blockDim.x) {
    float s = 0.f;
    for (int q = 0; q < rpi; ++q) s += red[(size_t)q * C + c];
    part[(size_t)blockIdx.x * C + c] = s;
  }
}

__global__ void colsum_blocks_kernel(const float* __restrict__ part, int blocks, int C, float* __restrict__ out,
                                     int accumulate) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double s = 0;
  for (int b = 0; b < blocks; ++b) s += (double)part[(size_t)b * C + c];
  out[c] = accumulate ? out[c] + (float)s : (float)s;
}

__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}

// inverted dropout in place on y [rows][C] (already ReLU'd): element i (row-major) is kept iff
// fmix32(key ^ fmix32(i)) >= thresh, key = fmix32(seed ^ fmix32(step * 0x9E3779B9 + task)), with
// (seed, step) read from device memory so a replayed CUDA graph draws the current step's mask
__global__ void dropout_kernel(float* __restrict__ y, int64_t n, const uint32_t* __restrict__ rng, int task,
                               uint32_t thresh, float scale) {
  const uint32_t key = fmix32(rng[0] ^ fmix32(rng[1] * 0x9E3779B9u + (uint32_t)task));
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t u = fmix32(key ^ fmix32((uint32_t)i));
    y[i] = u >= thresh ? y[i] * scale : 0.f;
  }
}

__global__ void rng_advance_kernel(uint32_t* rng) { rng[1] += 1u; }

int blocks_for(int64_t n, int per) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + per - 1) / per, 148 * 8)); }

}  // namespace

pooch_status lrn_fwd(const float* x, float* y, int64_t pixels, int C, cudaStream_t st) {
  if (C > 1024) return fail(POOCH_EUSAGE, "LRN: C <= 1024");
  const int64_t blocks = (pixels + kLrnPix - 1) / kLrnPix;
  count_launch();
  lrn_fwd_kernel<<<(unsigned)blocks, 256, kLrnPix * C * sizeof(float), st>>>(
      x, y, pixels, C, kLrnN / 2, kLrnK, kLrnAlpha / kLrnN, kLrnBeta);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

pooch_status lrn_bwd(const float* x, const float* gy, float* gx, int64_t pixels, int C, cudaStream_t st) {
  if (C > 1024) return fail(POOCH_EUSAGE, "LRN: C <= 1024");
  const int64_t blocks = (pixels + kLrnPix - 1) / kLrnPix;
  count_launch();
  lrn_bwd_kernel<<<(unsigned)blocks, 256, 2 * kLrnPix * C * sizeof(float), st>>>(
      x, gy, gx, pixels, C, kLrnN / 2, kLrnK, kLrnAlpha / kLrnN, kLrnBeta, 2.f * kLrnAlpha * kLrnBeta / kLrnN);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

size_t relu_mask_sum_ws_bytes(int C) { return (size_t)kSumBlocks * C * sizeof(float); }

pooch_status relu_mask_sum(float* g, const float* y, int64_t rows, int C, float scale, float* db, float* ws,
                           cudaStream_t st) {
  if (C % 4) return fail(POOCH_EUSAGE, "relu_mask_sum: C % 4 == 0");
  const int blocks = (int)std::min<int64_t>(kSumBlocks, std::max<int64_t>(1, (rows + 15) / 16));
  const int tpr = std::min(C / 4, 256);
  const int rpi = 256 / tpr;
  count_launch();
  relu_mask_sum_kernel<<<blocks, 256, (size_t)rpi * C * sizeof(float), st>>>(g, y, rows, C, scale, ws);
  count_launch();
  colsum_blocks_kernel<<<(C + 127) / 128, 128, 0, st>>>(ws, blocks, C, db, 0);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

pooch_status dropout_fwd(float* y, int64_t n, const uint32_t* rng, int task, float ratio, cudaStream_t st) {
  if (ratio <= 0.f) return POOCH_OK;
  if (ratio >= 1.f) return fail(POOCH_EUSAGE, "dropout ratio must be < 1");
  const double t = std::min((double)ratio * 4294967296.0, 4294967295.0);
  count_launch();
  dropout_kernel<<<blocks_for(n, 256), 256, 0, st>>>(y, n, rng, task, (uint32_t)t, 1.f / (1.f - ratio));
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

pooch_status rng_advance(uint32_t* rng, cudaStream_t st) {
  count_launch();
  rng_advance_kernel<<<1, 1, 0, st>>>(rng);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

}  // namespace pooch

using namespace pooch;

extern "C" pooch_status pooch_op_lrn_fwd(const float* x, float* y, int64_t pixels, int32_t C, void* stream) {
  if (!x || !y || pixels <= 0 || C <= 0 || C > 1024) return fail(POOCH_EUSAGE, "lrn_fwd: bad arguments");
  return lrn_fwd(x, y, pixels, C, (cudaStream_t)stream);
}

extern "C" pooch_status pooch_op_lrn_bwd(const float* x, const float* gy, float* gx, int64_t pixels, int32_t C,
                                         void* stream) {
  if (!x || !gy || !gx || pixels <= 0 || C <= 0 || C > 1024) return fail(POOCH_EUSAGE, "lrn_bwd: bad arguments");
  return lrn_bwd(x, gy, gx, pixels, C, (cudaStream_t)stream);
}
