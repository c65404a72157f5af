// igemm.cuh -- implicit-GEMM convolution / FC core on 5th-gen tensor cores (sm_100a).
//
// One CTA computes a 128 x BN fp32 tile D = A * B^T with tcgen05.mma kind::tf32
// (TF32 in, FP32 accumulate in TMEM), K consumed in blocks of 32 elements.
//
// Persistent and warp-specialised (igemm_kernel below): each CTA walks tiles with a stride of
// the grid and two TMEM accumulators, so the epilogue of tile i overlaps the mainloop of i+1.
//   warps 0-3  : epilogue -- tcgen05.ld TMEM -> registers -> fused epilogue (bias / ReLU, BN
//                partial sums) -> swizzled smem staging -> TMA store (or coalesced stores).
//                E2: warps 4-7 form a second epilogue group that drains the other half of the
//                accumulator's columns (a warp may only read TMEM lane quadrant warp % 4).
//   warps 4-7  : producers -- cp.async gathers of 16-B chunks into SWIZZLE_NONE core matrices,
//                or (TMA) one elected thread issuing the tensor-memory-accelerator boxes
//                (E2: that thread is warp 13).
//   warp 8     : TMEM allocator + single-thread MMA issuer (tcgen05.mma, tcgen05.commit).
//   warps 9-12 : auxiliary (3xTF32 residuals, wgrad transposes, AT: A hi / lo into TMEM).
//
// Pipeline: STAGES smem slots, mbarrier full/empty ring (TMA: expect-tx arrivals; 3xTF32: the
// auxiliary warps publish each stage after writing its residuals); the MMA thread's
// tcgen05.commit arrives on empty[] when the tensor core is done reading the slot and on
// tfull[] when an accumulator is complete.
//
// Modes (which tensors A and B are, and what the epilogue does):
//   CONV_FWD  : A = im2col(x) [M=N*Ho*Wo, K=R*S*C] (K-major gather), B = W [Cout, R*S*C];
//               epilogue stores y (NHWC) + deterministic per-tile BN partial sums.
//   CONV_DGRAD: A = dy gathered by the transposed-conv rule [M=N*H*W, K=R*S*Cout],
//               B = Wt [C, R*S*Cout]; epilogue stores (or accumulates into) dx.
//   CONV_WGRAD: A = dy^T [Cout, K=N*Ho*Wo], B = im2col(x)^T [R*S*C, K]; both are strided along
//               K in NHWC: the TMA path loads them MN-major (MNW: fed to the MMA as loaded; XF:
//               transposed in place by the auxiliary warps); the cp.async path gathers 16-B
//               (4-channel) chunks into 4x4 blocks that the auxiliary warps transpose
//               (WLoader / transpose_block);
//               split-K over pixels, the epilogue stores the split's partial dW (KRSC).
//   GEMM_TEST : plain K-major A [M][K], B [N][K], for unit tests of the core.
// (Operands are K-major -- SWIZZLE_NONE core matrices or SWIZZLE_128B TMA tiles -- except the
//  MNW wgrad, whose TMA boxes stay MN-major in the SWIZZLE_128B_BASE32B layout, the one MN-major
//  layout tcgen05 accepts for tf32.)
#pragma once
#include <cuda.h>

#include <cstdint>
#include <type_traits>

#include "ptx.cuh"

namespace pooch {

enum GemmMode { CONV_FWD = 0, CONV_DGRAD = 1, CONV_WGRAD = 2, GEMM_TEST = 3 };

struct GemmParams {
  // conv geometry (NHWC activations, KRSC weights)
  int N, H, W, C;        // input
  int K, R, S;           // output channels, filter
  int Ho, Wo, stride, pad;
  // GEMM view
  int M, Ng, Kg;
  // operands
  const float* a;        // FWD: x, DGRAD: dy, WGRAD: dy, TEST: A
  const float* b;        // FWD: W, DGRAD: Wt, WGRAD: x, TEST: B
  float* d;              // FWD: y, DGRAD: dx, WGRAD: partial ws [split][Cout][RSC], TEST: D
  int lda, ldb, ldd;     // TEST only
  // epilogue extras
  float* stat_sum;       // FWD: [Mtiles][K] per-tile column sums (nullptr: skip stats)
  float* stat_sq;        // FWD: [Mtiles][K] per-tile column sums of squares
  const float* bias;     // FWD (FC): per-column bias, nullable
  int accumulate;        // DGRAD: dx += result
  int kb_per_split;      // WGRAD / TEST: k-blocks handled by one blockIdx.z
  // TMA-fed FWD / DGRAD: an M-tile is a TW x TH x TN box of output pixels (rows = TW*TH*TN <= 128)
  int tw, th, tn;        // box of output pixels per tile
  int tiles_w, tiles_h, tiles_n;
  int hout, wout;        // output pixel grid of this GEMM (FWD: Ho x Wo, DGRAD: H x W)
  int cchunks;           // 32-channel chunks of the reduced channel dim (FWD: C/32, DGRAD: K/32)
  // TMA-fed WGRAD: a k-block is a TW x TH x TN box of 32 output pixels (tiles_* count the boxes);
  // wg_a_is_x = 1: A = im2col(x)^T [R*S*C] and B = dy^T [Cout] (the transposed orientation)
  int wg_a_is_x;
  int wg_cba, wg_cbb;    // 32-channel chunks per TMA box of A / B (5-D maps, chunk index outermost)
  // TMA-fed DGRAD, one output-parity class (a, b) of a stride-st conv: dx pixels (st*i + a, st*j + b)
  // receive the taps r = dg_r0 + st*t (t < dg_nr), s = dg_s0 + st*u (u < dg_ns) from dy pixel
  // (i + (a + pad - r)/st, j + (b + pad - s)/st); stride 1 is the single class a = b = 0
  int dg_a, dg_b, dg_r0, dg_s0, dg_nr, dg_ns;
  // TMA paths, fourth tensor dimension: images (2D: no taps, st3 = 1, pad3 = 0) or depth of a
  // 3D conv (batch 1): T taps, stride st3, padding pad3; n3 = extent of the output grid's fourth
  // dimension (PIXM epilogue); DGRAD classes along it: dg_c, dg_t0, dg_nt
  int T, st3, pad3, n3;
  int dg_c, dg_t0, dg_nt;
  // two-source input (a channel concatenation read in place): FWD A / WGRAD x channels
  // [c_split, C) come from the third tensor map; DGRAD columns [n_split, Ng) go to d2
  int c_split, n_split, accumulate2;
  float* d2;
  int epi_direct;        // 1: each thread stores its own row (no smem staging); experiments only
  // epilogue stores through the TMA (tma_d): 1 = 4-D box of output pixels {32 ch, tw, th, tn}
  // (PIXM, one dgrad class of stride 1), 2 = 2-D {32 cols, 128 rows} of a row-major [M][Ng]
  int tma_store;
  // TMA-fed FWD over a 4-channel input (the stem): a k-block is 8 taps x 4 channels; per tap one
  // 16-B-wide box of A (SWIZZLE_NONE, the K-major core-matrix layout) and one of B (stem4 = 1);
  // stem4 = 2 (SP kernels): one input patch per tile, the A rows gathered from it (patch_w = its
  // width in pixels)
  int stem4;
  int patch_w;
  // transform on load (XF kernels): the activation operand (FWD: A = x, WGRAD: x)
  // is relu(xf_scale[c] * v + xf_shift[c]) of the stored tensor; zero padding stays zero
  const float* xf_scale;
  const float* xf_shift;
  int relu;              // FWD: the epilogue applies max(v, 0) after the bias (AlexNet conv / FC)
};

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 elements per k-block (128 B per row)
constexpr int NUM_THREADS = 160;

template <int BN, int STAGES, bool X3 = false, bool AT = false, int NSTG = 1, int NEG = 1, bool SP = false>
struct GemmSmem {
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = BN * BK * 4;
  // 3xTF32: the stage also holds the residuals As = A - tf32(A), Bs = B - tf32(B) (AT: As lives
  // in TMEM, the stage is [A][B][Bs])
  // SP: no smem stages (A goes to TMEM from the patch); the whole weight matrix (<= 8 k-blocks)
  // and its residuals stay resident at offset 0: B of k-block kb at kb * B_BYTES, Bs at + BS_OFF
  static constexpr int SP_KB = 8;
  static constexpr int STAGE_BYTES = SP ? 0 : (AT ? A_BYTES + 2 * B_BYTES : (A_BYTES + B_BYTES) * (X3 ? 2 : 1));
  static constexpr int SMALL_OFF = A_BYTES + B_BYTES;
  static constexpr int BS_OFF = SP ? SP_KB * B_BYTES : (AT ? B_BYTES : SMALL_OFF);  // Bs relative to the B tile
  static constexpr int BAR_OFF = SP ? 2 * SP_KB * B_BYTES : STAGES * STAGE_BYTES;
  static constexpr int RED_OFF = BAR_OFF + (3 * STAGES + 16) * 8 + 16;
  // epilogue staging: per epilogue warp one 32 x 32 fp32 block (4 KB); together the 128 x 32
  // SWIZZLE_128B image of one column chunk of the tile (1024-B aligned for the TMA store)
  static constexpr int STG_OFF = (RED_OFF + 4 * BN * 4 * 2 + 1023) / 1024 * 1024;
  // NSTG = 2: two staging images, so a column chunk is staged while the TMA still reads the last;
  // NEG = 2 epilogue warp groups, each with its own NSTG images
  // SP: NPB input-patch buffers of up to 13 KB, loaded NPB - 1 tiles ahead
  static constexpr int NPB = 4;
  static constexpr int PATCH_BYTES = 13312;
  static constexpr int PATCH_OFF = STG_OFF + NEG * NSTG * 4 * 4096;
  static constexpr int TOTAL = PATCH_OFF + (SP ? NPB * PATCH_BYTES : 0) + 1024;
};

// ---------------------------------------------------------------------------------------
// K-major operand tile of ROWS rows x 32 k: chunk (row, j) -> ((j*(ROWS/8) + row/8)*128 + (row%8)*16)
template <int ROWS>
__device__ __forceinline__ uint32_t kmaj_off(int row, int j) {
  return (uint32_t)((j * (ROWS / 8) + (row >> 3)) * 128 + (row & 7) * 16);
}
// 3xTF32 split: the tensor core truncates fp32 operands to TF32 (measured, DESIGN.md
// Reading 27), so A*B ~= A*B + A*Bs + As*B with As = A - trunc_tf32(A) recovers ~fp32
// accuracy from three TF32 MMAs.
__device__ __forceinline__ float tf32_resid(float x) {
  return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}
// BN-ReLU on load (XF): y = relu(fma(v, scale, shift)) -- the BN-apply kernel's arithmetic
// (eltwise.cu bn_apply_kernel mode 0), so the fused and the stored paths agree bit for bit
__device__ __forceinline__ float bnrelu1(float v, float sc, float sh) { return fmaxf(__fmaf_rn(v, sc, sh), 0.f); }
__device__ __forceinline__ void split_chunk(uint32_t src, uint32_t dst) {
  float a, b, c, d;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "r"(src));
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "f"(tf32_resid(a)), "f"(tf32_resid(b)),
               "f"(tf32_resid(c)), "f"(tf32_resid(d))
               : "memory");
}

// ------------------------------------------------------------------------------ loaders
// Each producer thread (tid 0..127; warp w = tid/32, lane l) owns a fixed set of tile rows
// (K-major: ROWS/32 rows, 2 chunk columns) or MN groups (MN-major) for the whole k loop.

// ---- K-major row gathers (FWD A/B, DGRAD A/B, TEST K-major)
template <int MODE, int ROWS, bool IS_A>
struct KLoader {
  static constexpr int RPT = ROWS / 32;
  const float* rowp[RPT];   // FWD-A: image base of row's sample; B: row pointer
  int hi0[RPT], wi0[RPT];   // FWD-A: top-left input coords; DGRAD-A: h+pad, w+pad
  int nimg[RPT];
  bool valid[RPT];
  int lane, warp;
  // FWD-A with C < 32 (the stem): the tap (tr, ts) and channel tc of this thread's two 16-B
  // chunk columns for k-block cur, advanced incrementally (32 / C taps per k-block) instead of
  // re-deriving them with runtime divisions every k-block
  int tr[2], ts[2], tc[2];
  int cur = -2;

  __device__ void init(const GemmParams& p, int row0, int tid) {
    warp = tid >> 5;
    lane = tid & 31;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      int r = warp * (ROWS / 4) + i * 8 + (lane & 7);
      int gr = row0 + r;
      if constexpr (IS_A && MODE == CONV_FWD) {
        valid[i] = gr < p.M;
        int g = valid[i] ? gr : 0;
        int wo = g % p.Wo;
        int t = g / p.Wo;
        int ho = t % p.Ho;
        int n = t / p.Ho;
        rowp[i] = p.a + (size_t)n * p.H * p.W * p.C;
        hi0[i] = ho * p.stride - p.pad;
        wi0[i] = wo * p.stride - p.pad;
      } else if constexpr (IS_A && MODE == CONV_DGRAD) {
        valid[i] = gr < p.M;
        int g = valid[i] ? gr : 0;
        int w = g % p.W;
        int t = g / p.W;
        int h = t % p.H;
        int n = t / p.H;
        rowp[i] = p.a + (size_t)n * p.Ho * p.Wo * p.K;
        hi0[i] = h + p.pad;
        wi0[i] = w + p.pad;
      } else if constexpr (MODE == GEMM_TEST) {
        int lim = IS_A ? p.M : p.Ng;
        int ld = IS_A ? p.lda : p.ldb;
        valid[i] = gr < lim;
        rowp[i] = (IS_A ? p.a : p.b) + (size_t)(valid[i] ? gr : 0) * ld;
      } else {  // B operand of FWD / DGRAD: plain rows of the (transposed) weight
        valid[i] = gr < p.Ng;
        rowp[i] = p.b + (size_t)(valid[i] ? gr : 0) * p.Kg;
      }
    }
  }

  // residuals of the chunks this thread loaded into the tile at sbase -> tile at sbase + delta
  __device__ void split(uint32_t sbase, uint32_t delta) const {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int j = (lane >> 3) + 4 * h;
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        int row = warp * (ROWS / 4) + i * 8 + (lane & 7);
        uint32_t a = sbase + kmaj_off<ROWS>(row, j);
        split_chunk(a, a + delta);
      }
    }
  }

  __device__ void load(const GemmParams& p, uint32_t sbase, int kb) {
    if constexpr (IS_A && MODE == CONV_FWD) {
      if (p.C < BK && BK % p.C == 0) {
        if (kb == cur + 1) {  // next k-block: 32 / C more taps (at most a couple of row wraps)
          const int adv = BK / p.C;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            ts[h] += adv;
            while (ts[h] >= p.S) {
              ts[h] -= p.S;
              ++tr[h];
            }
          }
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int kk = kb * BK + ((lane >> 3) + 4 * h) * 4;
            const int rs = kk / p.C;
            tc[h] = kk - rs * p.C;
            tr[h] = rs / p.S;
            ts[h] = rs - tr[h] * p.S;
          }
        }
        cur = kb;
        const int WC = p.W * p.C;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = (lane >> 3) + 4 * h;
          const bool kok = tr[h] < p.R * p.T;  // taps past R*S are the K padding of the last k-block
#pragma unroll
          for (int i = 0; i < RPT; ++i) {
            const int hi = hi0[i] + tr[h], wi = wi0[i] + ts[h];
            const bool ok = kok && valid[i] && (unsigned)hi < (unsigned)p.H && (unsigned)wi < (unsigned)p.W;
            const float* src = ok ? rowp[i] + (hi * WC + wi * p.C + tc[h]) : p.a;
            const int row = warp * (ROWS / 4) + i * 8 + (lane & 7);
            ptx::cp_async16(sbase + kmaj_off<ROWS>(row, j), src, ok ? 16 : 0);
          }
        }
        return;
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int j = (lane >> 3) + 4 * h;
      int kk = kb * BK + j * 4;
      bool kok = kk < p.Kg;
      if constexpr (IS_A && MODE == CONV_FWD) {
        int rs = kok ? kk / p.C : 0;
        int c = kk - rs * p.C;
        int r = rs / p.S;
        int s = rs - r * p.S;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          int hi = hi0[i] + r, wi = wi0[i] + s;
          bool ok = kok && valid[i] && (unsigned)hi < (unsigned)p.H && (unsigned)wi < (unsigned)p.W;
          const float* src = ok ? rowp[i] + ((size_t)hi * p.W + wi) * p.C + c : p.a;
          int row = warp * (ROWS / 4) + i * 8 + (lane & 7);
          ptx::cp_async16(sbase + kmaj_off<ROWS>(row, j), src, ok ? 16 : 0);
        }
      } else if constexpr (IS_A && MODE == CONV_DGRAD) {
        // k = (r, s, cout): dx[n,h,w,:] += dy[n,(h+pad-r)/st,(w+pad-s)/st,cout] * W[cout,r,s,:]
        int rs = kok ? kk / p.K : 0;
        int co = kk - rs * p.K;
        int r = rs / p.S;
        int s = rs - r * p.S;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          int th = hi0[i] - r, tw = wi0[i] - s;
          int ho = th / p.stride, wo = tw / p.stride;
          bool ok = kok && valid[i] && th >= 0 && tw >= 0 && ho * p.stride == th && wo * p.stride == tw &&
                    ho < p.Ho && wo < p.Wo;
          const float* src = ok ? rowp[i] + ((size_t)ho * p.Wo + wo) * p.K + co : p.a;
          int row = warp * (ROWS / 4) + i * 8 + (lane & 7);
          ptx::cp_async16(sbase + kmaj_off<ROWS>(row, j), src, ok ? 16 : 0);
        }
      } else {
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          bool ok = kok && valid[i];
          const float* src = ok ? rowp[i] + kk : p.b;
          int row = warp * (ROWS / 4) + i * 8 + (lane & 7);
          ptx::cp_async16(sbase + kmaj_off<ROWS>(row, j), src, ok ? 16 : 0);
        }
      }
    }
  }
};

// ---- wgrad operands. Both are contiguous along M/N and strided along K (= pixels) in NHWC:
// A = dy^T [Cout][pixels], B = im2col(x)^T [R*S*C][pixels]. Producers cp.async each 16-B
// chunk (4 channels of one pixel) to the K-major position of the 4x4 (channel x pixel) block
// it belongs to -- the block's 64 B hold its four pixel-chunks untransposed -- and the
// transform warps transpose every block in place (plus the 3xTF32 residuals) before the
// MMA reads the stage. Warp pw (0..3) covers chunk blocks b = 8 pw .. 8 pw + 7 per tile:
// g = 8 (b & 3) + (l & 7) (channel group), k = 4 (b >> 2) + (l >> 3) (pixel) -- each
// instruction writes 4 whole core matrices (conflict-free) and reads 4 x 128 B of global.
template <bool IS_A>
struct WLoader {
  int lane, pw;
  const float* base[4];   // B: image-independent part of the address of the 4 owned groups
  int gr[4], gs[4], gc[4];
  bool gok[4];
  int mn0;

  __device__ void init(const GemmParams& p, int mn_start, int ptid) {
    pw = ptid >> 5;
    lane = ptid & 31;
    mn0 = mn_start;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int g = 8 * q + (lane & 7);
      int mn = mn_start + 4 * g;
      gok[q] = mn < (IS_A ? p.M : p.Ng);
      if (!IS_A) {
        int v = gok[q] ? mn : 0;
        int rs = v / p.C;
        gc[q] = v - rs * p.C;
        gr[q] = rs / p.S;
        gs[q] = rs - gr[q] * p.S;
      }
    }
  }

  __device__ void load(const GemmParams& p, uint32_t sbase, int kb) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {                 // the two pixels this thread touches
      int k = 4 * (2 * pw + h) + (lane >> 3);
      int pix = kb * BK + k;
      bool kok = pix < p.Kg;
      int n = 0, hb = 0, wb = 0;
      if (!IS_A && kok) {
        int wo = pix % p.Wo;
        int t = pix / p.Wo;
        int ho = t % p.Ho;
        n = t / p.Ho;
        hb = ho * p.stride - p.pad;
        wb = wo * p.stride - p.pad;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int g = 8 * q + (lane & 7);
        uint32_t dst = sbase + kmaj_off<128>(4 * g + (k & 3), k >> 2);
        const float* src;
        bool ok;
        if (IS_A) {
          ok = kok && gok[q];
          src = ok ? p.a + (size_t)pix * p.K + mn0 + 4 * g : p.a;
        } else {
          int hi = hb + gr[q], wi = wb + gs[q];
          ok = kok && gok[q] && (unsigned)hi < (unsigned)p.H && (unsigned)wi < (unsigned)p.W;
          src = ok ? p.b + (((size_t)n * p.H + hi) * p.W + wi) * p.C + gc[q] : p.b;
        }
        ptx::cp_async16(dst, src, ok ? 16 : 0);
      }
    }
  }
};

__device__ __forceinline__ float4 sel4v(const float4* u, int i) {  // u[i] without local memory
  float4 a = (i & 1) ? u[1] : u[0];
  float4 b = (i & 1) ? u[3] : u[2];
  return (i & 2) ? b : a;
}
__device__ __forceinline__ float comp(const float4& v, int c) {
  float a = (c & 1) ? v.y : v.x;
  float b = (c & 1) ? v.w : v.z;
  return (c & 2) ? b : a;
}

// In-place transpose of one 4x4 block (64 B at blk): chunk e holds pixel e's 4 channels on
// entry and channel e's 4 pixels on exit. Accesses are rotated by `rot` (bank-conflict free
// across an 8-lane phase). With X3 the residuals go to blk + delta.
template <bool X3>
__device__ __forceinline__ void transpose_block(uint32_t blk, int rot, uint32_t delta) {
  float4 u[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    int ce = (e + rot) & 3;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(u[e].x), "=f"(u[e].y), "=f"(u[e].z), "=f"(u[e].w)
                 : "r"(blk + ce * 16));
  }
  // u[e] = chunk (e + rot) & 3  ->  chunk q = u[(q - rot) & 3]
  float4 ch[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) ch[q] = sel4v(u, (q - rot) & 3);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    int c = (e + rot) & 3;    // output row (channel) c
    float x0 = comp(ch[0], c), x1 = comp(ch[1], c), x2 = comp(ch[2], c), x3 = comp(ch[3], c);
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(blk + c * 16), "f"(x0), "f"(x1), "f"(x2),
                 "f"(x3)
                 : "memory");
    if (X3)
      asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(blk + delta + c * 16), "f"(tf32_resid(x0)),
                   "f"(tf32_resid(x1)), "f"(tf32_resid(x2)), "f"(tf32_resid(x3))
                   : "memory");
  }
}

// In-place transpose of one TMA box of 32 pixels x 32 channels (4 KB, SWIZZLE_128B: 16-B chunk j
// of 128-B row r sits at chunk j ^ (r & 7)) into the K-major SWIZZLE_128B operand layout (row =
// channel, k = pixel). Lane l holds pixel l's row in registers, then writes column l of every
// channel row: each store instruction covers one 128-B row, conflict free. X3: residuals -> +delta.
// XF: the block holds 32 channels of the activation; lane l's pixel is replaced by
// relu(scale * v + shift) (scale / shift of channel c held by lane c), or 0 if !valid (padding).
template <bool X3, bool XF = false>
__device__ __forceinline__ void transpose32(uint32_t blk, int lane, uint32_t delta, bool valid = true,
                                            float scl = 0.f, float shl = 0.f) {
  float v[32];
#pragma unroll
  for (int j = 0; j < 8; ++j)
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v[4 * j]), "=f"(v[4 * j + 1]), "=f"(v[4 * j + 2]), "=f"(v[4 * j + 3])
                 : "r"(blk + lane * 128 + ((j ^ (lane & 7)) << 4)));
  if constexpr (XF) {
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const float sc = __shfl_sync(0xffffffffu, scl, c), sh = __shfl_sync(0xffffffffu, shl, c);
      v[c] = valid ? bnrelu1(v[c], sc, sh) : 0.f;
    }
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    const uint32_t a = blk + c * 128 + ((((lane >> 2) ^ (c & 7))) << 4) + (lane & 3) * 4;
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v[c]) : "memory");
    if (X3) asm volatile("st.shared.f32 [%0], %1;" ::"r"(a + delta), "f"(tf32_resid(v[c])) : "memory");
  }
}

// ------------------------------------------------------------------------------- kernel
// Butterfly transpose-reduce: on return lane l holds sum over the 32 lanes of v[l].
__device__ __forceinline__ float warp_transpose_sum32(float* v, int lane) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    bool upper = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < off; ++i) {
      float send = upper ? v[i] : v[i + off];
      float keep = upper ? v[i + off] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0];
}

// Persistent, warp-specialised kernel: each CTA walks tiles t = blockIdx.x + i*gridDim.x
// (M-tiles fastest, so concurrently running CTAs share the B tile in L2). Two TMEM
// accumulators let the epilogue of tile i overlap the mainloop of tile i+1.
//   warps 0-3 : epilogue (TMEM lane quadrant = warp), warps 4-7 : producers,
//   warp 8    : TMEM allocator + single-thread MMA issuer.
constexpr int NUM_THREADS_P = 288;      // 4 epilogue + 4 producer + 1 MMA warps
constexpr int NUM_THREADS_X3 = 416;     // + 4 residual ("split") warps for 3xTF32
// the auxiliary warps 9-12 compute 3xTF32 residuals and / or transpose wgrad operands
__host__ __device__ constexpr bool igemm_aux(int mode, bool x3, bool xf = false) {
  return x3 || xf || mode == CONV_WGRAD;
}
// E2: a second epilogue warp group (warps 4-7, the TMA producer moves to warp 13)
__host__ __device__ constexpr int igemm_threads(int mode, bool x3, bool xf = false, int naux = 4, bool e2 = false) {
  return (igemm_aux(mode, x3, xf) ? NUM_THREADS_P + 32 * naux : NUM_THREADS_P) + (e2 ? 32 : 0);
}


struct TileMap {
  int mt, nt, zt, kb_total, kbps;  // mt = M-tiles (TMA: tiles_n * tiles_h * tiles_w)
  bool nfast;                      // N-tiles fastest: co-running CTAs share the A (activation) tile
  __device__ void decode(int t, int& m0, int& n0, int& kb0, int& nkb, int bn) const {
    int m, n, z;
    if (nfast) {
      n = t % nt;
      const int r = t / nt;
      m = r % mt;
      z = r / mt;
    } else {
      m = t % mt;
      const int r = t / mt;
      n = r % nt;
      z = r / nt;
    }
    m0 = m * BM;
    n0 = n * bn;
    kb0 = z * kbps;
    nkb = max(0, min(kb_total, kb0 + kbps) - kb0);
  }
};

template <int MODE, int BN, int STAGES, bool X3 = false, bool TMA = false, bool XF = false, bool AT = false,
          int NSTG = 1, int NAUX = 4, bool MNW = false, bool E2 = false, bool SP = false, bool W2 = false,
          bool SPW = false>
__global__ void __launch_bounds__(igemm_threads(MODE, X3, XF, NAUX, E2), 1)
    igemm_kernel(const GemmParams p, const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                 const __grid_constant__ CUtensorMap tma_c, const __grid_constant__ CUtensorMap tma_d) {
  static_assert(!TMA || MODE != GEMM_TEST, "TMA path: conv fwd / dgrad / wgrad");
  // TMA tiles whose M rows are a box of output pixels (FWD / DGRAD); TMA wgrad boxes pixels along K
  constexpr bool PIXM = TMA && MODE != CONV_WGRAD;
  static_assert(!XF || (TMA && (MODE == CONV_FWD || MODE == CONV_WGRAD)), "XF: TMA-fed fwd / wgrad only");
  // NAUX > 4 auxiliary warps: only the TMA wgrad block loop distributes over them
  static_assert(NAUX == 4 || (MODE == CONV_WGRAD && TMA && !AT && !XF), "NAUX: TMA wgrad only");
  // MNW: TMA wgrad with both operands MN-major in shared memory -- the boxes land as [pixel][32
  // channels] rows in the SWIZZLE_128B_ATOM_32B layout, the only MN-major layout tcgen05 accepts
  // for tf32 (layout type SWIZZLE_128B_BASE32B), so no transposes:
  // the auxiliary warps only write the 3xTF32 residuals
  static_assert(!MNW || (MODE == CONV_WGRAD && TMA && !XF && NAUX == 4), "MNW: plain TMA wgrad");
  // AT: 3xTF32 with the A operand in TMEM -- the auxiliary warps move each stage's A tile (hi =
  // trunc_tf32(a), lo = a - hi) from shared memory into TMEM, so the three MMAs of a k-step read
  // only B / Bs from shared memory (A is re-read by every MMA, the dominant smem traffic at BN = 64)
  static_assert(!AT || (X3 && TMA && MODE != GEMM_TEST && (!XF || MODE == CONV_FWD)),
                "AT: 3xTF32 TMA fwd / dgrad / wgrad (with BN-ReLU on load: fwd only)");
  // W2 (BN = 64, A in TMEM): the weight tile and its residual, adjacent in shared memory, form one
  // 128-row B operand, so a k-step is two N = 128 MMAs -- lo * [B; Bs] and hi * [B; Bs] -- instead
  // of three N = 64 ones (an N = 64 tcgen05.mma runs at ~2/3 of the per-flop rate of N = 128, and
  // each k-block's barrier wait in the issuing thread stalls the narrow ones longer:
  // tools/mmaprobe). The accumulator is [A*B | A*Bs] (2 * BN columns); the epilogue adds the halves.
  // (MN-major wgrad, MNW: the B blocks and their residual blocks are 4 KB apart in one MN-major
  // run, so [B; Bs] is one 128-row operand with the same LBO)
  static_assert(!W2 || (AT && BN == 64 && (MODE != CONV_WGRAD || MNW)), "W2: AT fwd / dgrad / MN-major wgrad at BN = 64");
  constexpr uint32_t ACC_COLS = W2 ? 2u * BN : (uint32_t)BN;  // columns of one accumulator
  // W2 over a TMA-landed K-major A tile (not SP's gathered rows, not XF's transformed ones): the hi
  // products read A straight from the stage -- the tensor core truncates fp32 operands to TF32
  // (Reading 27), which is exactly hi -- so the auxiliary warps move only lo into TMEM (half the
  // tcgen05.st traffic per k-block, the same operand values: bit-identical products)
#ifdef POOCH_W2_HI_TMEM
  constexpr bool W2_HI_SMEM = false;
#else
  constexpr bool W2_HI_SMEM = W2 && !SP && !XF && !MNW && MODE != CONV_WGRAD;
#endif
  static_assert(!AT || 2 * ACC_COLS + 64 * STAGES <= 512, "AT: accumulators + A stages exceed TMEM");
  // E2: two epilogue warp groups drain each accumulator, one per half of its columns (the
  // 1x1 expand convs are epilogue-bound: TMEM -> smem staging -> BN partial sums -> TMA store);
  // warps 4-7 (idle besides the one TMA-issuing thread) become group 1, and the TMA producer
  // moves to warp 13 -- the TMEM lane quadrant a warp may read is warp % 4, so 4-7 cover all four
  static_assert(!E2 || (PIXM && X3 && NAUX == 4), "E2: 3xTF32 TMA fwd / dgrad");
  constexpr int NEG = E2 ? 2 : 1;
  // SP (stem patch, 4-channel input): per tile the producer loads the input patch under the
  // tile's output box once ((tw - 1) * stride + S wide, (th - 1) * stride + R high, 16 B per pixel,
  // zero-filled padding) and per k-block only the weight tile; the auxiliary warps gather each
  // A row's 8 taps x 4 channels from the patch straight into TMEM (hi / lo) -- instead of 16
  // narrow TMA boxes per k-block (stem4 = 1) or 16-B cp.async gathers
  static_assert(!SP || (AT && MODE == CONV_FWD && !XF), "SP: AT fwd");
  // SPW (stem patch wgrad, 4-channel input): the transposed MN-major wgrad (A = im2col(x)^T in
  // TMEM, B = dy^T MN-major) whose A operand is gathered from one input patch per k-block -- the
  // TMA box {4 channels, (tw - 1) * stride + S, (th - 1) * stride + R, 1 image} under the k-block's
  // tw x th pixel box, 16 B per pixel, zero-filled padding -- instead of per-tap 32-channel boxes
  // (a 4-channel input has no 32-channel chunks); lane = row (r, s, c) of A reads pixel k's tap at
  // patch ((k / tw) * stride + r, (k % tw) * stride + s), channel c
  static_assert(!SPW || (MODE == CONV_WGRAD && TMA && AT && MNW && X3), "SPW: 3xTF32 MN-major wgrad, A in TMEM");
  constexpr int PW = E2 ? 13 : 4;  // first producer warp
  constexpr uint32_t TMEM_COLS = AT ? 512u : 2u * BN;
  constexpr uint32_t A_TCOL = 2u * ACC_COLS;  // AT: stage s's hi tile at column A_TCOL + 64 s, lo at + 32
  constexpr bool AUX = igemm_aux(MODE, X3, XF);
  using SM = GemmSmem<BN, STAGES, X3, AT, NSTG, NEG, SP>;
  static_assert(!W2 || SP || SM::BS_OFF == SM::B_BYTES, "W2: Bs directly after B");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (ptx::smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint64_t* rawfull = tempty + 2;     // [STAGES] 3xTF32: raw operands landed (cp.async arrivals)
  uint64_t* pfull = rawfull + STAGES;  // [NPB] SP: input patch landed
  uint64_t* pempty = pfull + SM::NPB;  // [NPB] SP: the auxiliary warps are done with the patch
  uint64_t* bfull = pempty + SM::NPB;  // SP: the resident weight tiles landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 2);
  float* red = reinterpret_cast<float*>(smem + SM::RED_OFF);  // [4][BN] x2

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  TileMap tm;
  tm.mt = PIXM ? p.tiles_n * p.tiles_h * p.tiles_w : (p.M + BM - 1) / BM;
  tm.nt = (p.Ng + BN - 1) / BN;
  tm.kb_total = (TMA && MODE == CONV_WGRAD) ? p.tiles_n * p.tiles_h * p.tiles_w : (p.Kg + BK - 1) / BK;
  tm.kbps = p.kb_per_split > 0 ? p.kb_per_split : max(tm.kb_total, 1);
  tm.zt = p.kb_per_split > 0 ? (tm.kb_total + tm.kbps - 1) / tm.kbps : 1;
  // FWD / DGRAD: B is the (transposed) weight matrix -- at most a few MB, always L2-resident --
  // while A is the activation stream; with N-tiles fastest the CTAs working on one M-tile run
  // together and read its A rows from DRAM once instead of once per N-tile
  tm.nfast = (MODE == CONV_FWD || MODE == CONV_DGRAD) && tm.nt > 1;
  const int ntiles = tm.mt * tm.nt * tm.zt;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      // full: 128 producer (cp.async) or auxiliary-warp arrivals; 1 expect_tx arrival (TMA, no aux)
      ptx::mbar_init(&full[s], (TMA && !AUX) ? 1 : 32 * NAUX);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 128 * NEG);
    }
    for (int s = 0; s < STAGES; ++s) ptx::mbar_init(&rawfull[s], TMA ? 1 : 128);
    for (int a = 0; a < SM::NPB; ++a) {
      ptx::mbar_init(&pfull[a], 1);
      ptx::mbar_init(&pempty[a], 128);
    }
    ptx::mbar_init(bfull, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 8) ptx::tmem_alloc(tmem_slot, TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = ptx::smem_u32(smem);

  if (E2 ? warp == PW : (warp >= 4 && warp < 8)) {
    // ------------------------------------------------------------------ producers
    const int ptid = tid - 32 * PW;
    if constexpr (MODE == CONV_WGRAD && TMA) {
      // one elected thread: per k-block (a box of 32 output pixels) one 4-D TMA box per 32 rows
      // of each operand -- dy: 32 output channels x the pixel box; x: the 32 input channels of
      // one (r, s) tap over the box's input pixels (traversal stride = conv stride, padding
      // zero-filled). Rows past M / Ng are skipped: they only feed accumulator rows / columns
      // the epilogue never stores.
      if (ptid == 0) {
        ptx::tma_prefetch_desc(&tma_a);
        ptx::tma_prefetch_desc(&tma_b);
        if (p.c_split) ptx::tma_prefetch_desc(&tma_c);
        int it = 0;
        // per tile, the (at most (BM + BN) / 32) boxes' maps and tap offsets are fixed: decode them
        // once; per k-block only the pixel box moves (walked incrementally, no divisions), so the
        // single issuing thread keeps up with the MMAs of narrow (BN = 64) tiles
        constexpr int NBOX = (BM + BN) / 32;
        const CUtensorMap* bmap[NBOX];
        uint32_t bdst[NBOX];
        int bdx[NBOX], bdy[NBOX], bdz[NBOX], bch[NBOX];
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
          int m0, n0, kb0, nkb;
          tm.decode(t, m0, n0, kb0, nkb, BN);
          uint32_t bytes = 0;
          int nbox = 0;
          // one box = cb consecutive 32-channel chunks of the same tap over the pixel box; the
          // 5-D map puts the chunk index outermost, so the box lands as cb consecutive 4-KB blocks
          auto add_box = [&](uint32_t dst_off, const CUtensorMap* map, bool is_x, int row, int cb) {
            bdst[nbox] = dst_off;
            bytes += 4096u * cb;
            if (is_x) {
              // row = ((t * R + r) * S + s) * C + c; channels past c_split come from the second source
              const int rs = row / p.C;
              int c = row - rs * p.C;
              const int t3 = rs / (p.R * p.S), r2 = rs - t3 * p.R * p.S;
              const int r = r2 / p.S, sx = r2 - r * p.S;
              if (p.c_split && c >= p.c_split) {
                map = &tma_c;
                c -= p.c_split;
              }
              bmap[nbox] = map;
              bdx[nbox] = sx - p.pad;
              bdy[nbox] = r - p.pad;
              bdz[nbox] = t3 - p.pad3;
              bch[nbox] = c >> 5;
            } else {
              bmap[nbox] = map;
              bdx[nbox] = bdy[nbox] = bdz[nbox] = 0x40000000;   // marks a dy box (no stride / offset)
              bch[nbox] = row >> 5;
            }
            ++nbox;
          };
          if constexpr (SPW) {
            bytes += (uint32_t)p.patch_w * ((p.th - 1) * p.stride + p.R) * 16u;
          } else {
            for (int q = 0; q < BM / 32; q += p.wg_cba)
              if (m0 + 32 * q < p.M) add_box(q * 4096, &tma_a, p.wg_a_is_x != 0, m0 + 32 * q, p.wg_cba);
          }
          for (int q = 0; q < BN / 32; q += p.wg_cbb)
            if (n0 + 32 * q < p.Ng) add_box(SM::A_BYTES + q * 4096, &tma_b, p.wg_a_is_x == 0, n0 + 32 * q, p.wg_cbb);
          int bw = kb0 % p.tiles_w, bh = (kb0 / p.tiles_w) % p.tiles_h, bn = kb0 / (p.tiles_w * p.tiles_h);
          for (int kb = 0; kb < nkb; ++kb, ++it) {
            int s = it % STAGES;
            if (it >= STAGES) ptx::mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
            uint32_t st = sbase + s * SM::STAGE_BYTES;
            const int ow = bw * p.tw, oh = bh * p.th, on = bn * p.tn;
            ptx::mbar_arrive_expect_tx(&rawfull[s], bytes);
            if constexpr (SPW)  // the input patch under the pixel box (A region of the stage)
              ptx::tma_load_4d(st, &tma_a, &rawfull[s], 0, ow * p.stride - p.pad, oh * p.stride - p.pad, on);
            for (int i = 0; i < nbox; ++i) {
              if (bdx[i] == 0x40000000)
                ptx::tma_load_5d(st + bdst[i], bmap[i], &rawfull[s], 0, ow, oh, on, bch[i]);
              else
                ptx::tma_load_5d(st + bdst[i], bmap[i], &rawfull[s], 0, ow * p.stride + bdx[i], oh * p.stride + bdy[i],
                                 on * p.st3 + bdz[i], bch[i]);
            }
            if (++bw == p.tiles_w) {
              bw = 0;
              if (++bh == p.tiles_h) {
                bh = 0;
                ++bn;
              }
            }
          }
        }
      }
    } else if constexpr (MODE == CONV_WGRAD) {
      static_assert(BN == 128, "wgrad uses 128 x 128 tiles");
      WLoader<true> la;
      WLoader<false> lb;
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int m0, n0, kb0, nkb;
        tm.decode(t, m0, n0, kb0, nkb, BN);
        la.init(p, m0, ptid);
        lb.init(p, n0, ptid);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          int s = it % STAGES;
          if (it >= STAGES) ptx::mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
          uint32_t st = sbase + s * SM::STAGE_BYTES;
          const int k = kb0 + kb;
          la.load(p, st, k);
          lb.load(p, st + SM::A_BYTES, k);
          ptx::cp_async_arrive_noinc(&rawfull[s]);
        }
      }
      ptx::cp_async_wait<0>();
    } else if constexpr (TMA) {
      // one elected thread drives the tensor-memory accelerator: per k-block (r, s, 32-channel
      // chunk) a 4-D box of input (FWD: x, DGRAD: dy) pixels -- out-of-range rows / columns of the
      // padding are zero-filled by the TMA -- and a 2-D box of the (transposed) weight.
      if (ptid == 0) {
        ptx::tma_prefetch_desc(&tma_a);
        ptx::tma_prefetch_desc(&tma_b);
        if (p.c_split) ptx::tma_prefetch_desc(&tma_c);
        const uint32_t a_bytes = 32u * p.tw * p.th * p.tn * 4u;
        const uint32_t bytes = a_bytes + (uint32_t)BN * 32u * 4u;
        const int cred = MODE == CONV_FWD ? p.C : p.K;  // reduced channels
        int it = 0, jt = 0, jn = 0;
        if constexpr (SP) {  // the whole weight matrix, once: k-block kb's 64 x 32 tile at kb * B_BYTES
          ptx::mbar_arrive_expect_tx(bfull, (uint32_t)tm.kb_total * SM::B_BYTES);
          for (int kb = 0; kb < tm.kb_total; ++kb)
            ptx::tma_load_2d(sbase + kb * SM::B_BYTES * (W2 ? 2 : 1), &tma_b, bfull, kb * 32, 0);
        }
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++jt) {
          int m0, n0, kb0, nkb;
          tm.decode(t, m0, n0, kb0, nkb, BN);
          const int mt_i = m0 / BM;
          const int tw_i = mt_i % p.tiles_w;
          const int th_i = (mt_i / p.tiles_w) % p.tiles_h;
          const int tn_i = mt_i / (p.tiles_w * p.tiles_h);
          if constexpr (SP) {
            // input patches (box {4, patch_w, patch_h, 1} of the tensor map, zero-filled outside
            // the image) run NPB - 1 tiles ahead of the k-block relay
            while (jn <= jt + SM::NPB - 1) {
              const int tq = blockIdx.x + jn * gridDim.x;
              if (tq < ntiles) {
                int qm0, qn0, qkb0, qnkb;
                tm.decode(tq, qm0, qn0, qkb0, qnkb, BN);
                const int qi = qm0 / BM;
                const int qw = qi % p.tiles_w, qh = (qi / p.tiles_w) % p.tiles_h, qn = qi / (p.tiles_w * p.tiles_h);
                const int pb = jn % SM::NPB;
                if (jn >= SM::NPB) ptx::mbar_wait(&pempty[pb], ((jn / SM::NPB) - 1) & 1);
                ptx::mbar_arrive_expect_tx(&pfull[pb], (uint32_t)p.patch_w * ((p.th - 1) * p.stride + p.R) * 16u);
                ptx::tma_load_4d(sbase + SM::PATCH_OFF + pb * SM::PATCH_BYTES, &tma_a, &pfull[pb], 0,
                                 qw * p.tw * p.stride - p.pad, qh * p.th * p.stride - p.pad, qn);
              }
              ++jn;
            }
            (void)tw_i; (void)th_i; (void)tn_i;
#ifdef POOCH_SP_RELAY
            // (experiment) per k-block a relay: TMEM stage s is free again once its MMAs are done
            for (int kb = 0; kb < nkb; ++kb, ++it) {
              const int s = it % STAGES;
              if (it >= STAGES) ptx::mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
              ptx::mbar_arrive(&rawfull[s]);
            }
#endif
            continue;
          }
          // the k-block walks (tap, 32-channel chunk) with the chunk fastest: decode k = kb0 once per
          // tile, then advance incrementally (no per-k-block divisions in the single issuing thread,
          // which otherwise paces the narrow BN = 64 tiles)
          int cc = kb0 % p.cchunks, tap0 = kb0 / p.cchunks;
          int wt3, wr, ws;   // FWD: (t3, r, s) of the tap; DGRAD: the class-tap indices (tt, tr, ts)
          if (MODE == CONV_FWD) {
            wt3 = tap0 / (p.R * p.S);
            const int r2 = tap0 - wt3 * p.R * p.S;
            wr = r2 / p.S;
            ws = r2 - wr * p.S;
          } else {
            wt3 = tap0 / (p.dg_nr * p.dg_ns);
            const int t2 = tap0 - wt3 * p.dg_nr * p.dg_ns;
            wr = t2 / p.dg_ns;
            ws = t2 - wr * p.dg_ns;
          }
          // FWD: cw = cw0 + s; DGRAD: cw = cw0 - ts (the class selects taps whose offsets divide
          // exactly by the stride)
          const int cw0 = MODE == CONV_FWD ? tw_i * p.tw * p.stride - p.pad
                                           : tw_i * p.tw + (p.dg_b + p.pad - p.dg_s0) / p.stride;
          const int ch0 = MODE == CONV_FWD ? th_i * p.th * p.stride - p.pad
                                           : th_i * p.th + (p.dg_a + p.pad - p.dg_r0) / p.stride;
          const int c30 = MODE == CONV_FWD ? tn_i * p.tn * p.st3 - p.pad3
                                           : tn_i * p.tn + (p.dg_c + p.pad3 - p.dg_t0) / p.st3;
          for (int kb = 0; kb < nkb; ++kb, ++it) {
            int s = it % STAGES;
            if (it >= STAGES) ptx::mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
            uint32_t st = sbase + s * SM::STAGE_BYTES;
            uint64_t* bar = AUX ? &rawfull[s] : &full[s];
            const int k = kb0 + kb;
            int cw, chh, c3, rs;
            if (MODE == CONV_FWD) {  // tap = (t * R + r) * S + s over the [K][T][R][S][C] weights
              rs = (wt3 * p.R + wr) * p.S + ws;
              cw = cw0 + ws;
              chh = ch0 + wr;
              c3 = c30 + wt3;
            } else {
              const int r = p.dg_r0 + p.stride * wr, sx = p.dg_s0 + p.stride * ws, t3 = p.dg_t0 + p.st3 * wt3;
              rs = (t3 * p.R + r) * p.S + sx;
              cw = cw0 - ws;
              chh = ch0 - wr;
              c3 = c30 - wt3;
            }
            const int cck = cc;
            if (++cc == p.cchunks) {   // next tap
              cc = 0;
              const int ns = MODE == CONV_FWD ? p.S : p.dg_ns, nr = MODE == CONV_FWD ? p.R : p.dg_nr;
              if (++ws == ns) {
                ws = 0;
                if (++wr == nr) {
                  wr = 0;
                  ++wt3;
                }
              }
            }
            if (MODE == CONV_FWD && p.stem4) {
              // 8 taps of 4 channels: tap j's A box (16 B per output pixel) lands at j * BM * 16 and
              // its B box at j * BN * 16 -- SWIZZLE_NONE core matrices, K-adjacent ones BM*16 / BN*16
              // apart. Taps past R*S load fully out-of-bounds boxes: zeros, bytes still counted.
              const int ntap = p.R * p.S;
              ptx::mbar_arrive_expect_tx(bar, 8u * (16u * p.tw * p.th * p.tn + 16u * BN));
#pragma unroll 1
              for (int j = 0; j < 8; ++j) {
                const int tp = 8 * k + j;
                const bool live = tp < ntap;
                const int r = live ? tp / p.S : 0, sx = live ? tp - (tp / p.S) * p.S : 0;
                const int aw = live ? tw_i * p.tw * p.stride - p.pad + sx : -(1 << 20);
                const int ah = th_i * p.th * p.stride - p.pad + r;
                ptx::tma_load_4d(st + j * (BM * 16), &tma_a, bar, 0, aw, ah, tn_i * p.tn);
                ptx::tma_load_2d(st + SM::A_BYTES + j * (BN * 16), &tma_b, bar, live ? 4 * tp : (1 << 20), n0);
              }
              continue;
            }
            ptx::mbar_arrive_expect_tx(bar, bytes);
            if (MODE == CONV_FWD && p.c_split && cck * 32 >= p.c_split)
              ptx::tma_load_4d(st, &tma_c, bar, cck * 32 - p.c_split, cw, chh, c3);
            else
              ptx::tma_load_4d(st, &tma_a, bar, cck * 32, cw, chh, c3);
            ptx::tma_load_2d(st + SM::A_BYTES, &tma_b, bar, rs * cred + cck * 32, n0);
          }
        }
      }
    } else {
      KLoader<MODE, BM, true> la;
      KLoader<MODE, BN, false> lb;
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int m0, n0, kb0, nkb;
        tm.decode(t, m0, n0, kb0, nkb, BN);
        la.init(p, m0, ptid);
        lb.init(p, n0, ptid);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          int s = it % STAGES;
          if (it >= STAGES) ptx::mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
          uint32_t st = sbase + s * SM::STAGE_BYTES;
          la.load(p, st, kb0 + kb);
          lb.load(p, st + SM::A_BYTES, kb0 + kb);
          // the barrier completes when this thread's copies land: no wait in the producer
          ptx::cp_async_arrive_noinc(X3 ? &rawfull[s] : &full[s]);
        }
      }
      ptx::cp_async_wait<0>();
    }
  } else if (AUX && warp >= 9 && warp < 9 + NAUX) {  // (E2: warp 13 = 9 + NAUX is the producer)
    // ------------------------------------------------------------------ auxiliary warps
    // Per stage: wait for the raw operands, (wgrad) transpose every 4x4 block in place,
    // (3xTF32) write x - tf32(x) of every chunk, publish to the async proxy, arrive full[].
    const int stid = tid - 9 * 32;
    int it = 0;
    // XF forward: this thread's A chunks are rows (stid >> 3) + 16 i, physical 16-B chunk stid & 7
    // (logical chunk pj ^ (row & 7), the same for all eight rows); per tile the rows' top-left
    // input coordinates (hb, wb) and whether the row is an output pixel at all
    int hb[8], wb[8];
    unsigned rowv = 0;
    int jt = 0;
    if constexpr (SP) {  // residuals of the resident weight tiles, once
      ptx::mbar_wait(bfull, 0);
      // W2: B of k-block kb at kb * 2 * B_BYTES and its residual right after it; else Bs at + BS_OFF
      const int nch = tm.kb_total * SM::B_BYTES / 16, cpb = SM::B_BYTES / 16;
      for (int c = stid; c < nch; c += 128) {
        const uint32_t src = W2 ? sbase + (c / cpb) * 2 * SM::B_BYTES + (c % cpb) * 16 : sbase + c * 16;
        split_chunk(src, W2 ? src + SM::B_BYTES : src + SM::BS_OFF);
      }
    }
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++jt) {
      int m0, n0, kb0, nkb;
      tm.decode(t, m0, n0, kb0, nkb, BN);
      // SP: this thread's A row = output pixel (ph, pw) of the tile box; its taps read patch pixels
      // (ph * stride + r, pw * stride + s); (tr, ts) walks the taps of the k-block incrementally
      const int sp_row = 32 * (warp & 3) + lane;
      const bool sp_ok = sp_row < p.tw * p.th;
      const uint32_t sp_base = sbase + SM::PATCH_OFF + (jt % SM::NPB) * SM::PATCH_BYTES +
                               (uint32_t)(((sp_row / p.tw) * p.stride * p.patch_w + (sp_row % p.tw) * p.stride) * 16);
      int tr = 0, ts = 0, tap = 0;
      if constexpr (SP) ptx::mbar_wait(&pfull[jt % SM::NPB], (jt / SM::NPB) & 1);
      if constexpr (XF && MODE == CONV_FWD) {
        const int mt_i = m0 / BM;
        const int tw_i = mt_i % p.tiles_w, th_i = (mt_i / p.tiles_w) % p.tiles_h, tn_i = mt_i / (p.tiles_w * p.tiles_h);
        const int per = p.tw * p.th;
        rowv = 0;
#pragma unroll
        for (int i = 0; i < (AT ? 1 : 8); ++i) {
          // AT: one row per thread (lane of the warp's TMEM quadrant); else 8 rows of a chunk column
          const int row = AT ? 32 * (warp & 3) + lane : (stid >> 3) + 16 * i;
          const int nn = tn_i * p.tn + row / per, ho = th_i * p.th + (row / p.tw) % p.th, wo = tw_i * p.tw + row % p.tw;
          if (row < per * p.tn && nn < p.n3 && ho < p.hout && wo < p.wout) rowv |= 1u << i;
          hb[i] = ho * p.stride - p.pad;
          wb[i] = wo * p.stride - p.pad;
        }
      }
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        int s = it % STAGES;
        // XF: everything the transform needs that does not depend on the stage's data (scale /
        // shift loads from L2, padding masks) is done before waiting for the stage, so the
        // load latency overlaps the TMA instead of sitting between the TMA and the MMA
        float4 xsc = make_float4(0.f, 0.f, 0.f, 0.f), xsh = xsc;
        unsigned xvalid = 0;
        constexpr int WQ = ((BM + BN) / 32 + NAUX - 1) / NAUX;  // wgrad: 32x32 blocks per auxiliary warp
        float wscl[WQ], wshl[WQ];
        bool wval[WQ], wx[WQ];
#pragma unroll
        for (int q = 0; q < WQ; ++q) {
          wscl[q] = wshl[q] = 0.f;
          wval[q] = wx[q] = false;
        }
        if constexpr (XF && MODE == CONV_FWD) {
          const int k = kb0 + kb;
          const int tap = k / p.cchunks, cc = k - tap * p.cchunks;
          const int r = tap / p.S, sx = tap - r * p.S;
          if constexpr (AT) {  // lane-distributed: lane l holds channel cc*32 + l's scale / shift
            xsc.x = __ldg(p.xf_scale + cc * 32 + lane);
            xsh.x = __ldg(p.xf_shift + cc * 32 + lane);
            const int hi = hb[0] + r, wi = wb[0] + sx;
            if ((rowv & 1u) && (unsigned)hi < (unsigned)p.H && (unsigned)wi < (unsigned)p.W) xvalid = 1u;
          } else {
            const int jl = (stid & 7) ^ ((stid >> 3) & 7);
            xsc = __ldg(reinterpret_cast<const float4*>(p.xf_scale + cc * 32 + 4 * jl));
            xsh = __ldg(reinterpret_cast<const float4*>(p.xf_shift + cc * 32 + 4 * jl));
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int hi = hb[i] + r, wi = wb[i] + sx;
              if (((rowv >> i) & 1u) && (unsigned)hi < (unsigned)p.H && (unsigned)wi < (unsigned)p.W) xvalid |= 1u << i;
            }
          }
        }
        if constexpr (XF && MODE == CONV_WGRAD) {
          const int b = kb0 + kb;
          const int ow = (b % p.tiles_w) * p.tw, oh = ((b / p.tiles_w) % p.tiles_h) * p.th,
                    on = (b / (p.tiles_w * p.tiles_h)) * p.tn;
          const int wo = ow + lane % p.tw, ho = oh + (lane / p.tw) % p.th, nn = on + lane / (p.tw * p.th);
          const bool pix = nn < p.N && ho < p.Ho && wo < p.Wo;
#pragma unroll
          for (int q = 0; q < WQ; ++q) {
            const int bi = warp - 9 + 4 * q;
            const bool in_a = bi < BM / 32;
            if (bi >= (BM + BN) / 32 || in_a != (p.wg_a_is_x != 0)) continue;
            const int row = in_a ? m0 + 32 * bi : n0 + 32 * (bi - BM / 32);
            if (row >= (in_a ? p.M : p.Ng)) continue;  // box not loaded: rows never stored
            wx[q] = true;
            const int rs = row / p.C, ch = row - rs * p.C;
            const int r = rs / p.S, sx = rs - r * p.S;
            const int hi = ho * p.stride - p.pad + r, wi = wo * p.stride - p.pad + sx;
            wval[q] = pix && (unsigned)hi < (unsigned)p.H && (unsigned)wi < (unsigned)p.W;
            wscl[q] = __ldg(p.xf_scale + ch + lane);
            wshl[q] = __ldg(p.xf_shift + ch + lane);
          }
        }
#ifndef POOCH_SP_RELAY
        if constexpr (SP) {  // TMEM stage s is free once the MMAs that read it are done (no relay)
          if (it >= STAGES) ptx::mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
        } else
#endif
        ptx::mbar_wait(&rawfull[s], (it / STAGES) & 1);
        uint32_t st = sbase + s * SM::STAGE_BYTES;
        if constexpr (MNW && AT) {
          // A in TMEM from MN-major blocks: warp w owns A block w & 3 (its TMEM lane quadrant);
          // lane m gathers its 32 K values straight from the block's column m (row k at k * 128,
          // 32-B granule (m / 8) ^ (k & 3): conflict-free across the lanes), splits hi / lo and
          // stores both into this stage's TMEM columns; the B blocks get their residuals in place
          // (+ BS_OFF, same MN-major layout)
#pragma unroll
          for (int q = 0; q < WQ; ++q) {
            const int bi = (warp & 3) + 4 * q;
            if (bi >= (BM + BN) / 32) break;
            const uint32_t blk = st + bi * 4096;
            if (bi < BM / 32) {
              float v[32], lo[32];
              if constexpr (SPW) {
                // row (r, s, c) of im2col(x)^T; pixel k = (k % tw, k / tw) of the box (tw a power of
                // two, tw * th = 32); rows past R*S*4 are zero
                const int row = m0 + 32 * bi + lane;
                const bool ok = row < p.M;
                const int rs = row >> 2, r = rs / p.S, sx = rs - r * p.S;
                const uint32_t lb = st + (uint32_t)(((r * p.patch_w + sx) * 4 + (row & 3)) * 4);
                const int ltw = __ffs(p.tw) - 1;
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                  const uint32_t off = (uint32_t)((((k >> ltw) * p.patch_w + (k & (p.tw - 1))) * p.stride) * 16);
                  if (ok)
                    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[k]) : "r"(lb + off));
                  else
                    v[k] = 0.f;
                }
              } else {
#pragma unroll
              for (int k = 0; k < 32; ++k)
                asm volatile("ld.shared.f32 %0, [%1];"
                             : "=f"(v[k])
                             : "r"(blk + k * 128 + ((((lane >> 3) ^ (k & 3))) << 5) + (lane & 7) * 4));
              }
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const float hi = __uint_as_float(__float_as_uint(v[i]) & 0xFFFFE000u);
                lo[i] = v[i] - hi;
                v[i] = hi;
              }
              const uint32_t ta = tmem + ((uint32_t)(32 * bi) << 16) + A_TCOL + 64u * s;
              ptx::tmem_st32(ta, v);
              ptx::tmem_st32(ta + 32, lo);
            } else {
              const uint32_t bblk = st + SM::A_BYTES + (bi - BM / 32) * 4096;
#pragma unroll
              for (int c = lane; c < 256; c += 32) split_chunk(bblk + c * 16, bblk + SM::BS_OFF + c * 16);
            }
          }
          ptx::tmem_wait_st();
          ptx::tc_fence_before();
        } else if constexpr (MNW) {
          // MN-major operands: the residual of every element at the same offset + SMALL_OFF (the
          // layout is the same for both, so no index arithmetic)
          if constexpr (X3) {
            constexpr int CHUNKS = (BM + BN) * BK / 4;
#pragma unroll 4
            for (int c = stid; c < CHUNKS; c += 128) split_chunk(st + c * 16, st + SM::SMALL_OFF + c * 16);
          }
        } else if constexpr (MODE == CONV_WGRAD && TMA && AT) {
          // A in TMEM: warp w owns A block w & 3 (its TMEM lane quadrant): transpose it in place,
          // read its rows back (lane = row) and store hi / lo into this stage's TMEM columns; the B
          // blocks are transposed with their residuals into [B][Bs] as usual
#pragma unroll
          for (int q = 0; q < WQ; ++q) {
            const int bi = (warp & 3) + 4 * q;
            if (bi >= (BM + BN) / 32) break;
            if (bi < BM / 32) {
              const uint32_t blk = st + bi * 4096;
              transpose32<false>(blk, lane, 0);
              __syncwarp();
              float v[32], lo[32];
#pragma unroll
              for (int j = 0; j < 8; ++j)
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(v[4 * j]), "=f"(v[4 * j + 1]), "=f"(v[4 * j + 2]), "=f"(v[4 * j + 3])
                             : "r"(blk + lane * 128 + ((j ^ (lane & 7)) << 4)));
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const float hi = __uint_as_float(__float_as_uint(v[i]) & 0xFFFFE000u);
                lo[i] = v[i] - hi;
                v[i] = hi;
              }
              const uint32_t ta = tmem + ((uint32_t)(32 * bi) << 16) + A_TCOL + 64u * s;
              ptx::tmem_st32(ta, v);
              ptx::tmem_st32(ta + 32, lo);
            } else {
              transpose32<true>(st + bi * 4096, lane, SM::BS_OFF);
            }
          }
          ptx::tmem_wait_st();
          ptx::tc_fence_before();
        } else if constexpr (MODE == CONV_WGRAD && TMA) {
          // (BM + BN) / 32 TMA boxes, A's then B's, 4 KB each; residuals at the same offsets + SMALL_OFF
#pragma unroll
          for (int q = 0; q < WQ; ++q) {
            const int bi = warp - 9 + NAUX * q;
            if (bi >= (BM + BN) / 32) break;
            if (XF && wx[q])  // an activation block: BN-ReLU on load
              transpose32<X3, XF>(st + bi * 4096, lane, SM::SMALL_OFF, wval[q], wscl[q], wshl[q]);
            else
              transpose32<X3>(st + bi * 4096, lane, SM::SMALL_OFF);
          }
        } else if constexpr (XF && !AT && MODE == CONV_FWD) {
          // A: BN-ReLU on load (+ residual); B: residual only
          const int pj = stid & 7;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int row = (stid >> 3) + 16 * i;
            const bool valid = (xvalid >> i) & 1u;
            const uint32_t a = st + row * 128 + (pj << 4);
            float4 v;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
            v.x = valid ? bnrelu1(v.x, xsc.x, xsh.x) : 0.f;
            v.y = valid ? bnrelu1(v.y, xsc.y, xsh.y) : 0.f;
            v.z = valid ? bnrelu1(v.z, xsc.z, xsh.z) : 0.f;
            v.w = valid ? bnrelu1(v.w, xsc.w, xsh.w) : 0.f;
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                         : "memory");
            if constexpr (X3)
              asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a + SM::SMALL_OFF), "f"(tf32_resid(v.x)),
                           "f"(tf32_resid(v.y)), "f"(tf32_resid(v.z)), "f"(tf32_resid(v.w))
                           : "memory");
          }
          if constexpr (X3) {
            constexpr int BCH = BN * BK / 4;  // 16-B chunks of B
#pragma unroll 4
            for (int c = stid; c < BCH; c += 128)
              split_chunk(st + SM::A_BYTES + c * 16, st + SM::A_BYTES + SM::SMALL_OFF + c * 16);
          }
        } else if constexpr (MODE == CONV_WGRAD) {
          // 256 blocks in A (rows = Cout) and 256 in B (rows = R*S*C); block (g, j) = rows 4g..4g+3, k-chunk j
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            int bi = stid + 128 * (q & 1);
            int g = bi & 31, j = bi >> 5;
            uint32_t tile = st + (q < 2 ? 0 : SM::A_BYTES);
            transpose_block<X3>(tile + kmaj_off<128>(4 * g, j), (stid >> 1) & 3, SM::SMALL_OFF);
          }
        } else if constexpr (AT) {
          // A: warp w moves rows 32 (w % 4) .. +31 (its TMEM lane quadrant): lane = row, the row's 32
          // k-values from the SWIZZLE_128B tile, then hi / lo into this stage's TMEM columns
          {
            const int row = 32 * (warp & 3) + lane;
            float v[32], lo[32];
            if constexpr (SP) {  // taps 8 (kb0 + kb) .. +7 of this row from the patch (zeros past R*S)
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                if (sp_ok && tap < p.R * p.S && p.epi_direct != 6) {  // 6: timing experiment, no gathers
                  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                               : "=f"(v[4 * j]), "=f"(v[4 * j + 1]), "=f"(v[4 * j + 2]), "=f"(v[4 * j + 3])
                               : "r"(sp_base + (uint32_t)((tr * p.patch_w + ts) * 16)));
                } else {
                  v[4 * j] = v[4 * j + 1] = v[4 * j + 2] = v[4 * j + 3] = 0.f;
                }
                ++tap;
                if (++ts == p.S) {
                  ts = 0;
                  ++tr;
                }
              }
              if (kb == nkb - 1) ptx::mbar_arrive(&pempty[jt % SM::NPB]);  // the patch is in registers
            } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                           : "=f"(v[4 * j]), "=f"(v[4 * j + 1]), "=f"(v[4 * j + 2]), "=f"(v[4 * j + 3])
                           : "r"(st + row * 128 + ((j ^ (row & 7)) << 4)));
            }
            if constexpr (XF) {  // BN-ReLU on load: channel i's scale / shift from lane i
              const bool valid = xvalid & 1u;
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const float sc = __shfl_sync(0xffffffffu, xsc.x, i), sh = __shfl_sync(0xffffffffu, xsh.x, i);
                v[i] = valid ? bnrelu1(v[i], sc, sh) : 0.f;
              }
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float hi = __uint_as_float(__float_as_uint(v[i]) & 0xFFFFE000u);
              lo[i] = v[i] - hi;
              v[i] = hi;
            }
            const uint32_t ta = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + A_TCOL + 64u * s;
            if constexpr (W2_HI_SMEM) {  // hi is read by the tensor core from the stage itself
              ptx::tmem_st32(ta + 32, lo);
            } else if (!SP || p.epi_direct < 7) {  // 7 / 8: timing experiments (SP), no TMEM writes
              ptx::tmem_st32(ta, v);
              ptx::tmem_st32(ta + 32, lo);
            }
          }
          // B: residuals in shared memory, as in the plain 3xTF32 path (SP: resident, split once)
          constexpr int BCH = BN * BK / 4;
          if constexpr (!SP) {
#pragma unroll 4
            for (int c = stid; c < BCH; c += 128)
              split_chunk(st + SM::A_BYTES + c * 16, st + SM::A_BYTES + SM::BS_OFF + c * 16);
          }
          ptx::tmem_wait_st();
          ptx::tc_fence_before();
        } else {
          constexpr int CHUNKS = (BM + BN) * BK / 4;  // 16-B chunks of A and B (contiguous)
#pragma unroll 4
          for (int c = stid; c < CHUNKS; c += 128) split_chunk(st + c * 16, st + SM::SMALL_OFF + c * 16);
        }
        ptx::fence_proxy_async_smem();
        ptx::mbar_arrive(&full[s]);
      }
    }
  } else if (warp == 8) {
    // ------------------------------------------------------------------ MMA issuer
    constexpr uint32_t IDESC = ptx::idesc_tf32(BM, BN, false, false);
    // K-major SWIZZLE_NONE: LBO = distance of K-adjacent core matrices, SBO = 128 (M/N-adjacent)
    constexpr uint32_t A_LBO = BM * 16;
    constexpr uint32_t B_LBO = BN * 16;
    int it = 0, j = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
      int m0, n0, kb0, nkb;
      tm.decode(t, m0, n0, kb0, nkb, BN);
      const int ab = j & 1;
      if (j >= 2) ptx::mbar_wait(&tempty[ab], ((j >> 1) - 1) & 1);
      ptx::tc_fence_after();
      const uint32_t acc = tmem + ab * ACC_COLS;
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        int s = it % STAGES;
        ptx::mbar_wait(&full[s], (it / STAGES) & 1);
        ptx::tc_fence_after();
        if (lane == 0) {
          uint32_t sa = sbase + s * SM::STAGE_BYTES;
          uint32_t sb = SP ? sbase + (kb0 + kb) * SM::B_BYTES * (W2 ? 2 : 1) : sa + SM::A_BYTES;
          const bool sw = TMA && p.stem4 != 1;  // SWIZZLE_128B tiles, else the SWIZZLE_NONE core-matrix layout
          if constexpr (MNW) {
            // MN-major SWIZZLE_128B_BASE32B: a 4 KB block per 32 rows of A / B (LBO = 4096 between
            // them), pixel rows of 128 B, 4-row K groups 512 B apart (SBO); a k-step of 8 pixels
            // advances 8 rows = 1024 B
            constexpr uint32_t IDESC_MN = ptx::idesc_tf32(BM, BN, true, true);
            constexpr uint32_t IDESC_TMN = ptx::idesc_tf32(BM, BN, false, true);  // A K-major in TMEM
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const uint32_t ko = kk * 1024;
              const uint64_t ad = ptx::smem_desc(sa + ko, 4096, 512, 1);
              const uint64_t bd = ptx::smem_desc(sb + ko, 4096, 512, 1);
              if constexpr (AT && W2) {  // [B; Bs] as one 128-row MN-major operand (see the K-major W2 below)
                constexpr uint32_t IDESC_TMN2 = ptx::idesc_tf32(BM, 2 * BN, false, true);
                const uint32_t ta = tmem + A_TCOL + 64u * s + 8u * kk;
#ifdef POOCH_W2_FOUR
                ptx::mma_tf32_ts(acc, ta + 32, bd, IDESC_TMN2, (kb | kk) != 0 ? 1u : 0u);
                ptx::mma_tf32_ts(acc, ta, bd, IDESC_TMN2, 1u);
#else
                ptx::mma_tf32_ts(acc, ta, bd, IDESC_TMN2, (kb | kk) != 0 ? 1u : 0u);
                ptx::mma_tf32_ts(acc, ta + 32, bd, IDESC_TMN, 1u);
#endif
                (void)ad;
              } else if constexpr (AT) {  // A hi / lo from TMEM (this stage's columns), B / Bs MN-major
                const uint32_t ta = tmem + A_TCOL + 64u * s + 8u * kk;
                const uint64_t bsd = ptx::smem_desc(sb + SM::BS_OFF + ko, 4096, 512, 1);
                ptx::mma_tf32_ts(acc, ta + 32, bd, IDESC_TMN, (kb | kk) != 0 ? 1u : 0u);
                ptx::mma_tf32_ts(acc, ta, bsd, IDESC_TMN, 1u);
                ptx::mma_tf32_ts(acc, ta, bd, IDESC_TMN, 1u);
                (void)ad;
              } else if constexpr (X3) {
                const uint64_t asd = ptx::smem_desc(sa + SM::SMALL_OFF + ko, 4096, 512, 1);
                const uint64_t bsd = ptx::smem_desc(sb + SM::SMALL_OFF + ko, 4096, 512, 1);
                ptx::mma_tf32(acc, asd, bd, IDESC_MN, (kb | kk) != 0 ? 1u : 0u);
                ptx::mma_tf32(acc, ad, bsd, IDESC_MN, 1u);
                ptx::mma_tf32(acc, ad, bd, IDESC_MN, 1u);
              } else {
                ptx::mma_tf32(acc, ad, bd, IDESC_MN, (kb | kk) != 0 ? 1u : 0u);
              }
            }
          } else {
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            // SWIZZLE_NONE (cp.async / stem tiles): k-step = 2 core matrices; SWIZZLE_128B (TMA tiles):
            // 128-B rows in 1024-B atoms (SBO), k-step = +32 B inside the row
            const uint32_t ka = sw ? kk * 32 : kk * 2 * A_LBO, kbo = sw ? kk * 32 : kk * 2 * B_LBO;
            const uint32_t la = sw ? 16 : A_LBO, lb = sw ? 16 : B_LBO, sbo = sw ? 1024 : 128, lay = sw ? 2 : 0;
            uint64_t ad = ptx::smem_desc(sa + ka, la, sbo, lay);
            uint64_t bd = ptx::smem_desc(sb + kbo, lb, sbo, lay);
            if constexpr (W2) {
              // [B; Bs] as one 128-row operand: hi * [B; Bs] (N = 128: A*B's hi part and hi * Bs into
              // the two halves), then lo * B (N = 64, first half) -- the three 3xTF32 products at
              // 64 + 47 instead of 3 x 47 cycles per k-step (tools/mmaprobe); POOCH_W2_FOUR builds
              // the earlier lo * [B; Bs] + hi * [B; Bs] (a fourth, negligible product lo * Bs)
              constexpr uint32_t IDESC_W2 = ptx::idesc_tf32(BM, 2 * BN, false, false);
              const uint32_t ta = tmem + A_TCOL + 64u * s + 8u * kk;
#ifdef POOCH_W2_FOUR
              ptx::mma_tf32_ts(acc, ta + 32, bd, IDESC_W2, (kb | kk) != 0 ? 1u : 0u);
              ptx::mma_tf32_ts(acc, ta, bd, IDESC_W2, 1u);
#else
              if constexpr (W2_HI_SMEM)
                ptx::mma_tf32(acc, ad, bd, IDESC_W2, (kb | kk) != 0 ? 1u : 0u);
              else
                ptx::mma_tf32_ts(acc, ta, bd, IDESC_W2, (kb | kk) != 0 ? 1u : 0u);
              ptx::mma_tf32_ts(acc, ta + 32, bd, IDESC, 1u);
#endif
              (void)ad;
            } else if constexpr (AT) {  // A hi / lo from TMEM (this stage's columns), B / Bs from smem
              const uint32_t ta = tmem + A_TCOL + 64u * s + 8u * kk;
              uint64_t bsd = ptx::smem_desc(sb + SM::BS_OFF + kbo, lb, sbo, lay);
              ptx::mma_tf32_ts(acc, ta + 32, bd, IDESC, (kb | kk) != 0 ? 1u : 0u);
              ptx::mma_tf32_ts(acc, ta, bsd, IDESC, 1u);
              ptx::mma_tf32_ts(acc, ta, bd, IDESC, 1u);
              (void)ad;
            } else if constexpr (X3) {  // small terms first, then the big product
              uint64_t asd = ptx::smem_desc(sa + SM::SMALL_OFF + ka, la, sbo, lay);
              uint64_t bsd = ptx::smem_desc(sb + SM::SMALL_OFF + kbo, lb, sbo, lay);
              ptx::mma_tf32(acc, asd, bd, IDESC, (kb | kk) != 0 ? 1u : 0u);
              ptx::mma_tf32(acc, ad, bsd, IDESC, 1u);
              ptx::mma_tf32(acc, ad, bd, IDESC, 1u);
            } else {
              ptx::mma_tf32(acc, ad, bd, IDESC, (kb | kk) != 0 ? 1u : 0u);
            }
          }
          }  // MNW
          ptx::mma_commit(&empty[s]);
        }
        __syncwarp();
      }
      if (lane == 0) {
        if (nkb > 0) ptx::mma_commit(&tfull[ab]);
        else ptx::mbar_arrive(&tfull[ab]);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------------ epilogue
    // group eg (E2: warps 0-3 / 4-7) drains column chunks [eg * CPG, (eg + 1) * CPG) of the
    // accumulator; q4 = the warp's TMEM lane quadrant, etid = thread index within the group
    const int q4 = warp & 3;
    const int eg = E2 ? (warp >> 2) : 0;
    const int etid = tid - 128 * eg;
    constexpr int CPG = BN / 32 / NEG;
    const int row = q4 * 32 + lane;
    int j = 0;
    uint32_t chunk_seq = 0;  // column chunks staged so far (selects the staging image when NSTG = 2)
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
      int m0, n0, kb0, nkb;
      tm.decode(t, m0, n0, kb0, nkb, BN);
      const int ab = j & 1;
      ptx::mbar_wait_sleep(&tfull[ab], (j >> 1) & 1);
      ptx::tc_fence_after();
      if (p.epi_direct == 8) {  // timing experiment: hand the accumulator straight back
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[ab]);
        continue;
      }
      int gm = m0 + row;
      bool rok = gm < p.M;
      if constexpr (PIXM) {  // row -> (n, h, w) of the tile's pixel box
        const int mt_i = m0 / BM;
        const int tw_i = mt_i % p.tiles_w;
        const int th_i = (mt_i / p.tiles_w) % p.tiles_h;
        const int tn_i = mt_i / (p.tiles_w * p.tiles_h);
        const int per = p.tw * p.th;
        const int nn = tn_i * p.tn + row / per, hh = th_i * p.th + (row / p.tw) % p.th, ww = tw_i * p.tw + row % p.tw;
        rok = row < per * p.tn && nn < p.n3 && hh < p.hout && ww < p.wout;
        if (MODE == CONV_DGRAD)  // class grid -> dx pixel (st3*nn + c, st*hh + a, st*ww + b)
          gm = ((nn * p.st3 + p.dg_c) * p.H + hh * p.stride + p.dg_a) * p.W + ww * p.stride + p.dg_b;
        else
          gm = (nn * p.hout + hh) * p.wout + ww;
      }
      const uint32_t taddr = tmem + ab * ACC_COLS + ((uint32_t)(q4 * 32) << 16);
      const int z = t / (tm.mt * tm.nt);
      bool stats = false;
      if constexpr (MODE == CONV_FWD) stats = p.stat_sum != nullptr && p.epi_direct != 3;  // 3: experiment
      if (stats) ptx::named_bar_sync(1 + 2 * eg, 128);  // previous tile's reads of red[] done
      // E2 at BN = 128: the group's two column chunks in one pass -- one 64-column TMEM load, both
      // staging images filled behind one pair of barriers, two TMA stores in one bulk group, then
      // the BN partial sums of both (the per-chunk loop below pays its barriers / fence per chunk)
      const bool batched = E2 && CPG == 2 && NSTG == 2 && p.tma_store && p.epi_direct == 0;
      if (batched) {
        float v[64];
        const int c0 = eg * CPG;
        if (nkb > 0) {
          ptx::tmem_ld64(taddr + c0 * 32, v);
        } else {
#pragma unroll
          for (int i = 0; i < 64; ++i) v[i] = 0.f;
        }
        if constexpr (MODE == CONV_FWD) {
          if (p.bias != nullptr) {
#pragma unroll
            for (int i = 0; i < 64; ++i) v[i] += (n0 + c0 * 32 + i < p.Ng) ? __ldg(p.bias + n0 + c0 * 32 + i) : 0.f;
          }
          if (p.relu) {
#pragma unroll
            for (int i = 0; i < 64; ++i) v[i] = fmaxf(v[i], 0.f);
          }
        }
        const uint32_t img0 = sbase + SM::STG_OFF + eg * (NSTG * 16384u);
        if (etid == 0) ptx::bulk_wait_read0();  // this group's previous stores have read both images
        ptx::named_bar_sync(2 + 2 * eg, 128);
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const uint32_t stg = img0 + cc * 16384u + q4 * 4096;
#pragma unroll
          for (int jj = 0; jj < 8; ++jj)
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(stg + lane * 128 + ((jj ^ (lane & 7)) << 4)),
                         "f"(v[32 * cc + 4 * jj]), "f"(v[32 * cc + 4 * jj + 1]), "f"(v[32 * cc + 4 * jj + 2]),
                         "f"(v[32 * cc + 4 * jj + 3])
                         : "memory");
        }
        ptx::fence_proxy_async_smem();
        ptx::named_bar_sync(2 + 2 * eg, 128);
        if (etid == 0) {
          const int mt_i = m0 / BM;
          const int tw_i = mt_i % p.tiles_w, th_i = (mt_i / p.tiles_w) % p.tiles_h, tn_i = mt_i / (p.tiles_w * p.tiles_h);
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const int nb = n0 + (c0 + cc) * 32;
            const int accum = MODE == CONV_DGRAD ? ((p.n_split > 0 && nb >= p.n_split) ? p.accumulate2 : p.accumulate) : 0;
            if (nb < p.Ng) {
              if (p.tma_store == 1)
                ptx::tma_store_4d(&tma_d, img0 + cc * 16384u, nb, tw_i * p.tw, th_i * p.th, tn_i * p.tn, accum);
              else
                ptx::tma_store_2d(&tma_d, img0 + cc * 16384u, nb, m0, accum);
            }
          }
          ptx::bulk_commit();
        }
        if constexpr (MODE == CONV_FWD) {
          if (stats) {
            const unsigned okm = __ballot_sync(0xffffffffu, rok);
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
              const uint32_t stg = img0 + cc * 16384u + q4 * 4096;
              float p1[4] = {0.f, 0.f, 0.f, 0.f}, p2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
              for (int r = 0; r < 32; ++r) {
                float x;
                asm volatile("ld.shared.f32 %0, [%1];"
                             : "=f"(x)
                             : "r"(stg + r * 128 + ((((lane >> 2) ^ (r & 7))) << 4) + (lane & 3) * 4));
                x = ((okm >> r) & 1u) ? x : 0.f;
                p1[r & 3] += x;
                p2[r & 3] = fmaf(x, x, p2[r & 3]);
              }
              red[q4 * BN + (c0 + cc) * 32 + lane] = (p1[0] + p1[1]) + (p1[2] + p1[3]);
              red[4 * BN + q4 * BN + (c0 + cc) * 32 + lane] = (p2[0] + p2[1]) + (p2[2] + p2[3]);
            }
          }
        }
        __syncwarp();
      }
#pragma unroll 1
      for (int c = eg * CPG; c < (batched ? eg * CPG : (eg + 1) * CPG); ++c) {
        float v[32];
        if (nkb > 0) {
          ptx::tmem_ld32(taddr + c * 32, v);
          if constexpr (W2) {  // + the A * Bs half
            float v2[32];
            ptx::tmem_ld32(taddr + BN + c * 32, v2);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] += v2[i];
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.f;
        }
        const int nb = n0 + c * 32;
        if constexpr (MODE == CONV_FWD) {
          if (p.bias != nullptr) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] += (nb + i < p.Ng) ? __ldg(p.bias + nb + i) : 0.f;
          }
          if (p.relu) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
          }
        }
        // destination of row gmr, columns [col, col + 4) (gmr < 0: row not stored)
        auto dst_of = [&](int gmr, int col) -> float* {
          if constexpr (MODE == GEMM_TEST) {
            return p.d + (size_t)z * p.M * p.ldd + (size_t)gmr * p.ldd + col;
          } else if constexpr (MODE == CONV_WGRAD) {
            return p.d + ((size_t)z * p.M + gmr) * p.Ng + col;
          } else {
            if (MODE == CONV_DGRAD && p.n_split > 0)  // two-source input: split dx by channel
              return nb < p.n_split ? p.d + (size_t)gmr * p.n_split + col
                                    : p.d2 + (size_t)gmr * (p.Ng - p.n_split) + (col - p.n_split);
            return p.d + (size_t)gmr * p.Ng + col;
          }
        };
        const int accum = MODE == CONV_DGRAD ? ((p.n_split > 0 && nb >= p.n_split) ? p.accumulate2 : p.accumulate) : 0;
        if (p.epi_direct == 2) {
          // timing experiment only (POOCH_EPI_DIRECT=2): drain TMEM, store nothing
          if (rok && v[0] == 12345.f) p.d[0] = v[1];
        } else if (p.epi_direct == 1) {
          if (rok) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              if (nb + i < p.Ng) {
                float* dst = dst_of(gm, nb + i);
                float4 o = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                if (accum) {
                  float4 q = *reinterpret_cast<const float4*>(dst);
                  o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
                }
                *reinterpret_cast<float4*>(dst) = o;
              }
            }
          }
        } else {
          // Coalesced store: the warp stages its 32 rows x 32 columns in shared memory (16-B chunk j
          // of row r at chunk j ^ (r & 7): conflict free both ways), then each instruction writes
          // four whole 128-B row segments (lanes 8i..8i+7 = one row) instead of 32 scattered 16-B
          // pieces. DGRAD accumulation loads all eight old segments before adding (same fp32 add).
          // With p.tma_store the four warps' blocks form the tile's 128 x 32 SWIZZLE_128B image and
          // one thread hands it to the TMA (a plain store, or an fp32 add-reduce for accumulation).
          const uint32_t img = sbase + SM::STG_OFF + eg * (NSTG * 16384u) + (NSTG == 2 ? (chunk_seq & 1u) * 16384u : 0u);
          ++chunk_seq;
          const uint32_t stg = img + q4 * 4096;
          if (p.tma_store) {  // the TMA store that last used this staging image must have read it
            if (etid == 0) {
              if constexpr (NSTG == 2) ptx::bulk_wait_read1();
              else ptx::bulk_wait_read0();
            }
            ptx::named_bar_sync(2 + 2 * eg, 128);
          }
#pragma unroll
          for (int jj = 0; jj < 8; ++jj)
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(stg + lane * 128 + ((jj ^ (lane & 7)) << 4)),
                         "f"(v[4 * jj]), "f"(v[4 * jj + 1]), "f"(v[4 * jj + 2]), "f"(v[4 * jj + 3])
                         : "memory");
          __syncwarp();
          if (p.tma_store) {
            ptx::fence_proxy_async_smem();
            ptx::named_bar_sync(2 + 2 * eg, 128);
            if (etid == 0) {
              if (p.tma_store == 1) {
                const int mt_i = m0 / BM;
                const int tw_i = mt_i % p.tiles_w, th_i = (mt_i / p.tiles_w) % p.tiles_h, tn_i = mt_i / (p.tiles_w * p.tiles_h);
                ptx::tma_store_4d(&tma_d, img, nb, tw_i * p.tw, th_i * p.th, tn_i * p.tn, accum);
              } else {
                ptx::tma_store_2d(&tma_d, img, nb, m0, accum);
              }
              ptx::bulk_commit();
            }
          }
          if (!p.tma_store && p.epi_direct != 4) {  // 4: experiment, no stores
          const int q = lane & 7;
          const int col = nb + 4 * q;
          float* dsts[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = 4 * i + (lane >> 3);
            const int gmr = __shfl_sync(0xffffffffu, gm, r);
            const int okr = __shfl_sync(0xffffffffu, rok ? 1 : 0, r);
            dsts[i] = (okr && col < p.Ng) ? dst_of(gmr, col) : nullptr;
          }
          float4 old[8];
          if (MODE == CONV_DGRAD && accum) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              old[i] = dsts[i] ? *reinterpret_cast<const float4*>(dsts[i]) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = 4 * i + (lane >> 3);
            float4 o;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(o.x), "=f"(o.y), "=f"(o.z), "=f"(o.w)
                         : "r"(stg + r * 128 + ((q ^ (r & 7)) << 4)));
            if (MODE == CONV_DGRAD && accum) {
              o.x += old[i].x; o.y += old[i].y; o.z += old[i].z; o.w += old[i].w;
            }
            if (dsts[i]) *reinterpret_cast<float4*>(dsts[i]) = o;
          }
          }
          if constexpr (MODE == CONV_FWD) {
            if (stats) {
              // per-tile BN partial sums straight from the staged block: lane = column, rows in
              // order (deterministic), rows outside the output grid masked
              const unsigned okm = __ballot_sync(0xffffffffu, rok);
              float p1[4] = {0.f, 0.f, 0.f, 0.f}, p2[4] = {0.f, 0.f, 0.f, 0.f};  // 4 short chains
#pragma unroll
              for (int r = 0; r < 32; ++r) {
                float x;
                asm volatile("ld.shared.f32 %0, [%1];"
                             : "=f"(x)
                             : "r"(stg + r * 128 + ((((lane >> 2) ^ (r & 7))) << 4) + (lane & 3) * 4));
                x = ((okm >> r) & 1u) ? x : 0.f;
                p1[r & 3] += x;
                p2[r & 3] = fmaf(x, x, p2[r & 3]);
              }
              red[q4 * BN + c * 32 + lane] = (p1[0] + p1[1]) + (p1[2] + p1[3]);
              red[4 * BN + q4 * BN + c * 32 + lane] = (p2[0] + p2[1]) + (p2[2] + p2[3]);
            }
          }
          __syncwarp();
        }
        if constexpr (MODE == CONV_FWD) {
          if (stats && p.epi_direct == 1) {
            float sq[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              v[i] = rok ? v[i] : 0.f;
              sq[i] = v[i] * v[i];
            }
            float s1 = warp_transpose_sum32(v, lane);
            float s2 = warp_transpose_sum32(sq, lane);
            red[q4 * BN + c * 32 + lane] = s1;
            red[4 * BN + q4 * BN + c * 32 + lane] = s2;
          }
        }
      }
      // accumulator drained: hand the TMEM buffer back to the MMA warp
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[ab]);
      if constexpr (MODE == CONV_FWD) {
        if (stats) {
          ptx::named_bar_sync(1 + 2 * eg, 128);
          const int mt_idx = m0 / BM;
          for (int jj = eg * (BN / NEG) + etid; jj < (eg + 1) * (BN / NEG); jj += 128) {
            int n = n0 + jj;
            if (n < p.Ng) {
              float a = ((red[jj] + red[BN + jj]) + red[2 * BN + jj]) + red[3 * BN + jj];
              float b = ((red[4 * BN + jj] + red[5 * BN + jj]) + red[6 * BN + jj]) + red[7 * BN + jj];
              p.stat_sum[(size_t)mt_idx * p.Ng + n] = a;
              p.stat_sq[(size_t)mt_idx * p.Ng + n] = b;
            }
          }
        }
      }
    }
  }
  if ((tid == 0 || (E2 && tid == 128)) && p.tma_store) ptx::bulk_wait0();  // the epilogue's TMA stores are complete
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, TMEM_COLS);
  }
}

}  // namespace pooch
