// conv.cu -- launchers for the tcgen05 implicit-GEMM convolution passes (fwd, dgrad, wgrad)
// and the FC layer (a 1x1 "conv" on a 1x1 image), plus the split-K reduction of wgrad.
//
// 2D convs use NHWC activations and KRSC weights; 3D convs (BASELINE config 4, batch 1) use
// DHWC activations and KTRSC weights: the fourth TMA dimension is the image index in 2D and
// the depth (with its own taps, stride and padding) in 3D. A conv may read the channel
// concatenation of two tensors in place (the U-Net's skip connections).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "common.h"
#include "conv.h"
#include "igemm.cuh"

namespace pooch {

ConvGeom conv_geom(const pooch_conv_desc& d) {
  ConvGeom g{d.N, d.H, d.W, d.C, d.K, d.R, d.S, d.stride, d.pad, 0, 0, d.precision};
  g.Ho = (d.H + 2 * d.pad - d.R) / d.stride + 1;
  g.Wo = (d.W + 2 * d.pad - d.S) / d.stride + 1;
  g.D = d.D;
  g.C1 = d.C1;
  g.groups = d.groups > 1 ? d.groups : 1;
  g.stride_d = d.D > 0 ? d.stride_d : 0;
  g.Do = d.D > 0 ? (d.D + 2 * d.pad - d.R) / g.sd() + 1 : 0;
  return g;
}

bool conv_shape_ok(const ConvGeom& g) {
  bool ok = g.N > 0 && g.H > 0 && g.W > 0 && g.C > 0 && g.K > 0 && g.R > 0 && g.S > 0 && g.stride > 0 &&
            g.pad >= 0 && g.C % 4 == 0 && g.K % 4 == 0 && g.Ho > 0 && g.Wo > 0;
  if (g.groups > 1) return ok && g.C1 == 0 && gconv_shape_ok(g);
  if (g.stride_d > 0 && g.sd() > 2) return false;
  if (g.is3d() || g.C1 > 0) {
    // the 3D / two-source convs run only on the TMA-fed kernels (the launchers fail with
    // POOCH_EUSAGE if the driver offers no tensor maps); this check is structural
    ok = ok && g.C % 32 == 0 && g.K % 32 == 0 && g.stride <= 2;
    if (g.is3d()) ok = ok && g.N == 1 && g.R == g.S && g.Do > 0;
    if (g.C1 > 0) ok = ok && g.C1 % 32 == 0 && g.C1 < g.C;
  }
  return ok;
}

static CUtensorMap g_zero_map;  // placeholder parameter for the cp.async paths

template <int MODE, int BN, bool X3 = false, bool TMA = false, bool XF = false, bool AT = false, bool MNW = false,
          bool E2 = false, bool SP = false, bool W2 = false, bool SPW = false>
static pooch_status launch_igemm(const GemmParams& p, dim3 grid, cudaStream_t st, const CUtensorMap* ta = nullptr,
                                 const CUtensorMap* tb = nullptr, const CUtensorMap* tc = nullptr,
                                 const CUtensorMap* td = nullptr) {
  // deepest ring that fits 227 KB next to the epilogue staging / reduction buffers: a k-block's
  // MMAs take only 0.2-0.4 us, less than the TMA -> (3xTF32 split / wgrad transpose) -> MMA
  // latency, so the ring depth sets the throughput of the short-K and narrow (BN = 64) layers
  // AT fwd / dgrad: two epilogue staging images (the TMA store of one column chunk overlaps the
  // staging of the next; more than 3-4 ring stages measured no faster, so the smem goes here)
  // E2 (two epilogue warp groups, each with its own images): one image per group at BN = 64
  // (one column chunk per group per tile), so the ring keeps its depth
  constexpr int NEG = E2 ? 2 : 1;
  constexpr int NSTG = (AT && MODE != CONV_WGRAD) ? ((E2 && BN == 64) ? 1 : 2) : 1;
  constexpr int STAGE_B = GemmSmem<BN, 1, X3, AT, NSTG, NEG, SP>::STAGE_BYTES;
  constexpr int FIXED_B = GemmSmem<BN, 1, X3, AT, NSTG, NEG, SP>::TOTAL - STAGE_B + 64;
  constexpr int STAGES_SM = SP ? 8 : std::max(2, std::min(8, (227 * 1024 - FIXED_B) / std::max(STAGE_B, 1)));
  // AT: each stage also holds 64 TMEM columns (A hi / lo) next to the two accumulators
  constexpr int STAGES = AT ? std::min(STAGES_SM, (512 - 2 * BN * (W2 ? 2 : 1)) / 64) : STAGES_SM;
  constexpr int SMEM = GemmSmem<BN, STAGES, X3, AT, NSTG, NEG, SP>::TOTAL;
  // TMA wgrad at BN = 64 (3xTF32): six blocks of 32x32 per stage -> six auxiliary warps, one
  // block each, instead of four warps doing one or two (the transposes bound these layers)
  constexpr int NAUX = (MODE == CONV_WGRAD && TMA && X3 && BN == 64 && !AT && !XF && !MNW) ? 6 : 4;
  auto kern = igemm_kernel<MODE, BN, STAGES, X3, TMA, XF, AT, NSTG, NAUX, MNW, E2, SP, W2, SPW>;
  static bool configured = false;
  if (!configured) {
    POOCH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    configured = true;
  }
  if (grid.x == 0 || grid.y == 0 || grid.z == 0) return POOCH_OK;
  // persistent: one CTA per SM (smem-limited), tiles strided over the grid
  int64_t tiles = (int64_t)grid.x * grid.y * grid.z;
  int ctas = (int)std::min<int64_t>(tiles, 148);
  count_launch();
  kern<<<ctas, igemm_threads(MODE, X3, XF, NAUX, E2), SMEM, st>>>(p, ta ? *ta : g_zero_map, tb ? *tb : g_zero_map,
                                                          tc ? *tc : g_zero_map, td ? *td : g_zero_map);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

// TMA wgrad with MN-major operands, no transposes (POOCH_WGRAD_MN=0: the transposing kernels)
static bool mn_wgrad() {
  static int on = getenv("POOCH_WGRAD_MN") ? atoi(getenv("POOCH_WGRAD_MN")) : 1;
  return on != 0;
}

// the transpose-free 3xTF32 wgrad with its A operand in TMEM (POOCH_WGRAD_AT=0: A in smem)
static bool mn_wgrad_at() {
  static int on = getenv("POOCH_WGRAD_AT") ? atoi(getenv("POOCH_WGRAD_AT")) : 1;
  return on != 0;
}

// 3xTF32 TMA fwd / dgrad with the A operand in TMEM (POOCH_A_TMEM=0 disables)
static bool a_in_tmem() {
  static int on = getenv("POOCH_A_TMEM") ? atoi(getenv("POOCH_A_TMEM")) : 1;
  return on != 0;
}

// two epilogue warp groups for the AT fwd / dgrad kernels (POOCH_EPI2: 0 off, 1 BN = 128 only,
// 2 all tile widths, the default: 1x1 expand fwd 23 % and 1x1 reduce dgrad 20 % faster, the
// rest 0-4 %; profiles/r02_kernel_experiments.md)
// BN = 64 AT fwd / dgrad with two N = 128 MMAs per k-step over [B; Bs] (igemm.cuh W2;
// POOCH_W2=0: three N = 64 MMAs)
static bool w2() {
  static int on = getenv("POOCH_W2") ? atoi(getenv("POOCH_W2")) : 1;
  return on != 0;
}
// the same for the MN-major A-in-TMEM wgrad at BN = 64 (POOCH_WGRAD_W2: 0 off, 1 the stem patch
// wgrad only -- the default: 0.88 -> 0.80 ms at batch 256 --, 2 every BN = 64 MN-major wgrad, which
// measured 0-4 % slower for the stage-1 layers: W2's 128 accumulator columns leave TMEM for 4
// A stages instead of 6)
static int wgrad_w2() {
  static int on = getenv("POOCH_WGRAD_W2") ? atoi(getenv("POOCH_WGRAD_W2")) : 1;
  return on;
}

static int epi2() {
  static int on = getenv("POOCH_EPI2") ? atoi(getenv("POOCH_EPI2")) : 2;
  return on;
}

template <int MODE, bool TMA = false>
static pooch_status launch_bn(int bn, const GemmParams& p, dim3 grid, cudaStream_t st, int prec = 0,
                              const CUtensorMap* ta = nullptr, const CUtensorMap* tb = nullptr,
                              const CUtensorMap* tc = nullptr, const CUtensorMap* td = nullptr) {
  if constexpr (TMA && (MODE == CONV_FWD || MODE == CONV_WGRAD)) {
    if (p.xf_scale) {  // BN-ReLU on load
      if (prec) {
        if constexpr (MODE == CONV_FWD) {  // the A operand (rebuilt on load) goes to TMEM
          if (a_in_tmem()) {
            // the plain AT kernels' epilogue groups and BN = 64 MMA split (E2, W2), so the fused
            // step stays bit-identical to the plain one (W2 sums A*B and A*Bs separately)
            if (epi2() >= 2 && bn == 64 && w2())
              return launch_igemm<MODE, 64, true, true, true, true, false, true, false, true>(p, grid, st, ta, tb, tc, td);
            if (epi2() >= 1 && bn == 128)
              return launch_igemm<MODE, 128, true, true, true, true, false, true>(p, grid, st, ta, tb, tc, td);
            switch (bn) {
              case 64: return launch_igemm<MODE, 64, true, true, true, true>(p, grid, st, ta, tb, tc, td);
              case 128: return launch_igemm<MODE, 128, true, true, true, true>(p, grid, st, ta, tb, tc, td);
            }
          }
        }
        switch (bn) {
          case 64: return launch_igemm<MODE, 64, true, true, true>(p, grid, st, ta, tb, tc, td);
          case 128: return launch_igemm<MODE, 128, true, true, true>(p, grid, st, ta, tb, tc, td);
        }
      } else {
        switch (bn) {
          case 64: return launch_igemm<MODE, 64, false, true, true>(p, grid, st, ta, tb, tc, td);
          case 128: return launch_igemm<MODE, 128, false, true, true>(p, grid, st, ta, tb, tc, td);
          case 256: return launch_igemm<MODE, 256, false, true, true>(p, grid, st, ta, tb, tc, td);
        }
      }
      return fail(POOCH_EUSAGE, "bad tile width %d", bn);
    }
  } else {
    if (p.xf_scale) return fail(POOCH_EUSAGE, "BN-ReLU on load needs the TMA-fed fwd / wgrad kernels");
  }
  if (prec) {
    if constexpr (TMA && MODE != GEMM_TEST) {
      // wgrad: A in TMEM pays off at BN = 128 (stages 2-4: 3-12 % faster) but not at BN = 64
      // (stage 1, 6-9 % slower: the extra read-back of the transposed A blocks)
      if constexpr (MODE == CONV_FWD) {
        if (p.stem4 == 2) {  // the patch-gather stem (AT, one output tile width of 64)
          if (bn != 64) return fail(POOCH_EUSAGE, "patch stem: tile width 64 only (got %d)", bn);
          if (w2()) return launch_igemm<MODE, 64, true, true, false, true, false, true, true, true>(p, grid, st, ta, tb, tc, td);
          return launch_igemm<MODE, 64, true, true, false, true, false, true, true>(p, grid, st, ta, tb, tc, td);
        }
      }
      if (a_in_tmem() && !p.stem4 && (MODE != CONV_WGRAD || bn == 128)) {
        if constexpr (MODE != CONV_WGRAD) {
          if (epi2() >= 2 && bn == 64) {
            if (w2()) return launch_igemm<MODE, 64, true, true, false, true, false, true, false, true>(p, grid, st, ta, tb, tc, td);
            return launch_igemm<MODE, 64, true, true, false, true, false, true>(p, grid, st, ta, tb, tc, td);
          }
          if (epi2() >= 1 && bn == 128) return launch_igemm<MODE, 128, true, true, false, true, false, true>(p, grid, st, ta, tb, tc, td);
        }
        switch (bn) {
          case 64: return launch_igemm<MODE, 64, true, true, false, true>(p, grid, st, ta, tb, tc, td);
          case 128: return launch_igemm<MODE, 128, true, true, false, true>(p, grid, st, ta, tb, tc, td);
        }
      }
    }
    switch (bn) {
      case 64: return launch_igemm<MODE, 64, true, TMA>(p, grid, st, ta, tb, tc, td);
      case 128: return launch_igemm<MODE, 128, true, TMA>(p, grid, st, ta, tb, tc, td);
    }
    return fail(POOCH_EUSAGE, "3xTF32 supports tile widths 64 / 128 (got %d)", bn);
  }
  switch (bn) {
    case 64: return launch_igemm<MODE, 64, false, TMA>(p, grid, st, ta, tb, tc, td);
    case 128: return launch_igemm<MODE, 128, false, TMA>(p, grid, st, ta, tb, tc, td);
    case 256: return launch_igemm<MODE, 256, false, TMA>(p, grid, st, ta, tb, tc, td);
  }
  return fail(POOCH_EUSAGE, "bad tile width %d", bn);
}

// ---- TMA tensor maps (cuTensorMapEncodeTiled through the runtime's driver entry point)
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn();
static bool tma_enabled() {
  static int on = getenv("POOCH_NO_TMA") ? 0 : 1;
  return on != 0 && encode_fn() != nullptr;
}
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)f;
  });
  return fn;
}

// Activation map: dims {C, W, H, N3} (N3 = images in 2D, depth in 3D); box {32, tw*st, th*st,
// tn*st3}, traversal strides {1, st, st, st3}.
static bool map_act(CUtensorMap* m, const float* base, int N3, int H, int W, int C, int tw, int th, int tn, int st,
                    int st3) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N3};
  cuuint64_t strides[3] = {(cuuint64_t)C * 4, (cuuint64_t)W * C * 4, (cuuint64_t)H * W * C * 4};
  cuuint32_t box[4] = {32, (cuuint32_t)(tw * st), (cuuint32_t)(th * st), (cuuint32_t)(tn * st3)};
  cuuint32_t es[4] = {1, (cuuint32_t)st, (cuuint32_t)st, (cuuint32_t)st3};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// 5-D view of an activation for wgrad: dims {32, W, H, N3, C/32} (the 32-channel chunk index
// outermost, stride 128 B); box {32, tw*st, th*st, tn*st3, cb} lands as cb consecutive
// [pixel][32] blocks.
static bool map_act_chunks(CUtensorMap* m, const float* base, int N3, int H, int W, int C, int tw, int th, int tn,
                           int st, int st3, int cb, bool mn = false) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[5] = {32, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N3, (cuuint64_t)(C / 32)};
  cuuint64_t strides[4] = {(cuuint64_t)C * 4, (cuuint64_t)W * C * 4, (cuuint64_t)H * W * C * 4, 128};
  cuuint32_t box[5] = {32, (cuuint32_t)(tw * st), (cuuint32_t)(th * st), (cuuint32_t)(tn * st3), (cuuint32_t)cb};
  cuuint32_t es[5] = {1, (cuuint32_t)st, (cuuint32_t)st, (cuuint32_t)st3, 1};
  // mn: the MN-major tf32 operand layout of the transpose-free wgrad (128-B rows swizzled in
  // 32-B atoms; igemm.cuh MNW), else SWIZZLE_128B for the in-place transposes
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, (void*)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            mn ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2-D row-major matrix [rows][cols]: box {32 cols, bn rows}
static bool map_2d(CUtensorMap* m, const float* base, int rows, int cols, int bn) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)bn};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// Epilogue stores through the TMA (POOCH_NO_TMA_STORE=1: per-thread stores, for A/B tests)
static bool tma_store_enabled() {
  static int on = (getenv("POOCH_NO_TMA_STORE") || (getenv("POOCH_EPI_DIRECT") && atoi(getenv("POOCH_EPI_DIRECT")) == 4)) ? 0 : 1;
  return on != 0 && encode_fn() != nullptr;
}

// 4-D strided view {C, w, h, n} of an NHWC / NDHWC tensor for TMA stores: element (c, x, y, z)
// at base + c + x * sw + y * sh + z * sn (floats); box {32, bw, bh, bn}, SWIZZLE_128B.
static bool map_view4(CUtensorMap* m, float* base, int C, int w, int h, int n, int64_t sw, int64_t sh, int64_t sn,
                      int bw, int bh, int bnn) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
  cuuint64_t strides[3] = {(cuuint64_t)sw * 4, (cuuint64_t)sh * 4, (cuuint64_t)sn * 4};
  cuuint32_t box[4] = {32, (cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bnn};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// Output-pixel box per M-tile: maximise useful rows / (tiles * 128). In 2D the box spans several
// images only when it covers whole image heights; in 3D it is any w x h x d box.
struct PixBox {
  int tw, th, tn, tiles_w, tiles_h, tiles_n;
};
static PixBox choose_box(int N3, int Ho, int Wo, int st, int st3, bool three) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int, int, int>, PixBox> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_tuple(N3, Ho, Wo, st, st3, (int)three);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  PixBox best{1, 1, 1, Wo, Ho, N3};
  double best_eff = -1;
  for (int tw = 1; tw <= std::min(Wo, 128) && tw * st <= 256; ++tw)
    for (int th = 1; th <= std::min(Ho, 128 / tw) && th * st <= 256; ++th) {
      int tnmax = (three || th >= Ho) ? std::min(std::min(N3, 256 / st3), 128 / (tw * th)) : 1;
      for (int tn = 1; tn <= tnmax; ++tn) {
        int tx = (Wo + tw - 1) / tw, ty = (Ho + th - 1) / th, tz = (N3 + tn - 1) / tn;
        double eff = (double)N3 * Ho * Wo / ((double)tx * ty * tz * 128.0);
        if (eff > best_eff + 1e-12 || (std::abs(eff - best_eff) <= 1e-12 && tw > best.tw)) {
          best_eff = eff;
          best = PixBox{tw, th, tn, tx, ty, tz};
        }
      }
    }
  cache[key] = best;
  return best;
}

static bool fwd_uses_tma(const ConvGeom& g) { return tma_enabled() && g.C % 32 == 0 && g.stride <= 2; }
// 4-channel 2D input (the stem, the tiny CNN's first conv) through TMA boxes of one tap each:
// correct (parity-tested) but opt-in (POOCH_STEM_TMA=1) -- 16 TMA issues per k-block measured at
// ~120 ns each make it 1.8x slower than the cp.async gathers (stem fwd, batch 256: 2.29 vs 1.25 ms)
static bool fwd_uses_stem4(const ConvGeom& g) {
  static int on = getenv("POOCH_STEM_TMA") ? atoi(getenv("POOCH_STEM_TMA")) : 0;
  return on && tma_enabled() && g.C == 4 && !g.is3d() && g.C1 == 0 && g.stride <= 2;
}
static bool dgrad_uses_tma(const ConvGeom& g) { return tma_enabled() && g.K % 32 == 0 && g.stride <= 2; }

// The patch-gather stem (igemm.cuh SP): a 4-channel 2D input, 3xTF32, at most 64 output channels,
// and the patch under a 16 x 8 output box within 13 KB (the ResNet stem's 7x7 / 2: 37 x 21 pixels,
// 12.4 KB). POOCH_STEM_PATCH=0 disables it (then the cp.async gathers).
struct StemBox { int tw, th, pw, ph; };
static StemBox stem_box(const ConvGeom& g) {
  StemBox b{16, 8, 0, 0};
  if (g.Wo <= 8) { b.tw = 8; b.th = 16; }
  b.pw = (b.tw - 1) * g.stride + g.S;
  b.ph = (b.th - 1) * g.stride + g.R;
  return b;
}
static bool fwd_uses_stem_patch(const ConvGeom& g) {
  static int on = getenv("POOCH_STEM_PATCH") ? atoi(getenv("POOCH_STEM_PATCH")) : 1;
  if (!on || !tma_enabled() || g.C != 4 || g.is3d() || g.C1 > 0 || g.groups > 1 || !g.prec || g.K > 64) return false;
  const StemBox b = stem_box(g);
  // the patch within 16 KB; the weight matrix resident (at most 8 k-blocks of 8 taps)
  return b.pw * b.ph * 16 <= 13312 && b.pw <= 256 && b.ph <= 256 && g.R * g.S <= 64;
}

static int pick_bn(int n, int prec = 0) {
  return n <= 64 ? 64 : ((n <= 128 || prec) ? 128 : 256);
}

static int epi_direct() {  // POOCH_EPI_DIRECT=1: unstaged epilogue stores (A/B experiments)
  static int v = getenv("POOCH_EPI_DIRECT") ? atoi(getenv("POOCH_EPI_DIRECT")) : 0;
  return v;
}

static GemmParams base_params(const ConvGeom& g) {
  GemmParams p{};
  p.epi_direct = epi_direct();
  p.N = g.N; p.H = g.H; p.W = g.W; p.C = g.C;
  p.K = g.K; p.R = g.R; p.S = g.S;
  p.Ho = g.Ho; p.Wo = g.Wo; p.stride = g.stride; p.pad = g.pad;
  p.T = g.T();
  p.st3 = g.sd();
  p.pad3 = g.pd();
  p.dg_nt = 1;
  return p;
}

// fourth-dimension extents of the input and output grids
static int in3(const ConvGeom& g) { return g.is3d() ? g.D : g.N; }
static int out3(const ConvGeom& g) { return g.is3d() ? g.Do : g.N; }
static int64_t out_pixels(const ConvGeom& g) { return (int64_t)out3(g) * g.Ho * g.Wo; }

int conv_stat_tiles(const ConvGeom& g) {
  if (g.groups > 1) return gconv_stat_tiles(g);
  if (fwd_uses_stem_patch(g)) {
    const StemBox sb = stem_box(g);
    return ((g.Wo + sb.tw - 1) / sb.tw) * ((g.Ho + sb.th - 1) / sb.th) * g.N;
  }
  if (fwd_uses_tma(g) || fwd_uses_stem4(g)) {
    PixBox b = choose_box(out3(g), g.Ho, g.Wo, g.stride, g.sd(), g.is3d());
    return b.tiles_w * b.tiles_h * b.tiles_n;
  }
  return (int)((out_pixels(g) + 127) / 128);
}

pooch_status launch_conv_fwd(const ConvGeom& g, const float* x, const float* w, float* y, float* stat_sum,
                             float* stat_sq, const float* bias, cudaStream_t st, const float* x1,
                             const float* xf_scale, const float* xf_shift, bool relu) {
  if (g.groups > 1) {
    if (bias || x1 || xf_scale || relu) return fail(POOCH_EUSAGE, "grouped conv: plain fwd only");
    return gconv_fwd(g, x, w, y, stat_sum, stat_sq, st);
  }
  GemmParams p = base_params(g);
  p.relu = relu ? 1 : 0;
  if (xf_scale && (!fwd_uses_tma(g) || g.is3d() || g.C1 > 0 || !xf_shift))
    return fail(POOCH_EUSAGE, "BN-ReLU on load: 2D single-source conv with C %% 32 == 0 and stride <= 2 only");
  p.xf_scale = xf_scale;
  p.xf_shift = xf_shift;
  p.M = (int)out_pixels(g);
  p.Ng = g.K;
  p.Kg = g.T() * g.R * g.S * g.C;
  p.a = x; p.b = w; p.d = y;
  p.stat_sum = stat_sum; p.stat_sq = stat_sq; p.bias = bias;
  int bn = pick_bn(g.K, g.prec);
  if (fwd_uses_tma(g)) {
    const int st3 = p.st3;
    PixBox b = choose_box(out3(g), g.Ho, g.Wo, g.stride, st3, g.is3d());
    p.tw = b.tw; p.th = b.th; p.tn = b.tn;
    p.tiles_w = b.tiles_w; p.tiles_h = b.tiles_h; p.tiles_n = b.tiles_n;
    p.hout = g.Ho; p.wout = g.Wo; p.n3 = out3(g);
    p.cchunks = g.C / 32;
    const int c0 = g.C1 > 0 ? g.C1 : g.C;
    CUtensorMap ta, tb, tc;
    if (!map_act(&ta, x, in3(g), g.H, g.W, c0, b.tw, b.th, b.tn, g.stride, st3) ||
        !map_2d(&tb, w, g.K, g.T() * g.R * g.S * g.C, bn))
      return fail(POOCH_ECUDA, "cuTensorMapEncodeTiled failed (conv fwd)");
    if (g.C1 > 0) {
      p.c_split = g.C1;
      if (!map_act(&tc, x1, in3(g), g.H, g.W, g.C - g.C1, b.tw, b.th, b.tn, g.stride, st3))
        return fail(POOCH_ECUDA, "cuTensorMapEncodeTiled failed (conv fwd, second source)");
    }
    dim3 grid(b.tiles_w * b.tiles_h * b.tiles_n, (p.Ng + bn - 1) / bn, 1);
    CUtensorMap td;
    if (tma_store_enabled() &&
        map_view4(&td, y, g.K, g.Wo, g.Ho, out3(g), g.K, (int64_t)g.Wo * g.K, (int64_t)g.Ho * g.Wo * g.K, b.tw, b.th, b.tn))
      p.tma_store = 1;
    return launch_bn<CONV_FWD, true>(bn, p, grid, st, g.prec, &ta, &tb, g.C1 > 0 ? &tc : nullptr,
                                     p.tma_store ? &td : nullptr);
  }
  if (fwd_uses_stem_patch(g) && !xf_scale) {
    const StemBox sb = stem_box(g);
    p.tw = sb.tw; p.th = sb.th; p.tn = 1;
    p.tiles_w = (g.Wo + sb.tw - 1) / sb.tw; p.tiles_h = (g.Ho + sb.th - 1) / sb.th; p.tiles_n = g.N;
    p.hout = g.Ho; p.wout = g.Wo; p.n3 = g.N;
    p.stem4 = 2;
    p.patch_w = sb.pw;
    p.Kg = g.R * g.S * 4;
    p.cchunks = 1;
    CUtensorMap ta, tb;
    auto fn = encode_fn();
    // A: the input patch, box {4 channels, pw, ph, 1 image}, no swizzle (16 B per pixel, dense)
    cuuint64_t dims[4] = {4, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.N};
    cuuint64_t strides[3] = {16, (cuuint64_t)g.W * 16, (cuuint64_t)g.H * g.W * 16};
    cuuint32_t box[4] = {4, (cuuint32_t)sb.pw, (cuuint32_t)sb.ph, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    // B: the [K][R*S*4] weight matrix, box {32 k, 64 rows}, SWIZZLE_128B (K-major); the last
    // k-block's columns past R*S*4 are zero-filled
    cuuint64_t bd[2] = {(cuuint64_t)g.R * g.S * 4, (cuuint64_t)g.K};
    cuuint64_t bs[1] = {(cuuint64_t)g.R * g.S * 16};
    cuuint32_t bb[2] = {32, 64};
    cuuint32_t be[2] = {1, 1};
    if (fn(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS ||
        fn(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)w, bd, bs, bb, be, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS)
      return fail(POOCH_ECUDA, "cuTensorMapEncodeTiled failed (patch stem)");
    dim3 grid(p.tiles_w * p.tiles_h * p.tiles_n, 1, 1);
    CUtensorMap td;
    if (tma_store_enabled() &&
        map_view4(&td, y, g.K, g.Wo, g.Ho, g.N, g.K, (int64_t)g.Wo * g.K, (int64_t)g.Ho * g.Wo * g.K, sb.tw, sb.th, 1))
      p.tma_store = 1;
    return launch_bn<CONV_FWD, true>(64, p, grid, st, g.prec, &ta, &tb, nullptr, p.tma_store ? &td : nullptr);
  }
  if (fwd_uses_stem4(g) && !xf_scale) {
    PixBox b = choose_box(g.N, g.Ho, g.Wo, g.stride, 1, false);
    p.tw = b.tw; p.th = b.th; p.tn = b.tn;
    p.tiles_w = b.tiles_w; p.tiles_h = b.tiles_h; p.tiles_n = b.tiles_n;
    p.hout = g.Ho; p.wout = g.Wo; p.n3 = g.N;
    p.stem4 = 1;
    p.Kg = (g.R * g.S + 7) / 8 * 32;  // 8 taps per k-block; taps past R*S are zero boxes
    p.cchunks = 1;
    CUtensorMap ta, tb;
    auto fn = encode_fn();
    // A: {4 channels, W, H, N}, box {4, tw*st, th*st, tn}, traversal stride st, no swizzle
    cuuint64_t dims[4] = {4, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.N};
    cuuint64_t strides[3] = {16, (cuuint64_t)g.W * 16, (cuuint64_t)g.H * g.W * 16};
    cuuint32_t box[4] = {4, (cuuint32_t)(b.tw * g.stride), (cuuint32_t)(b.th * g.stride), (cuuint32_t)b.tn};
    cuuint32_t es[4] = {1, (cuuint32_t)g.stride, (cuuint32_t)g.stride, 1};
    // B: the [K][R*S*4] weight matrix, box {4 (one tap), bn rows}
    cuuint64_t bd[2] = {(cuuint64_t)g.R * g.S * 4, (cuuint64_t)g.K};
    cuuint64_t bs[1] = {(cuuint64_t)g.R * g.S * 16};
    cuuint32_t bb[2] = {4, (cuuint32_t)bn};
    cuuint32_t be[2] = {1, 1};
    if (fn(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS ||
        fn(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)w, bd, bs, bb, be, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS)
      return fail(POOCH_ECUDA, "cuTensorMapEncodeTiled failed (4-channel conv fwd)");
    dim3 grid(b.tiles_w * b.tiles_h * b.tiles_n, (p.Ng + bn - 1) / bn, 1);
    CUtensorMap td;
    if (tma_store_enabled() &&
        map_view4(&td, y, g.K, g.Wo, g.Ho, g.N, g.K, (int64_t)g.Wo * g.K, (int64_t)g.Ho * g.Wo * g.K, b.tw, b.th, b.tn))
      p.tma_store = 1;
    return launch_bn<CONV_FWD, true>(bn, p, grid, st, g.prec, &ta, &tb, nullptr, p.tma_store ? &td : nullptr);
  }
  if (g.is3d() || g.C1 > 0) return fail(POOCH_EUSAGE, "3D / two-source conv needs the TMA path");
  dim3 grid((p.M + BM - 1) / BM, (p.Ng + bn - 1) / bn, 1);
  CUtensorMap td;
  if (tma_store_enabled() && map_2d(&td, y, p.M, g.K, BM)) p.tma_store = 2;
  return launch_bn<CONV_FWD>(bn, p, grid, st, g.prec, nullptr, nullptr, nullptr, p.tma_store ? &td : nullptr);
}

pooch_status launch_conv_dgrad(const ConvGeom& g, const float* dy, const float* wt, float* dx, bool accumulate,
                               cudaStream_t st, float* dx1, bool accumulate1) {
  if (g.groups > 1) {  // wt: the plain [K][taps][C / groups] weight (no transpose)
    if (dx1) return fail(POOCH_EUSAGE, "grouped conv: one source");
    return gconv_dgrad(g, dy, wt, dx, accumulate, st);
  }
  GemmParams p = base_params(g);
  p.M = (int)((int64_t)in3(g) * g.H * g.W);
  p.Ng = g.C;
  p.Kg = g.T() * g.R * g.S * g.K;
  p.a = dy; p.b = wt; p.d = dx;
  p.accumulate = accumulate ? 1 : 0;
  if (g.C1 > 0) {
    p.n_split = g.C1;
    p.d2 = dx1;
    p.accumulate2 = accumulate1 ? 1 : 0;
  }
  int bn = pick_bn(g.C, g.prec);
  if (dgrad_uses_tma(g)) {
    // stride st: one launch per output-parity class (a, b[, c]); each is a stride-1 correlation of
    // dy with the taps of that class (sub-pixel decomposition), so every A box is a dense dy box.
    // A class with no taps (e.g. odd pixels of a 1x1 stride-2 conv) runs with K = 0: its epilogue
    // stores zeros (or leaves dx unchanged when accumulating).
    const int s_ = g.stride, s3 = p.st3;
    CUtensorMap tb;
    if (!map_2d(&tb, wt, g.C, g.T() * g.R * g.S * g.K, bn))
      return fail(POOCH_ECUDA, "cuTensorMapEncodeTiled failed (dgrad W)");
    auto first_tap = [](int cls, int pad, int st_) { return ((cls + pad) % st_ + st_) % st_; };
    auto ntaps = [](int t0, int k, int st_) { return t0 < k ? (k - t0 + st_ - 1) / st_ : 0; };
    for (int cz = 0; cz < s3; ++cz)
      for (int a = 0; a < s_; ++a)
        for (int bb = 0; bb < s_; ++bb) {
          const int dc = g.is3d() ? (g.D - cz + s3 - 1) / s3 : g.N;
          const int hc = (g.H - a + s_ - 1) / s_, wc = (g.W - bb + s_ - 1) / s_;
          if (hc <= 0 || wc <= 0 || dc <= 0) continue;
          GemmParams q = p;
          q.dg_a = a; q.dg_b = bb; q.dg_c = cz;
          q.dg_r0 = first_tap(a, g.pad, s_);
          q.dg_s0 = first_tap(bb, g.pad, s_);
          q.dg_t0 = g.is3d() ? first_tap(cz, g.pd(), s3) : 0;
          q.dg_nr = ntaps(q.dg_r0, g.R, s_);
          q.dg_ns = ntaps(q.dg_s0, g.S, s_);
          q.dg_nt = g.is3d() ? ntaps(q.dg_t0, g.R, s3) : 1;
          q.Kg = q.dg_nt * q.dg_nr * q.dg_ns * g.K;
          if (q.Kg == 0 && accumulate && (g.C1 == 0 || accumulate1)) continue;  // nothing reaches these pixels
          PixBox b = choose_box(dc, hc, wc, 1, 1, g.is3d());
          q.tw = b.tw; q.th = b.th; q.tn = b.tn;
          q.tiles_w = b.tiles_w; q.tiles_h = b.tiles_h; q.tiles_n = b.tiles_n;
          q.hout = hc; q.wout = wc; q.n3 = dc;
          q.cchunks = g.K / 32;
          CUtensorMap ta;
          if (!map_act(&ta, dy, out3(g), g.Ho, g.Wo, g.K, b.tw, b.th, b.tn, 1, 1))
            return fail(POOCH_ECUDA, "cuTensorMapEncodeTiled failed (conv dgrad)");
          dim3 grid(b.tiles_w * b.tiles_h * b.tiles_n, (p.Ng + bn - 1) / bn, 1);
          // this class's dx pixels as a strided 4-D view for the TMA store (plain, or fp32
          // add-reduce when accumulating); the two-source split keeps the per-thread stores
          CUtensorMap td;
          q.tma_store = 0;
          if (tma_store_enabled() && g.C1 == 0) {
            const int64_t hw = (int64_t)g.H * g.W * g.C;
            float* base = dx + ((int64_t)(g.is3d() ? cz : 0) * g.H + a) * g.W * g.C + (int64_t)bb * g.C;
            if (map_view4(&td, base, g.C, wc, hc, dc, (int64_t)s_ * g.C, (int64_t)s_ * g.W * g.C,
                          g.is3d() ? (int64_t)s3 * hw : hw, b.tw, b.th, b.tn))
              q.tma_store = 1;
          }
          POOCH_CHECK((launch_bn<CONV_DGRAD, true>(bn, q, grid, st, g.prec, &ta, &tb, nullptr,
                                                   q.tma_store ? &td : nullptr)));
        }
    return POOCH_OK;
  }
  if (g.is3d() || g.C1 > 0) return fail(POOCH_EUSAGE, "3D / two-source conv needs the TMA path");
  dim3 grid((p.M + BM - 1) / BM, (p.Ng + bn - 1) / bn, 1);
  return launch_bn<CONV_DGRAD>(bn, p, grid, st, g.prec);
}

// ---- wgrad: split-K over pixels into a workspace, then a fixed-order reduction.
// TMA path (C, Cout multiples of 32, stride <= 2): a k-block is a box of exactly 32 output
// pixels; the operand whose GEMM side is <= 64 rows becomes B with BN = 64, so a 64-channel
// layer does not pad the 128-row A tile (when that is x, A = im2col(x)^T and the reduction
// transposes the workspace [split][RSC][Cout] into KRSC).
struct WgradPlan {
  bool tma, swap, spw;
  int bn, mt, nt, kb, splits, kb_per_split;
  PixBox box;
};

static PixBox choose_kbox(int N3, int Ho, int Wo, int st, int st3, bool one_image = false) {
  PixBox best{};
  int64_t best_boxes = -1;
  for (int tw = 1; tw <= 32; tw *= 2)
    for (int th = 1; tw * th <= 32; th *= 2) {
      int tn = 32 / (tw * th);
      if (one_image && tn != 1) continue;
      if (tw * st > 256 || th * st > 256 || tn * st3 > 256) continue;
      int64_t tx = (Wo + tw - 1) / tw, ty = (Ho + th - 1) / th, tz = (N3 + tn - 1) / tn;
      int64_t boxes = tx * ty * tz;
      if (best_boxes < 0 || boxes < best_boxes || (boxes == best_boxes && tw > best.tw)) {
        best_boxes = boxes;
        best = PixBox{tw, th, tn, (int)tx, (int)ty, (int)tz};
      }
    }
  return best;
}

// k-blocks (32 pixels each) one wgrad split may accumulate: 2048 = 65,536 pixels, where the
// measured 3xTF32 wgrad error is ~4e-4 rel-L2 (2.3-3.5e-4 at 50 K pixels per split, 7e-4 at 100 K;
// DESIGN.md Reading 43) -- binding only at the benchmark batches (ResNet-50 at batch 2560: stage-1
// splits of ~8,700 k-blocks otherwise), not at batch 256; POOCH_WGRAD_KMAX overrides (0: no cap)
static int wgrad_kmax() {
  const char* e = getenv("POOCH_WGRAD_KMAX");  // read per call: tools/acc_probe.py switches it in-process
  return e ? atoi(e) : 2048;
}

static bool wgrad_uses_tma(const ConvGeom& g) {
  return tma_enabled() && g.C % 32 == 0 && g.K % 32 == 0 && g.stride <= 2;
}

// The stem-patch wgrad (igemm.cuh SPW): a 4-channel 2D input, 3xTF32, at most 64 output
// channels, one image per 32-pixel box, the patch under the box within the stage's 16 KB A region.
// POOCH_STEM_PATCH_WGRAD=0 disables it (then the cp.async gathers).
static bool wgrad_uses_stem_patch(const ConvGeom& g, const PixBox& b) {
  static int on = getenv("POOCH_STEM_PATCH_WGRAD") ? atoi(getenv("POOCH_STEM_PATCH_WGRAD")) : 1;
  if (!on || !tma_enabled() || g.C != 4 || g.is3d() || g.C1 > 0 || g.groups > 1 || !g.prec || g.K > 64 ||
      g.K % 32 != 0 || g.stride > 2 || !mn_wgrad() || !mn_wgrad_at())
    return false;
  const int pw = (b.tw - 1) * g.stride + g.S, ph = (b.th - 1) * g.stride + g.R;
  return b.tn == 1 && pw <= 256 && ph <= 256 && pw * ph * 16 <= BM * BK * 4;
}

static WgradPlan wgrad_plan(const ConvGeom& g) {
  WgradPlan w{};
  int rsc = g.T() * g.R * g.S * g.C;
  w.tma = wgrad_uses_tma(g);
  if (!w.tma && g.C == 4 && !g.is3d()) {
    const PixBox b = choose_kbox(g.N, g.Ho, g.Wo, g.stride, 1, true);
    if (wgrad_uses_stem_patch(g, b)) w.tma = w.spw = true;
  }
  int M = g.K, Ng = rsc;
  w.bn = 128;
  if (w.tma) {
    w.box = choose_kbox(out3(g), g.Ho, g.Wo, g.stride, g.sd(), w.spw);
    if (const char* e = w.spw ? nullptr : getenv("POOCH_KBOX")) {  // profiling experiments only
      int a = 0, b = 0, c = 0;
      if (sscanf(e, "%d,%d,%d", &a, &b, &c) == 3 && a * b * c == 32)
        w.box = PixBox{a, b, c, (g.Wo + a - 1) / a, (g.Ho + b - 1) / b, (out3(g) + c - 1) / c};
    }
    w.kb = w.box.tiles_w * w.box.tiles_h * w.box.tiles_n;
    if ((g.K <= 64 && rsc > 64) || w.spw) {
      w.swap = true;
      M = rsc;
      Ng = g.K;
    }
    if (Ng <= 64) w.bn = 64;
  } else {
    w.kb = (int)((out_pixels(g) + BK - 1) / BK);
  }
  w.mt = (M + BM - 1) / BM;
  w.nt = (Ng + w.bn - 1) / w.bn;
  const int64_t tiles = (int64_t)w.mt * w.nt;
  // split-K count from a small cost model in units of one k-block (~0.7 us on a busy SM): waves of
  // persistent CTAs x (k-blocks per split + ~6 for pipeline fill and epilogue), plus the workspace
  // write + reduction read (8 B per dW element per split at ~6.5 TB/s ~ 4.5 MB per k-block time)
  const double ws_per_split = 8.0 * g.K * rsc / 4.5e6;
  // accuracy cap on a split's length (wgrad_kmax): the search starts at the smallest split count
  // that respects it, so the cost model still picks the wave-filling count above it
  const int kmax = wgrad_kmax();
  const int s_min = kmax > 0 ? std::max(1, (w.kb + kmax - 1) / kmax) : 1;
  double best = 1e300;
  w.splits = s_min;
  for (int s = s_min; s <= std::max(s_min, w.kb / 4); ++s) {
    const int64_t waves = (tiles * s + 147) / 148;
    const double cost = (double)waves * ((w.kb + s - 1) / s + 6) + (s > 1 ? s * ws_per_split : 0.0);
    if (cost < best - 1e-9) {
      best = cost;
      w.splits = s;
    }
  }
  if (const char* e = getenv("POOCH_WGRAD_SPLITS")) w.splits = std::max(1, std::min(atoi(e), w.kb));
  // accuracy cap on a split's length: the tensor core's fp32 accumulation is biased (its error grows
  // linearly with the number of accumulated MMAs: 3xTF32 GEMM rel-L2 4.5e-6 at K = 576, 2.3e-4 at
  // K = 32768, measured), so no split accumulates more than wgrad_kmax() k-blocks in TMEM; the
  // split partials are summed in fixed order with round-to-nearest fp32 adds by the reduction
  if (kmax > 0) w.splits = std::max(w.splits, s_min);
  w.kb_per_split = (w.kb + w.splits - 1) / w.splits;
  w.splits = (w.kb + w.kb_per_split - 1) / w.kb_per_split;
  return w;
}

size_t conv_wgrad_ws_bytes(const ConvGeom& g) {
  if (g.groups > 1) return gconv_wgrad_ws_bytes(g);
  WgradPlan w = wgrad_plan(g);
  return (w.splits > 1 || w.swap) ? (size_t)w.splits * g.K * g.T() * g.R * g.S * g.C * sizeof(float) : 0;
}

__global__ void splitk_reduce_kernel(const float4* __restrict__ ws, float4* __restrict__ out, int64_t n4,
                                     int splits) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = ws[i];
    for (int s = 1; s < splits; ++s) {
      float4 b = ws[(int64_t)s * n4 + i];
      a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    }
    out[i] = a;
  }
}

// ws [split][rows][cols] -> out [cols][rows] = sum over splits (in split order), 32 x 32 tiles
__global__ void splitk_reduce_t_kernel(const float* __restrict__ ws, float* __restrict__ out, int rows, int cols,
                                       int splits) {
  __shared__ float tile[32][33];
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  const int64_t plane = (int64_t)rows * cols;
  for (int i = ty; i < 32; i += 8) {
    int r = r0 + i, c = c0 + tx;
    float a = 0.f;
    if (r < rows && c < cols) {
      const float* q = ws + (int64_t)r * cols + c;
      a = q[0];
      for (int s = 1; s < splits; ++s) a += q[s * plane];
    }
    tile[i][tx] = a;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    int c = c0 + i, r = r0 + tx;
    if (c < cols && r < rows) out[(int64_t)c * rows + r] = tile[tx][i];
  }
}

pooch_status launch_conv_wgrad(const ConvGeom& g, const float* x, const float* dy, float* dw, float* ws,
                               size_t ws_bytes, cudaStream_t st, const float* x1, const float* xf_scale,
                               const float* xf_shift) {
  if (g.groups > 1) {
    if (x1 || xf_scale) return fail(POOCH_EUSAGE, "grouped conv: plain wgrad only");
    return gconv_wgrad(g, x, dy, dw, ws, ws_bytes, st);
  }
  WgradPlan w = wgrad_plan(g);
  GemmParams p = base_params(g);
  if (xf_scale && (!w.tma || g.is3d() || g.C1 > 0 || !xf_shift))
    return fail(POOCH_EUSAGE, "BN-ReLU on load: TMA-fed 2D single-source wgrad only");
  p.xf_scale = xf_scale;
  p.xf_shift = xf_shift;
  const int rsc = g.T() * g.R * g.S * g.C;
  p.M = w.swap ? rsc : g.K;
  p.Ng = w.swap ? g.K : rsc;
  p.Kg = (int)out_pixels(g);
  p.a = dy; p.b = x;
  p.kb_per_split = w.kb_per_split;
  bool use_ws = w.splits > 1 || w.swap;
  if (use_ws && ws_bytes < conv_wgrad_ws_bytes(g))
    return fail(POOCH_EUSAGE, "wgrad workspace too small: %zu < %zu", ws_bytes, conv_wgrad_ws_bytes(g));
  p.d = use_ws ? ws : dw;
  dim3 grid(w.mt, w.nt, w.splits);
  if (w.tma) {
    const int st3 = p.st3;
    p.tw = w.box.tw; p.th = w.box.th; p.tn = w.box.tn;
    p.tiles_w = w.box.tiles_w; p.tiles_h = w.box.tiles_h; p.tiles_n = w.box.tiles_n;
    p.hout = g.Ho; p.wout = g.Wo; p.n3 = out3(g);
    p.wg_a_is_x = w.swap ? 1 : 0;
    // chunks per box: the largest power of two <= 4 dividing the channel count in chunks (so a
    // box never straddles two taps or the two sources) and no larger than the tile
    auto cb_of = [](int ch, int rows) {
      int cb = 4;
      while (cb > 1 && ((ch / 32) % cb != 0 || 32 * cb > rows)) cb >>= 1;
      return cb;
    };
    const int cb_dy = cb_of(g.K, w.swap ? w.bn : BM);
    const int cx_rows = w.swap ? BM : w.bn;
    int cb_x = cb_of(g.C, cx_rows);
    if (g.C1 > 0) cb_x = std::min(cb_of(g.C1, cx_rows), cb_of(g.C - g.C1, cx_rows));
    p.wg_cba = w.swap ? cb_x : cb_dy;
    p.wg_cbb = w.swap ? cb_dy : cb_x;
    const int c0 = g.C1 > 0 ? g.C1 : g.C;
    // transpose-free MN-major operands (igemm.cuh MNW) unless BN-ReLU-on-load rewrites them
    const bool mn = mn_wgrad() && !p.xf_scale;
    CUtensorMap tdy, tx, tx1;
    if (!map_act_chunks(&tdy, dy, out3(g), g.Ho, g.Wo, g.K, w.box.tw, w.box.th, w.box.tn, 1, 1, cb_dy, mn) ||
        (!w.spw && !map_act_chunks(&tx, x, in3(g), g.H, g.W, c0, w.box.tw, w.box.th, w.box.tn, g.stride, st3, cb_x, mn)))
      return fail(POOCH_ECUDA, "cuTensorMapEncodeTiled failed (conv wgrad)");
    if (g.C1 > 0) {
      p.c_split = g.C1;
      if (!map_act_chunks(&tx1, x1, in3(g), g.H, g.W, g.C - g.C1, w.box.tw, w.box.th, w.box.tn, g.stride, st3, cb_x,
                          mn))
        return fail(POOCH_ECUDA, "cuTensorMapEncodeTiled failed (conv wgrad, second source)");
    }
    if (w.spw) {  // A: the input patch, box {4 channels, pw, ph, 1 image}, no swizzle (16 B per pixel)
      const int pw = (w.box.tw - 1) * g.stride + g.S, ph = (w.box.th - 1) * g.stride + g.R;
      p.patch_w = pw;
      auto fn = encode_fn();
      cuuint64_t dims[4] = {4, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.N};
      cuuint64_t strides[3] = {16, (cuuint64_t)g.W * 16, (cuuint64_t)g.H * g.W * 16};
      cuuint32_t box[4] = {4, (cuuint32_t)pw, (cuuint32_t)ph, 1};
      cuuint32_t es[4] = {1, 1, 1, 1};
      if (fn(&tx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
          CUDA_SUCCESS)
        return fail(POOCH_ECUDA, "cuTensorMapEncodeTiled failed (patch wgrad)");
      if (wgrad_w2() >= 1)
        POOCH_CHECK((launch_igemm<CONV_WGRAD, 64, true, true, false, true, true, false, false, true, true>(
            p, grid, st, &tx, &tdy)));
      else
        POOCH_CHECK((launch_igemm<CONV_WGRAD, 64, true, true, false, true, true, false, false, false, true>(
            p, grid, st, &tx, &tdy)));
    } else {
    const CUtensorMap* ta = w.swap ? &tx : &tdy;
    const CUtensorMap* tb = w.swap ? &tdy : &tx;
    const CUtensorMap* tc = g.C1 > 0 ? &tx1 : nullptr;
    if (mn) {
      if (g.prec) {
        // A in TMEM (hi / lo gathered from the MN-major blocks) unless POOCH_WGRAD_AT=0
        if (mn_wgrad_at()) {
          if (w.bn == 64 && wgrad_w2() >= 2)
            POOCH_CHECK((launch_igemm<CONV_WGRAD, 64, true, true, false, true, true, false, false, true>(p, grid, st, ta, tb, tc)));
          else if (w.bn == 64) POOCH_CHECK((launch_igemm<CONV_WGRAD, 64, true, true, false, true, true>(p, grid, st, ta, tb, tc)));
          else POOCH_CHECK((launch_igemm<CONV_WGRAD, 128, true, true, false, true, true>(p, grid, st, ta, tb, tc)));
        } else if (w.bn == 64) POOCH_CHECK((launch_igemm<CONV_WGRAD, 64, true, true, false, false, true>(p, grid, st, ta, tb, tc)));
        else POOCH_CHECK((launch_igemm<CONV_WGRAD, 128, true, true, false, false, true>(p, grid, st, ta, tb, tc)));
      } else {
        if (w.bn == 64) POOCH_CHECK((launch_igemm<CONV_WGRAD, 64, false, true, false, false, true>(p, grid, st, ta, tb, tc)));
        else if (w.bn == 128) POOCH_CHECK((launch_igemm<CONV_WGRAD, 128, false, true, false, false, true>(p, grid, st, ta, tb, tc)));
        else POOCH_CHECK((launch_igemm<CONV_WGRAD, 256, false, true, false, false, true>(p, grid, st, ta, tb, tc)));
      }
    } else {
      POOCH_CHECK((launch_bn<CONV_WGRAD, true>(w.bn, p, grid, st, g.prec, ta, tb, tc)));
    }
    }  // !spw
  } else if (g.is3d() || g.C1 > 0) {
    return fail(POOCH_EUSAGE, "3D / two-source conv needs the TMA path");
  } else if (g.prec) {
    POOCH_CHECK((launch_igemm<CONV_WGRAD, 128, true>(p, grid, st)));
  } else {
    POOCH_CHECK((launch_igemm<CONV_WGRAD, 128, false>(p, grid, st)));
  }
  if (w.swap) {
    count_launch();
    dim3 rg((g.K + 31) / 32, (rsc + 31) / 32);
    splitk_reduce_t_kernel<<<rg, dim3(32, 8), 0, st>>>(ws, dw, rsc, g.K, w.splits);
    POOCH_CUDA(cudaGetLastError());
  } else if (use_ws) {
    int64_t n4 = (int64_t)g.K * p.Ng / 4;
    int blocks = (int)std::min<int64_t>((n4 + 255) / 256, 148 * 8);
    count_launch();
    splitk_reduce_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const float4*>(ws), reinterpret_cast<float4*>(dw),
                                                  n4, w.splits);
    POOCH_CUDA(cudaGetLastError());
  }
  return POOCH_OK;
}

}  // namespace pooch

using namespace pooch;

extern "C" pooch_status pooch_op_conv_fwd(const pooch_conv_desc* d, const float* x, const float* w, float* y,
                                          float* stat_sum, float* stat_sq, void* stream) {
  if (!d || !x || !w || !y) return fail(POOCH_EUSAGE, "null argument");
  ConvGeom g = conv_geom(*d);
  if (g.C1 != 0 || !conv_shape_ok(g)) return fail(POOCH_EUSAGE, "unsupported conv shape");
  if ((stat_sum == nullptr) != (stat_sq == nullptr)) return fail(POOCH_EUSAGE, "stat_sum/stat_sq must pair");
  return launch_conv_fwd(g, x, w, y, stat_sum, stat_sq, nullptr, (cudaStream_t)stream);
}

extern "C" pooch_status pooch_op_conv_dgrad(const pooch_conv_desc* d, const float* dy, const float* wt, float* dx,
                                            int32_t accumulate, void* stream) {
  if (!d || !dy || !wt || !dx) return fail(POOCH_EUSAGE, "null argument");
  ConvGeom g = conv_geom(*d);
  if (g.C1 != 0 || !conv_shape_ok(g)) return fail(POOCH_EUSAGE, "unsupported conv shape");
  return launch_conv_dgrad(g, dy, wt, dx, accumulate != 0, (cudaStream_t)stream);
}

extern "C" size_t pooch_op_conv_wgrad_ws_bytes(const pooch_conv_desc* d) {
  if (!d) return 0;
  return conv_wgrad_ws_bytes(conv_geom(*d));
}

extern "C" pooch_status pooch_op_conv_wgrad(const pooch_conv_desc* d, const float* x, const float* dy, float* dw,
                                            float* ws, size_t ws_bytes, void* stream) {
  if (!d || !x || !dy || !dw) return fail(POOCH_EUSAGE, "null argument");
  ConvGeom g = conv_geom(*d);
  if (g.C1 != 0 || !conv_shape_ok(g)) return fail(POOCH_EUSAGE, "unsupported conv shape");
  return launch_conv_wgrad(g, x, dy, dw, ws, ws_bytes, (cudaStream_t)stream);
}

extern "C" pooch_status pooch_op_conv_fwd2(const pooch_conv_desc* d, const float* x0, const float* x1, const float* w,
                                           float* y, float* stat_sum, float* stat_sq, void* stream) {
  if (!d || !x0 || !x1 || !w || !y) return fail(POOCH_EUSAGE, "null argument");
  ConvGeom g = conv_geom(*d);
  if (g.C1 <= 0 || !conv_shape_ok(g)) return fail(POOCH_EUSAGE, "unsupported two-source conv shape");
  if ((stat_sum == nullptr) != (stat_sq == nullptr)) return fail(POOCH_EUSAGE, "stat_sum/stat_sq must pair");
  return launch_conv_fwd(g, x0, w, y, stat_sum, stat_sq, nullptr, (cudaStream_t)stream, x1);
}

extern "C" pooch_status pooch_op_conv_dgrad2(const pooch_conv_desc* d, const float* dy, const float* wt, float* dx0,
                                             float* dx1, int32_t accumulate0, int32_t accumulate1, void* stream) {
  if (!d || !dy || !wt || !dx0 || !dx1) return fail(POOCH_EUSAGE, "null argument");
  ConvGeom g = conv_geom(*d);
  if (g.C1 <= 0 || !conv_shape_ok(g)) return fail(POOCH_EUSAGE, "unsupported two-source conv shape");
  return launch_conv_dgrad(g, dy, wt, dx0, accumulate0 != 0, (cudaStream_t)stream, dx1, accumulate1 != 0);
}

extern "C" pooch_status pooch_op_conv_wgrad2(const pooch_conv_desc* d, const float* x0, const float* x1,
                                             const float* dy, float* dw, float* ws, size_t ws_bytes, void* stream) {
  if (!d || !x0 || !x1 || !dy || !dw) return fail(POOCH_EUSAGE, "null argument");
  ConvGeom g = conv_geom(*d);
  if (g.C1 <= 0 || !conv_shape_ok(g)) return fail(POOCH_EUSAGE, "unsupported two-source conv shape");
  return launch_conv_wgrad(g, x0, dy, dw, ws, ws_bytes, (cudaStream_t)stream, x1);
}

extern "C" pooch_status pooch_op_gemm_test(const float* A, const float* B, float* D, int32_t M, int32_t N,
                                           int32_t K, int32_t a_mn, int32_t b_mn, int32_t bn, int32_t splits,
                                           void* stream) {
  if (!A || !B || !D || M <= 0 || N <= 0 || K <= 0 || splits < 1) return fail(POOCH_EUSAGE, "bad gemm args");
  if (M % 4 || N % 4 || K % 4) return fail(POOCH_EUSAGE, "M, N, K must be multiples of 4");
  // a_mn / b_mn are reserved (MN-major operands are not supported); a_mn == 2 selects 3xTF32
  int test_prec = 0;
  if (a_mn == 2) {
    test_prec = 1;
    a_mn = 0;
  }
  if (a_mn || b_mn) return fail(POOCH_EUSAGE, "MN-major operands are not supported (K-major only)");
  GemmParams p{};
  p.epi_direct = epi_direct();
  p.M = M; p.Ng = N; p.Kg = K;
  p.a = A; p.b = B; p.d = D;
  p.lda = K;
  p.ldb = K;
  p.ldd = N;
  int kb = (K + BK - 1) / BK;
  p.kb_per_split = (kb + splits - 1) / splits;
  dim3 grid((M + BM - 1) / BM, (N + bn - 1) / bn, splits);
  return launch_bn<GEMM_TEST>(bn, p, grid, (cudaStream_t)stream, b_mn == 0 && a_mn == 0 ? test_prec : 0);
}

extern "C" pooch_status pooch_op_conv_fwd_bnrelu(const pooch_conv_desc* d, const float* x, const float* scale,
                                                 const float* shift, const float* w, float* y, float* stat_sum,
                                                 float* stat_sq, void* stream) {
  if (!d || !x || !scale || !shift || !w || !y) return fail(POOCH_EUSAGE, "null argument");
  ConvGeom g = conv_geom(*d);
  if (!conv_shape_ok(g)) return fail(POOCH_EUSAGE, "unsupported conv shape");
  return launch_conv_fwd(g, x, w, y, stat_sum, stat_sq, nullptr, (cudaStream_t)stream, nullptr, scale, shift);
}

extern "C" pooch_status pooch_op_conv_wgrad_bnrelu(const pooch_conv_desc* d, const float* x, const float* scale,
                                                   const float* shift, const float* dy, float* dw, float* ws,
                                                   size_t ws_bytes, void* stream) {
  if (!d || !x || !scale || !shift || !dy || !dw) return fail(POOCH_EUSAGE, "null argument");
  ConvGeom g = conv_geom(*d);
  if (!conv_shape_ok(g)) return fail(POOCH_EUSAGE, "unsupported conv shape");
  return launch_conv_wgrad(g, x, dy, dw, ws, ws_bytes, (cudaStream_t)stream, nullptr, scale, shift);
}

extern "C" int64_t pooch_op_conv_stat_tiles(const pooch_conv_desc* d) {
  if (!d) return 0;
  return conv_stat_tiles(conv_geom(*d));
}
