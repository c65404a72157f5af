// conv.cu -- launchers for the tcgen05 implicit-GEMM convolution passes (fwd, dgrad, wgrad)
// and the FC layer (a 1x1 "conv" on a 1x1 image), plus the split-K reduction of wgrad.
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
  return g;
}

bool conv_shape_ok(const ConvGeom& g) {
  return g.N > 0 && g.H > 0 && g.W > 0 && g.C > 0 && g.K > 0 && g.R > 0 && g.S > 0 && g.stride > 0 &&
         g.pad >= 0 && g.C % 4 == 0 && g.K % 4 == 0 && g.Ho > 0 && g.Wo > 0;
}

static CUtensorMap g_zero_map;  // placeholder parameter for the cp.async paths

template <int MODE, int BN, bool X3 = false, bool TMA = false>
static pooch_status launch_igemm(const GemmParams& p, dim3 grid, cudaStream_t st, const CUtensorMap* ta = nullptr,
                                 const CUtensorMap* tb = nullptr) {
  // deepest ring that fits 227 KB: TMA wgrad has the longest load -> MMA latency (TMA, then an
  // in-place transpose by the auxiliary warps), so it gets every stage that fits
  constexpr int STAGE_B = (BM + BN) * BK * 4 * (X3 ? 2 : 1);
  constexpr int STAGES = (MODE == CONV_WGRAD && TMA) ? std::min(8, (200 * 1024) / STAGE_B) : (X3 ? 3 : 4);
  constexpr int SMEM = GemmSmem<BN, STAGES, X3>::TOTAL;
  auto kern = igemm_kernel<MODE, BN, STAGES, X3, TMA>;
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
  kern<<<ctas, igemm_threads(MODE, X3), SMEM, st>>>(p, ta ? *ta : g_zero_map, tb ? *tb : g_zero_map);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

template <int MODE, bool TMA = false>
static pooch_status launch_bn(int bn, const GemmParams& p, dim3 grid, cudaStream_t st, int prec = 0,
                              const CUtensorMap* ta = nullptr, const CUtensorMap* tb = nullptr) {
  if (prec) {
    switch (bn) {
      case 64: return launch_igemm<MODE, 64, true, TMA>(p, grid, st, ta, tb);
      case 128: return launch_igemm<MODE, 128, true, TMA>(p, grid, st, ta, tb);
    }
    return fail(POOCH_EUSAGE, "3xTF32 supports tile widths 64 / 128 (got %d)", bn);
  }
  switch (bn) {
    case 64: return launch_igemm<MODE, 64, false, TMA>(p, grid, st, ta, tb);
    case 128: return launch_igemm<MODE, 128, false, TMA>(p, grid, st, ta, tb);
    case 256: return launch_igemm<MODE, 256, false, TMA>(p, grid, st, ta, tb);
  }
  return fail(POOCH_EUSAGE, "bad tile width %d", bn);
}

// ---- TMA tensor maps (cuTensorMapEncodeTiled through the runtime's driver entry point)
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

// 4-D NHWC activation map: dims {C, W, H, N}; box {32, tw*st, th*st, tn}, traversal stride st.
static bool map_nhwc(CUtensorMap* m, const float* base, int N, int H, int W, int C, int tw, int th, int tn, int st) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  cuuint64_t strides[3] = {(cuuint64_t)C * 4, (cuuint64_t)W * C * 4, (cuuint64_t)H * W * C * 4};
  cuuint32_t box[4] = {32, (cuuint32_t)(tw * st), (cuuint32_t)(th * st), (cuuint32_t)tn};
  cuuint32_t es[4] = {1, (cuuint32_t)st, (cuuint32_t)st, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// 5-D view of an NHWC activation for wgrad: dims {32, W, H, N, C/32} (the 32-channel chunk index
// outermost, stride 128 B); box {32, tw*st, th*st, tn, cb} lands as cb consecutive [pixel][32] blocks.
static bool map_nhwc_chunks(CUtensorMap* m, const float* base, int N, int H, int W, int C, int tw, int th, int tn,
                            int st, int cb) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[5] = {32, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N, (cuuint64_t)(C / 32)};
  cuuint64_t strides[4] = {(cuuint64_t)C * 4, (cuuint64_t)W * C * 4, (cuuint64_t)H * W * C * 4, 128};
  cuuint32_t box[5] = {32, (cuuint32_t)(tw * st), (cuuint32_t)(th * st), (cuuint32_t)tn, (cuuint32_t)cb};
  cuuint32_t es[5] = {1, (cuuint32_t)st, (cuuint32_t)st, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, (void*)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
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

// Output-pixel box per M-tile: maximise useful rows / (tiles * 128).
struct PixBox {
  int tw, th, tn, tiles_w, tiles_h, tiles_n;
};
static PixBox choose_box(int N, int Ho, int Wo, int st) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int>, PixBox> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_tuple(N, Ho, Wo, st);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  PixBox best{1, 1, 1, Wo, Ho, N};
  double best_eff = -1;
  for (int tw = 1; tw <= std::min(Wo, 128) && tw * st <= 256; ++tw)
    for (int th = 1; th <= std::min(Ho, 128 / tw) && th * st <= 256; ++th) {
      int tnmax = th >= Ho ? std::min(std::min(N, 256), 128 / (tw * th)) : 1;
      for (int tn = 1; tn <= tnmax; ++tn) {
        int tx = (Wo + tw - 1) / tw, ty = (Ho + th - 1) / th, tz = (N + tn - 1) / tn;
        double eff = (double)N * Ho * Wo / ((double)tx * ty * tz * 128.0);
        if (eff > best_eff + 1e-12 || (std::abs(eff - best_eff) <= 1e-12 && tw > best.tw)) {
          best_eff = eff;
          best = PixBox{tw, th, tn, tx, ty, tz};
        }
      }
    }
  cache[key] = best;
  return best;
}

static bool tma_enabled() {
  static int on = getenv("POOCH_NO_TMA") ? 0 : 1;
  return on != 0 && encode_fn() != nullptr;
}

static bool fwd_uses_tma(const ConvGeom& g) { return tma_enabled() && g.C % 32 == 0 && g.stride <= 2; }
static bool dgrad_uses_tma(const ConvGeom& g) { return tma_enabled() && g.K % 32 == 0 && g.stride <= 2; }

static int pick_bn(int n, int prec = 0) {
  return n <= 64 ? 64 : ((n <= 128 || prec) ? 128 : 256);
}

static GemmParams base_params(const ConvGeom& g) {
  GemmParams p{};
  p.N = g.N; p.H = g.H; p.W = g.W; p.C = g.C;
  p.K = g.K; p.R = g.R; p.S = g.S;
  p.Ho = g.Ho; p.Wo = g.Wo; p.stride = g.stride; p.pad = g.pad;
  return p;
}

int conv_stat_tiles(const ConvGeom& g) {
  if (fwd_uses_tma(g)) {
    PixBox b = choose_box(g.N, g.Ho, g.Wo, g.stride);
    return b.tiles_w * b.tiles_h * b.tiles_n;
  }
  return (g.N * g.Ho * g.Wo + 127) / 128;
}

pooch_status launch_conv_fwd(const ConvGeom& g, const float* x, const float* w, float* y, float* stat_sum,
                             float* stat_sq, const float* bias, cudaStream_t st) {
  GemmParams p = base_params(g);
  p.M = g.N * g.Ho * g.Wo;
  p.Ng = g.K;
  p.Kg = g.R * g.S * g.C;
  p.a = x; p.b = w; p.d = y;
  p.stat_sum = stat_sum; p.stat_sq = stat_sq; p.bias = bias;
  int bn = pick_bn(g.K, g.prec);
  if (fwd_uses_tma(g)) {
    PixBox b = choose_box(g.N, g.Ho, g.Wo, g.stride);
    p.tw = b.tw; p.th = b.th; p.tn = b.tn;
    p.tiles_w = b.tiles_w; p.tiles_h = b.tiles_h; p.tiles_n = b.tiles_n;
    p.hout = g.Ho; p.wout = g.Wo;
    p.cchunks = g.C / 32;
    CUtensorMap ta, tb;
    if (!map_nhwc(&ta, x, g.N, g.H, g.W, g.C, b.tw, b.th, b.tn, g.stride) ||
        !map_2d(&tb, w, g.K, g.R * g.S * g.C, bn))
      return fail(POOCH_ECUDA, "cuTensorMapEncodeTiled failed (conv fwd)");
    dim3 grid(b.tiles_w * b.tiles_h * b.tiles_n, (p.Ng + bn - 1) / bn, 1);
    return launch_bn<CONV_FWD, true>(bn, p, grid, st, g.prec, &ta, &tb);
  }
  dim3 grid((p.M + BM - 1) / BM, (p.Ng + bn - 1) / bn, 1);
  return launch_bn<CONV_FWD>(bn, p, grid, st, g.prec);
}

pooch_status launch_conv_dgrad(const ConvGeom& g, const float* dy, const float* wt, float* dx, bool accumulate,
                               cudaStream_t st) {
  GemmParams p = base_params(g);
  p.M = g.N * g.H * g.W;
  p.Ng = g.C;
  p.Kg = g.R * g.S * g.K;
  p.a = dy; p.b = wt; p.d = dx;
  p.accumulate = accumulate ? 1 : 0;
  int bn = pick_bn(g.C, g.prec);
  if (dgrad_uses_tma(g)) {
    // stride st: one launch per output-parity class (a, b); each is a stride-1 correlation of dy
    // with the taps of that class (sub-pixel decomposition), so every A box is a dense dy box.
    // A class with no taps (e.g. odd pixels of a 1x1 stride-2 conv) runs with K = 0: its epilogue
    // stores zeros (or leaves dx unchanged when accumulating).
    const int s_ = g.stride;
    CUtensorMap tb;
    if (!map_2d(&tb, wt, g.C, g.R * g.S * g.K, bn)) return fail(POOCH_ECUDA, "cuTensorMapEncodeTiled failed (dgrad W)");
    for (int a = 0; a < s_; ++a)
      for (int bb = 0; bb < s_; ++bb) {
        const int hc = (g.H - a + s_ - 1) / s_, wc = (g.W - bb + s_ - 1) / s_;
        if (hc <= 0 || wc <= 0) continue;
        GemmParams q = p;
        q.dg_a = a; q.dg_b = bb;
        q.dg_r0 = ((a + g.pad) % s_ + s_) % s_;
        q.dg_s0 = ((bb + g.pad) % s_ + s_) % s_;
        q.dg_nr = q.dg_r0 < g.R ? (g.R - q.dg_r0 + s_ - 1) / s_ : 0;
        q.dg_ns = q.dg_s0 < g.S ? (g.S - q.dg_s0 + s_ - 1) / s_ : 0;
        q.Kg = q.dg_nr * q.dg_ns * g.K;
        if (q.Kg == 0 && accumulate) continue;  // nothing reaches these pixels: dx stays as it is
        PixBox b = choose_box(g.N, hc, wc, 1);
        q.tw = b.tw; q.th = b.th; q.tn = b.tn;
        q.tiles_w = b.tiles_w; q.tiles_h = b.tiles_h; q.tiles_n = b.tiles_n;
        q.hout = hc; q.wout = wc;
        q.cchunks = g.K / 32;
        CUtensorMap ta;
        if (!map_nhwc(&ta, dy, g.N, g.Ho, g.Wo, g.K, b.tw, b.th, b.tn, 1))
          return fail(POOCH_ECUDA, "cuTensorMapEncodeTiled failed (conv dgrad)");
        dim3 grid(b.tiles_w * b.tiles_h * b.tiles_n, (p.Ng + bn - 1) / bn, 1);
        POOCH_CHECK((launch_bn<CONV_DGRAD, true>(bn, q, grid, st, g.prec, &ta, &tb)));
      }
    return POOCH_OK;
  }
  dim3 grid((p.M + BM - 1) / BM, (p.Ng + bn - 1) / bn, 1);
  return launch_bn<CONV_DGRAD>(bn, p, grid, st, g.prec);
}

// ---- wgrad: split-K over pixels into a workspace, then a fixed-order reduction.
// TMA path (C, Cout multiples of 32, stride <= 2): a k-block is a box of exactly 32 output
// pixels; the operand whose GEMM side is <= 64 rows becomes B with BN = 64, so a 64-channel
// layer does not pad the 128-row A tile (when that is x, A = im2col(x)^T and the reduction
// transposes the workspace [split][RSC][Cout] into KRSC).
struct WgradPlan {
  bool tma, swap;
  int bn, mt, nt, kb, splits, kb_per_split;
  PixBox box;
};

static PixBox choose_kbox(int N, int Ho, int Wo, int st) {
  PixBox best{};
  int64_t best_boxes = -1;
  for (int tw = 1; tw <= 32; tw *= 2)
    for (int th = 1; tw * th <= 32; th *= 2) {
      int tn = 32 / (tw * th);
      if (tw * st > 256 || th * st > 256) continue;
      int64_t tx = (Wo + tw - 1) / tw, ty = (Ho + th - 1) / th, tz = (N + tn - 1) / tn;
      int64_t boxes = tx * ty * tz;
      if (best_boxes < 0 || boxes < best_boxes || (boxes == best_boxes && tw > best.tw)) {
        best_boxes = boxes;
        best = PixBox{tw, th, tn, (int)tx, (int)ty, (int)tz};
      }
    }
  return best;
}

static bool wgrad_uses_tma(const ConvGeom& g) {
  return tma_enabled() && g.C % 32 == 0 && g.K % 32 == 0 && g.stride <= 2;
}

static WgradPlan wgrad_plan(const ConvGeom& g) {
  WgradPlan w{};
  int rsc = g.R * g.S * g.C;
  w.tma = wgrad_uses_tma(g);
  int M = g.K, Ng = rsc;
  w.bn = 128;
  if (w.tma) {
    w.box = choose_kbox(g.N, g.Ho, g.Wo, g.stride);
    if (const char* e = getenv("POOCH_KBOX")) {  // profiling experiments only
      int a = 0, b = 0, c = 0;
      if (sscanf(e, "%d,%d,%d", &a, &b, &c) == 3 && a * b * c == 32)
        w.box = PixBox{a, b, c, (g.Wo + a - 1) / a, (g.Ho + b - 1) / b, (g.N + c - 1) / c};
    }
    w.kb = w.box.tiles_w * w.box.tiles_h * w.box.tiles_n;
    if (g.K <= 64 && rsc > 64) {
      w.swap = true;
      M = rsc;
      Ng = g.K;
    }
    if (Ng <= 64) w.bn = 64;
  } else {
    w.kb = (g.N * g.Ho * g.Wo + BK - 1) / BK;
  }
  w.mt = (M + BM - 1) / BM;
  w.nt = (Ng + w.bn - 1) / w.bn;
  const int64_t tiles = (int64_t)w.mt * w.nt;
  // split-K count from a small cost model in units of one k-block (~0.7 us on a busy SM): waves of
  // persistent CTAs x (k-blocks per split + ~6 for pipeline fill and epilogue), plus the workspace
  // write + reduction read (8 B per dW element per split at ~6.5 TB/s ~ 4.5 MB per k-block time)
  const double ws_per_split = 8.0 * g.K * rsc / 4.5e6;
  double best = 1e300;
  w.splits = 1;
  for (int s = 1; s <= std::max(1, w.kb / 4); ++s) {
    const int64_t waves = (tiles * s + 147) / 148;
    const double cost = (double)waves * ((w.kb + s - 1) / s + 6) + (s > 1 ? s * ws_per_split : 0.0);
    if (cost < best - 1e-9) {
      best = cost;
      w.splits = s;
    }
  }
  if (const char* e = getenv("POOCH_WGRAD_SPLITS")) w.splits = std::max(1, std::min(atoi(e), w.kb));
  w.kb_per_split = (w.kb + w.splits - 1) / w.splits;
  w.splits = (w.kb + w.kb_per_split - 1) / w.kb_per_split;
  return w;
}

size_t conv_wgrad_ws_bytes(const ConvGeom& g) {
  WgradPlan w = wgrad_plan(g);
  return (w.splits > 1 || w.swap) ? (size_t)w.splits * g.K * g.R * g.S * g.C * sizeof(float) : 0;
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
                               size_t ws_bytes, cudaStream_t st) {
  WgradPlan w = wgrad_plan(g);
  GemmParams p = base_params(g);
  const int rsc = g.R * g.S * g.C;
  p.M = w.swap ? rsc : g.K;
  p.Ng = w.swap ? g.K : rsc;
  p.Kg = g.N * g.Ho * g.Wo;
  p.a = dy; p.b = x;
  p.kb_per_split = w.kb_per_split;
  bool use_ws = w.splits > 1 || w.swap;
  if (use_ws && ws_bytes < conv_wgrad_ws_bytes(g))
    return fail(POOCH_EUSAGE, "wgrad workspace too small: %zu < %zu", ws_bytes, conv_wgrad_ws_bytes(g));
  p.d = use_ws ? ws : dw;
  dim3 grid(w.mt, w.nt, w.splits);
  if (w.tma) {
    p.tw = w.box.tw; p.th = w.box.th; p.tn = w.box.tn;
    p.tiles_w = w.box.tiles_w; p.tiles_h = w.box.tiles_h; p.tiles_n = w.box.tiles_n;
    p.hout = g.Ho; p.wout = g.Wo;
    p.wg_a_is_x = w.swap ? 1 : 0;
    // chunks per box: the largest power of two <= 4 dividing the channel count in chunks (so a
    // box never straddles two taps) and no larger than the tile
    auto cb_of = [](int ch, int rows) {
      int cb = 4;
      while (cb > 1 && ((ch / 32) % cb != 0 || 32 * cb > rows)) cb >>= 1;
      return cb;
    };
    const int cb_dy = cb_of(g.K, w.swap ? w.bn : BM), cb_x = cb_of(g.C, w.swap ? BM : w.bn);
    p.wg_cba = w.swap ? cb_x : cb_dy;
    p.wg_cbb = w.swap ? cb_dy : cb_x;
    CUtensorMap tdy, tx;
    if (!map_nhwc_chunks(&tdy, dy, g.N, g.Ho, g.Wo, g.K, w.box.tw, w.box.th, w.box.tn, 1, cb_dy) ||
        !map_nhwc_chunks(&tx, x, g.N, g.H, g.W, g.C, w.box.tw, w.box.th, w.box.tn, g.stride, cb_x))
      return fail(POOCH_ECUDA, "cuTensorMapEncodeTiled failed (conv wgrad)");
    const CUtensorMap* ta = w.swap ? &tx : &tdy;
    const CUtensorMap* tb = w.swap ? &tdy : &tx;
    POOCH_CHECK((launch_bn<CONV_WGRAD, true>(w.bn, p, grid, st, g.prec, ta, tb)));
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
  if (!conv_shape_ok(g)) return fail(POOCH_EUSAGE, "unsupported conv shape");
  if ((stat_sum == nullptr) != (stat_sq == nullptr)) return fail(POOCH_EUSAGE, "stat_sum/stat_sq must pair");
  return launch_conv_fwd(g, x, w, y, stat_sum, stat_sq, nullptr, (cudaStream_t)stream);
}

extern "C" pooch_status pooch_op_conv_dgrad(const pooch_conv_desc* d, const float* dy, const float* wt, float* dx,
                                            int32_t accumulate, void* stream) {
  if (!d || !dy || !wt || !dx) return fail(POOCH_EUSAGE, "null argument");
  ConvGeom g = conv_geom(*d);
  if (!conv_shape_ok(g)) return fail(POOCH_EUSAGE, "unsupported conv shape");
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
  if (!conv_shape_ok(g)) return fail(POOCH_EUSAGE, "unsupported conv shape");
  return launch_conv_wgrad(g, x, dy, dw, ws, ws_bytes, (cudaStream_t)stream);
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

extern "C" int64_t pooch_op_conv_stat_tiles(const pooch_conv_desc* d) {
  if (!d) return 0;
  return conv_stat_tiles(conv_geom(*d));
}
