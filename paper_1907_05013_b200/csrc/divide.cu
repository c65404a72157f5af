// divide.cu -- intra-layer division (ooc_cuDNN style; "Ito's
// ooc_cuDNN library performs data-swapping after dividing each computation and data ...
// ooc_cuDNN supports NNs where memory consumption of a single layer exceeds the GPU memory
// capacity. By integrating PoocH and ooc_cuDNN, PoocH will support NNs of wider ranges").
//
// A layer whose maps do not fit the device runs on HOST-resident tensors (pinned) in chunks of
// depth rows (3D, batch 1 -- the paper's 3D-image case): each chunk's input slab (with
// its halo rows for a convolution) is copied in, the same kernels as the undivided layer run on
// it, and the chunk's output is copied out, on three streams with two buffer sets so the copies
// of chunk j+1 / j-1 overlap the kernels of chunk j. Layers:
//   conv3d fwd (+ the BN statistics of its output, accumulated over chunks in fp64)
//   BN-ReLU apply; BN-ReLU backward (pass 1: per-channel sums over all chunks; pass 2: apply)
//   conv3d dgrad (each chunk of input rows gathers the dy rows it needs); conv3d wgrad (chunk
//   partials summed in chunk order).
// The sub-convolution of a slab pads H and W only (ConvGeom::pad_d = 0): its depth halo is real
// rows or zero rows at the volume's faces, so every output element is computed by the same
// kernel over the same taps as in the undivided layer (conv fwd / dgrad results equal the
// undivided kernels' bit for bit; the statistics and wgrad partial sums regroup).
#include <cuda_runtime.h>

#include <algorithm>

#include "common.h"
#include "conv.h"
#include "eltwise.h"

namespace pooch {

namespace {

struct Engine {
  cudaStream_t comp, h2d, d2h;
  cudaEvent_t loaded[2] = {nullptr, nullptr}, computed[2] = {nullptr, nullptr}, freed[2] = {nullptr, nullptr};
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  bool used[2] = {false, false};
  pooch_status init(void* const* streams) {
    comp = (cudaStream_t)streams[0];
    h2d = (cudaStream_t)streams[1];
    d2h = (cudaStream_t)streams[2];
    for (int b = 0; b < 2; ++b) {
      POOCH_CUDA(cudaEventCreateWithFlags(&loaded[b], cudaEventDisableTiming));
      POOCH_CUDA(cudaEventCreateWithFlags(&computed[b], cudaEventDisableTiming));
      POOCH_CUDA(cudaEventCreateWithFlags(&freed[b], cudaEventDisableTiming));
    }
    POOCH_CUDA(cudaEventCreate(&t0));
    POOCH_CUDA(cudaEventCreate(&t1));
    POOCH_CUDA(cudaEventRecord(t0, h2d));
    POOCH_CUDA(cudaStreamWaitEvent(comp, t0, 0));
    POOCH_CUDA(cudaStreamWaitEvent(d2h, t0, 0));
    return POOCH_OK;
  }
  // before the loads of a chunk into buffer set b: its previous user has finished
  pooch_status begin_load(int b) {
    if (used[b]) POOCH_CUDA(cudaStreamWaitEvent(h2d, freed[b], 0));
    used[b] = true;
    return POOCH_OK;
  }
  pooch_status loads_done(int b) {
    POOCH_CUDA(cudaEventRecord(loaded[b], h2d));
    POOCH_CUDA(cudaStreamWaitEvent(comp, loaded[b], 0));
    return POOCH_OK;
  }
  // after the kernels of buffer set b: the stores wait for them (store = true), or the set is
  // free as soon as they are done
  pooch_status kernels_done(int b, bool store) {
    POOCH_CUDA(cudaEventRecord(computed[b], comp));
    if (store) {
      POOCH_CUDA(cudaStreamWaitEvent(d2h, computed[b], 0));
    } else {
      POOCH_CUDA(cudaEventRecord(freed[b], comp));
    }
    return POOCH_OK;
  }
  pooch_status stores_done(int b) {
    POOCH_CUDA(cudaEventRecord(freed[b], d2h));
    return POOCH_OK;
  }
  pooch_status finish(double* ms) {
    POOCH_CUDA(cudaEventRecord(computed[0], d2h));
    POOCH_CUDA(cudaStreamWaitEvent(comp, computed[0], 0));
    POOCH_CUDA(cudaEventRecord(computed[1], h2d));
    POOCH_CUDA(cudaStreamWaitEvent(comp, computed[1], 0));
    POOCH_CUDA(cudaEventRecord(t1, comp));
    POOCH_CUDA(cudaEventSynchronize(t1));
    float f = 0.f;
    POOCH_CUDA(cudaEventElapsedTime(&f, t0, t1));
    if (ms) *ms = f;
    return POOCH_OK;
  }
  ~Engine() {
    for (int b = 0; b < 2; ++b) {
      if (loaded[b]) cudaEventDestroy(loaded[b]);
      if (computed[b]) cudaEventDestroy(computed[b]);
      if (freed[b]) cudaEventDestroy(freed[b]);
    }
    if (t0) cudaEventDestroy(t0);
    if (t1) cudaEventDestroy(t1);
  }
};

// bump allocator over the caller's workspace (256-byte aligned pieces)
struct Carve {
  char* base;
  size_t cap, used = 0;
  void* take(size_t bytes) {
    void* p = base + used;
    used = (used + bytes + 255) / 256 * 256;
    return p;
  }
  static size_t need(std::initializer_list<size_t> parts) {
    size_t t = 0;
    for (size_t p : parts) t += (p + 255) / 256 * 256;
    return t;
  }
};

// rows [lo, lo + n) of a host volume of D rows (row_floats each) into dev; rows outside [0, D)
// are zero-filled
pooch_status load_rows(float* dev, const float* host, int64_t lo, int64_t n, int64_t D, size_t row_floats,
                       cudaStream_t st, uint64_t* bytes) {
  const int64_t a = std::max<int64_t>(lo, 0), b = std::min<int64_t>(lo + n, D);
  if (a > lo) POOCH_CUDA(cudaMemsetAsync(dev, 0, (size_t)(a - lo) * row_floats * 4, st));
  if (b > a) {
    POOCH_CUDA(cudaMemcpyAsync(dev + (size_t)(a - lo) * row_floats, host + (size_t)a * row_floats,
                               (size_t)(b - a) * row_floats * 4, cudaMemcpyHostToDevice, st));
    *bytes += (uint64_t)(b - a) * row_floats * 4;
  }
  const int64_t end = lo + n;
  if (end > std::max(b, lo)) {
    const int64_t z0 = std::max(b, lo);
    POOCH_CUDA(cudaMemsetAsync(dev + (size_t)(z0 - lo) * row_floats, 0, (size_t)(end - z0) * row_floats * 4, st));
  }
  return POOCH_OK;
}

bool div_conv_ok(const ConvGeom& g) {
  return g.is3d() && g.groups <= 1 && g.C1 == 0 && conv_shape_ok(g) && g.sd() == g.stride && g.R >= g.sd();
}

// the sub-convolution of output depth rows [o0, o0 + r): a slab of (r - 1) * s + k input rows
// starting at o0 * s - pad, padded in H / W only
ConvGeom slab_geom(const ConvGeom& g, int r) {
  ConvGeom q = g;
  q.D = (r - 1) * g.sd() + g.R;
  q.Do = r;
  q.pad_d = 0;
  return q;
}

__global__ void add_kernel(float4* __restrict__ acc, const float4* __restrict__ v, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = acc[i];
    const float4 b = v[i];
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    acc[i] = a;
  }
}

pooch_status add_into(float* acc, const float* v, int64_t n, cudaStream_t st) {
  const int64_t n4 = n / 4;
  count_launch();
  add_kernel<<<(int)std::min<int64_t>((n4 + 255) / 256, 148 * 8), 256, 0, st>>>(
      reinterpret_cast<float4*>(acc), reinterpret_cast<const float4*>(v), n4);
  POOCH_CUDA(cudaGetLastError());
  return POOCH_OK;
}

void fill_info(pooch_div_info* info, int chunks, int rows, double ms, uint64_t in, uint64_t out) {
  if (!info) return;
  info->chunks = chunks;
  info->rows_per_chunk = rows;
  info->ms = ms;
  info->h2d_bytes = in;
  info->d2h_bytes = out;
}

}  // namespace

}  // namespace pooch

using namespace pooch;

// ------------------------------------------------------------------------------ conv fwd
static size_t fwd_need(const ConvGeom& g, int r) {
  const ConvGeom q = slab_geom(g, r);
  const size_t in = (size_t)q.D * g.H * g.W * g.C * 4, out = (size_t)r * g.Ho * g.Wo * g.K * 4;
  const size_t tiles = (size_t)std::max(conv_stat_tiles(q), conv_stat_tiles(slab_geom(g, (g.Do - 1) % r + 1))) * g.K * 4;
  return Carve::need({in, in, out, out, tiles, tiles, (size_t)2 * g.K * 8});
}

extern "C" pooch_status pooch_div_conv3d_fwd(const pooch_conv_desc* d, const float* x_host, const float* w_dev,
                                             float* y_host, const float* gamma, const float* beta, float* stats,
                                             void* ws, size_t ws_bytes, void* const* streams, pooch_div_info* info) {
  if (!d || !x_host || !w_dev || !y_host || !ws || !streams) return fail(POOCH_EUSAGE, "null argument");
  const ConvGeom g = conv_geom(*d);
  if (!div_conv_ok(g)) return fail(POOCH_EUSAGE, "divided conv: 3D dense single-source conv, uniform stride");
  if (stats && (!gamma || !beta)) return fail(POOCH_EUSAGE, "divided conv: BN statistics need gamma / beta");
  int r = g.Do;
  while (r > 0 && fwd_need(g, r) > ws_bytes) --r;
  if (r == 0) return fail(POOCH_EINFEASIBLE, "divided conv: one output row needs %zu B > workspace %zu B",
                          fwd_need(g, 1), ws_bytes);
  const ConvGeom q = slab_geom(g, r);
  Carve cv{static_cast<char*>(ws), ws_bytes};
  const size_t in_f = (size_t)q.D * g.H * g.W * g.C, out_f = (size_t)r * g.Ho * g.Wo * g.K;
  float* xin[2] = {(float*)cv.take(in_f * 4), (float*)cv.take(in_f * 4)};
  float* yout[2] = {(float*)cv.take(out_f * 4), (float*)cv.take(out_f * 4)};
  const int tiles_max = std::max(conv_stat_tiles(q), conv_stat_tiles(slab_geom(g, (g.Do - 1) % r + 1)));
  float* ts = (float*)cv.take((size_t)tiles_max * g.K * 4);
  float* tq = (float*)cv.take((size_t)tiles_max * g.K * 4);
  double* acc = (double*)cv.take((size_t)2 * g.K * 8);
  Engine e;
  POOCH_CHECK(e.init(streams));
  if (stats) POOCH_CUDA(cudaMemsetAsync(acc, 0, (size_t)2 * g.K * 8, e.comp));
  const size_t in_row = (size_t)g.H * g.W * g.C, out_row = (size_t)g.Ho * g.Wo * g.K;
  uint64_t bin = 0, bout = 0;
  int j = 0;
  for (int o0 = 0; o0 < g.Do; o0 += r, ++j) {
    const int b = j & 1, n = std::min(r, g.Do - o0);
    const ConvGeom qj = slab_geom(g, n);
    POOCH_CHECK(e.begin_load(b));
    POOCH_CHECK(load_rows(xin[b], x_host, (int64_t)o0 * g.sd() - g.pd(), qj.D, g.D, in_row, e.h2d, &bin));
    POOCH_CHECK(e.loads_done(b));
    POOCH_CHECK(launch_conv_fwd(qj, xin[b], w_dev, yout[b], stats ? ts : nullptr, stats ? tq : nullptr, nullptr,
                                e.comp));
    if (stats) POOCH_CHECK(bn_acc_tiles(ts, tq, conv_stat_tiles(qj), g.K, acc, e.comp));
    POOCH_CHECK(e.kernels_done(b, true));
    POOCH_CUDA(cudaMemcpyAsync(y_host + (size_t)o0 * out_row, yout[b], (size_t)n * out_row * 4,
                               cudaMemcpyDeviceToHost, e.d2h));
    bout += (uint64_t)n * out_row * 4;
    POOCH_CHECK(e.stores_done(b));
  }
  if (stats)
    POOCH_CHECK(bn_finalize_sums(acc, g.K, (int64_t)g.Do * g.Ho * g.Wo, gamma, beta, stats, stats + g.K,
                                 stats + 2 * g.K, stats + 3 * g.K, e.comp));
  double ms = 0;
  POOCH_CHECK(e.finish(&ms));
  fill_info(info, j, r, ms, bin, bout);
  return POOCH_OK;
}

// ------------------------------------------------------------------------------ BN-ReLU fwd / bwd
extern "C" pooch_status pooch_div_bn_relu_fwd(const float* c_host, const float* stats, float* y_host, int64_t rows,
                                              int64_t row_floats, int32_t C, void* ws, size_t ws_bytes,
                                              void* const* streams, pooch_div_info* info) {
  if (!c_host || !stats || !y_host || !ws || !streams || rows <= 0 || C <= 0 || C % 4 || row_floats % C)
    return fail(POOCH_EUSAGE, "divided BN-ReLU: bad arguments");
  int64_t r = std::min<int64_t>(rows, (int64_t)(ws_bytes / (4 * (size_t)row_floats * 4 + 1024)));
  while (r > 0 && Carve::need({(size_t)r * row_floats * 4, (size_t)r * row_floats * 4, (size_t)r * row_floats * 4,
                               (size_t)r * row_floats * 4}) > ws_bytes)
    --r;
  if (r <= 0) return fail(POOCH_EINFEASIBLE, "divided BN-ReLU: one row does not fit the workspace");
  Carve cv{static_cast<char*>(ws), ws_bytes};
  float* in[2] = {(float*)cv.take((size_t)r * row_floats * 4), (float*)cv.take((size_t)r * row_floats * 4)};
  float* out[2] = {(float*)cv.take((size_t)r * row_floats * 4), (float*)cv.take((size_t)r * row_floats * 4)};
  Engine e;
  POOCH_CHECK(e.init(streams));
  uint64_t bin = 0, bout = 0;
  int j = 0;
  for (int64_t z = 0; z < rows; z += r, ++j) {
    const int b = j & 1;
    const int64_t n = std::min(r, rows - z);
    POOCH_CHECK(e.begin_load(b));
    POOCH_CHECK(load_rows(in[b], c_host, z, n, rows, row_floats, e.h2d, &bin));
    POOCH_CHECK(e.loads_done(b));
    POOCH_CHECK(bn_apply_relu(in[b], stats + 2 * C, stats + 3 * C, nullptr, nullptr, nullptr, 0, out[b],
                              n * row_floats / C, C, e.comp));
    POOCH_CHECK(e.kernels_done(b, true));
    POOCH_CUDA(cudaMemcpyAsync(y_host + (size_t)z * row_floats, out[b], (size_t)n * row_floats * 4,
                               cudaMemcpyDeviceToHost, e.d2h));
    bout += (uint64_t)n * row_floats * 4;
    POOCH_CHECK(e.stores_done(b));
  }
  double ms = 0;
  POOCH_CHECK(e.finish(&ms));
  fill_info(info, j, (int)r, ms, bin, bout);
  return POOCH_OK;
}

extern "C" pooch_status pooch_div_bn_relu_bwd(const float* c_host, const float* gy_host, const float* stats,
                                              const float* gamma, float* dgamma, float* dbeta, float* gx_host,
                                              int64_t rows, int64_t row_floats, int32_t C, void* ws, size_t ws_bytes,
                                              void* const* streams, pooch_div_info* info) {
  if (!c_host || !gy_host || !stats || !gamma || !dgamma || !dbeta || !gx_host || !ws || !streams || rows <= 0 ||
      C <= 0 || C % 4 || C > 2048 || row_floats % C)
    return fail(POOCH_EUSAGE, "divided BN-ReLU backward: bad arguments");
  const int64_t pix_row = row_floats / C;
  auto need = [&](int64_t r) {
    const size_t s = (size_t)r * row_floats * 4;
    return Carve::need({s, s, s, s, s, s, bn_relu_bwd_partial_ws_bytes(r * pix_row, C), (size_t)2 * C * 8,
                        (size_t)3 * C * 4});
  };
  int64_t r = std::min<int64_t>(rows, (int64_t)(ws_bytes / (6 * (size_t)row_floats * 4)));
  while (r > 0 && need(r) > ws_bytes) --r;
  if (r <= 0) return fail(POOCH_EINFEASIBLE, "divided BN-ReLU backward: one row does not fit the workspace");
  Carve cv{static_cast<char*>(ws), ws_bytes};
  const size_t cf = (size_t)r * row_floats;
  float* cin[2] = {(float*)cv.take(cf * 4), (float*)cv.take(cf * 4)};
  float* gin[2] = {(float*)cv.take(cf * 4), (float*)cv.take(cf * 4)};
  float* gout[2] = {(float*)cv.take(cf * 4), (float*)cv.take(cf * 4)};
  float* bws = (float*)cv.take(bn_relu_bwd_partial_ws_bytes(r * pix_row, C));
  double* acc = (double*)cv.take((size_t)2 * C * 8);
  float* coef = (float*)cv.take((size_t)3 * C * 4);
  BnBwdArgs a{};
  a.sa = stats + 2 * C; a.ta = stats + 3 * C; a.mean_a = stats; a.invstd_a = stats + C;
  a.gamma_a = gamma; a.dgamma_a = dgamma; a.dbeta_a = dbeta;
  a.mode = 0;
  a.C = C;
  Engine e;
  POOCH_CHECK(e.init(streams));
  POOCH_CUDA(cudaMemsetAsync(acc, 0, (size_t)2 * C * 8, e.comp));
  uint64_t bin = 0, bout = 0;
  int j = 0;
  // pass 1: per-channel sum dz, sum dz * xhat over every chunk (fp64, chunk order)
  for (int64_t z = 0; z < rows; z += r, ++j) {
    const int b = j & 1;
    const int64_t n = std::min(r, rows - z);
    POOCH_CHECK(e.begin_load(b));
    POOCH_CHECK(load_rows(cin[b], c_host, z, n, rows, row_floats, e.h2d, &bin));
    POOCH_CHECK(load_rows(gin[b], gy_host, z, n, rows, row_floats, e.h2d, &bin));
    POOCH_CHECK(e.loads_done(b));
    BnBwdArgs q = a;
    q.a = cin[b]; q.gy = gin[b]; q.rows = n * row_floats / C;
    POOCH_CHECK(bn_relu_bwd_partial(q, bws, acc, e.comp));
    POOCH_CHECK(e.kernels_done(b, false));
  }
  POOCH_CHECK(bn_relu_bwd_finalize(a, acc, rows * row_floats / C, coef, e.comp));
  // pass 2: gx = gamma invstd (dz - sum dz / M - xhat sum dz xhat / M), chunk by chunk
  for (int64_t z = 0; z < rows; z += r, ++j) {
    const int b = j & 1;
    const int64_t n = std::min(r, rows - z);
    POOCH_CHECK(e.begin_load(b));
    POOCH_CHECK(load_rows(cin[b], c_host, z, n, rows, row_floats, e.h2d, &bin));
    POOCH_CHECK(load_rows(gin[b], gy_host, z, n, rows, row_floats, e.h2d, &bin));
    POOCH_CHECK(e.loads_done(b));
    BnBwdArgs q = a;
    q.a = cin[b]; q.gy = gin[b]; q.ga = gout[b]; q.rows = n * row_floats / C;
    POOCH_CHECK(bn_relu_bwd_apply(q, coef, e.comp));
    POOCH_CHECK(e.kernels_done(b, true));
    POOCH_CUDA(cudaMemcpyAsync(gx_host + (size_t)z * row_floats, gout[b], (size_t)n * row_floats * 4,
                               cudaMemcpyDeviceToHost, e.d2h));
    bout += (uint64_t)n * row_floats * 4;
    POOCH_CHECK(e.stores_done(b));
  }
  double ms = 0;
  POOCH_CHECK(e.finish(&ms));
  fill_info(info, j, (int)r, ms, bin, bout);
  return POOCH_OK;
}

// ------------------------------------------------------------------------------ conv dgrad / wgrad
// dgrad, input rows [a, a + ri): the dy rows [o0, o1) that reach them and the virtual input slab
// [o0 * s - p, (o1 - 1) * s - p + k) those rows cover (it contains [a, a + ri))
static void dgrad_span(const ConvGeom& g, int a, int ri, int& o0, int& o1) {
  const int s = g.sd(), p = g.pd(), k = g.R;
  const int lo = a + p - k + 1;                 // first output row reaching input row a
  o0 = std::max(0, lo <= 0 ? 0 : (lo + s - 1) / s);
  o1 = std::min(g.Do, (a + ri - 1 + p) / s + 1);
}

// the largest dy-row and dx-row counts any chunk of ri input rows needs (exact, over all chunks)
static void dgrad_rows(const ConvGeom& g, int ri, int& dy_rows, int& dx_rows) {
  dy_rows = 1;
  dx_rows = ri;
  for (int a = 0; a < g.D; a += ri) {
    const int n = std::min(ri, g.D - a);
    int o0, o1;
    dgrad_span(g, a, n, o0, o1);
    if (o1 <= o0) continue;
    const int slab0 = o0 * g.sd() - g.pd(), dp = (o1 - o0 - 1) * g.sd() + g.R;
    dy_rows = std::max(dy_rows, o1 - o0);
    dx_rows = std::max(dx_rows, std::max(dp, (a - slab0) + n));
  }
}

static size_t dgrad_need(const ConvGeom& g, int ri) {
  int dyr, dxr;
  dgrad_rows(g, ri, dyr, dxr);
  const size_t dy = (size_t)dyr * g.Ho * g.Wo * g.K * 4, dx = (size_t)dxr * g.H * g.W * g.C * 4;
  return Carve::need({dy, dy, dx, dx});
}

extern "C" pooch_status pooch_div_conv3d_dgrad(const pooch_conv_desc* d, const float* gy_host, const float* wt_dev,
                                               float* gx_host, void* ws, size_t ws_bytes, void* const* streams,
                                               pooch_div_info* info) {
  if (!d || !gy_host || !wt_dev || !gx_host || !ws || !streams) return fail(POOCH_EUSAGE, "null argument");
  const ConvGeom g = conv_geom(*d);
  if (!div_conv_ok(g)) return fail(POOCH_EUSAGE, "divided conv: 3D dense single-source conv, uniform stride");
  int ri = g.D;
  while (ri > 0 && dgrad_need(g, ri) > ws_bytes) --ri;
  if (ri == 0) return fail(POOCH_EINFEASIBLE, "divided dgrad: one input row does not fit the workspace");
  int o0, o1, dyr, dxr;
  dgrad_rows(g, ri, dyr, dxr);
  const size_t dy_f = (size_t)dyr * g.Ho * g.Wo * g.K;
  const size_t dx_f = (size_t)dxr * g.H * g.W * g.C;
  Carve cv{static_cast<char*>(ws), ws_bytes};
  float* dyb[2] = {(float*)cv.take(dy_f * 4), (float*)cv.take(dy_f * 4)};
  float* dxb[2] = {(float*)cv.take(dx_f * 4), (float*)cv.take(dx_f * 4)};
  Engine e;
  POOCH_CHECK(e.init(streams));
  const size_t in_row = (size_t)g.H * g.W * g.C, out_row = (size_t)g.Ho * g.Wo * g.K;
  uint64_t bin = 0, bout = 0;
  int j = 0;
  for (int a = 0; a < g.D; a += ri, ++j) {
    const int b = j & 1, n = std::min(ri, g.D - a);
    dgrad_span(g, a, n, o0, o1);
    const int slab0 = o0 * g.sd() - g.pd();
    POOCH_CHECK(e.begin_load(b));
    if (o1 > o0) {
      POOCH_CHECK(load_rows(dyb[b], gy_host, o0, o1 - o0, g.Do, out_row, e.h2d, &bin));
      POOCH_CHECK(e.loads_done(b));
      const ConvGeom qj = slab_geom(g, o1 - o0);
      POOCH_CHECK(launch_conv_dgrad(qj, dyb[b], wt_dev, dxb[b], false, e.comp));
      // input rows past the slab (beyond the last output's reach) have zero gradient
      const int tail = (a - slab0) + n - qj.D;
      if (tail > 0) POOCH_CUDA(cudaMemsetAsync(dxb[b] + (size_t)qj.D * in_row, 0, (size_t)tail * in_row * 4, e.comp));
    } else {  // no output row reaches these input rows: their gradient is zero
      POOCH_CHECK(e.loads_done(b));
      POOCH_CUDA(cudaMemsetAsync(dxb[b], 0, (size_t)n * in_row * 4, e.comp));
    }
    POOCH_CHECK(e.kernels_done(b, true));
    const size_t off = o1 > o0 ? (size_t)(a - slab0) * in_row : 0;
    POOCH_CUDA(cudaMemcpyAsync(gx_host + (size_t)a * in_row, dxb[b] + off, (size_t)n * in_row * 4,
                               cudaMemcpyDeviceToHost, e.d2h));
    bout += (uint64_t)n * in_row * 4;
    POOCH_CHECK(e.stores_done(b));
  }
  double ms = 0;
  POOCH_CHECK(e.finish(&ms));
  fill_info(info, j, ri, ms, bin, bout);
  return POOCH_OK;
}

static size_t wgrad_need(const ConvGeom& g, int r) {
  const ConvGeom q = slab_geom(g, r);
  const size_t x = (size_t)q.D * g.H * g.W * g.C * 4, dy = (size_t)r * g.Ho * g.Wo * g.K * 4;
  const size_t dw = (size_t)g.K * g.T() * g.R * g.S * g.C * 4;
  return Carve::need({x, x, dy, dy, dw, std::max(conv_wgrad_ws_bytes(q), conv_wgrad_ws_bytes(slab_geom(g, (g.Do - 1) % r + 1)))});
}

extern "C" pooch_status pooch_div_conv3d_wgrad(const pooch_conv_desc* d, const float* x_host, const float* gy_host,
                                               float* dw_dev, void* ws, size_t ws_bytes, void* const* streams,
                                               pooch_div_info* info) {
  if (!d || !x_host || !gy_host || !dw_dev || !ws || !streams) return fail(POOCH_EUSAGE, "null argument");
  const ConvGeom g = conv_geom(*d);
  if (!div_conv_ok(g)) return fail(POOCH_EUSAGE, "divided conv: 3D dense single-source conv, uniform stride");
  int r = g.Do;
  while (r > 0 && wgrad_need(g, r) > ws_bytes) --r;
  if (r == 0) return fail(POOCH_EINFEASIBLE, "divided wgrad: one output row does not fit the workspace");
  const ConvGeom q = slab_geom(g, r);
  Carve cv{static_cast<char*>(ws), ws_bytes};
  const size_t x_f = (size_t)q.D * g.H * g.W * g.C, dy_f = (size_t)r * g.Ho * g.Wo * g.K;
  const int64_t dw_n = (int64_t)g.K * g.T() * g.R * g.S * g.C;
  float* xb[2] = {(float*)cv.take(x_f * 4), (float*)cv.take(x_f * 4)};
  float* dyb[2] = {(float*)cv.take(dy_f * 4), (float*)cv.take(dy_f * 4)};
  float* part = (float*)cv.take((size_t)dw_n * 4);
  // the workspace of the full chunk and of the ragged last one
  const size_t wws_bytes = std::max(conv_wgrad_ws_bytes(q), conv_wgrad_ws_bytes(slab_geom(g, (g.Do - 1) % r + 1)));
  float* wws = (float*)cv.take(wws_bytes);
  Engine e;
  POOCH_CHECK(e.init(streams));
  const size_t in_row = (size_t)g.H * g.W * g.C, out_row = (size_t)g.Ho * g.Wo * g.K;
  uint64_t bin = 0;
  int j = 0;
  for (int o0 = 0; o0 < g.Do; o0 += r, ++j) {
    const int b = j & 1, n = std::min(r, g.Do - o0);
    const ConvGeom qj = slab_geom(g, n);
    POOCH_CHECK(e.begin_load(b));
    POOCH_CHECK(load_rows(xb[b], x_host, (int64_t)o0 * g.sd() - g.pd(), qj.D, g.D, in_row, e.h2d, &bin));
    POOCH_CHECK(load_rows(dyb[b], gy_host, o0, n, g.Do, out_row, e.h2d, &bin));
    POOCH_CHECK(e.loads_done(b));
    // chunk 0 writes dw; later chunks add their partial (chunk order)
    POOCH_CHECK(launch_conv_wgrad(qj, xb[b], dyb[b], j == 0 ? dw_dev : part, wws, wws_bytes, e.comp));
    if (j > 0) POOCH_CHECK(add_into(dw_dev, part, dw_n, e.comp));
    POOCH_CHECK(e.kernels_done(b, false));
  }
  double ms = 0;
  POOCH_CHECK(e.finish(&ms));
  fill_info(info, j, r, ms, bin, 0);
  return POOCH_OK;
}
