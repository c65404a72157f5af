// peer.cu -- the gradient allreduce over peer memory (Sec. 1 names
// data parallelism): the library's own collective, without NCCL.
//
// Every rank owns one cudaMalloc'd exchange buffer, exported with cudaIpcGetMemHandle and
// mapped by every other rank (cudaIpcOpenMemHandle: NVLink / NVSwitch peer memory between
// GPUs, or plain device memory when several processes share one GPU). Its layout:
//   [0, 32 KB)   arrival flags: slot s, rank p at word s * kMaxWorld + p (written by rank p)
//   [32, 64 KB)  this rank's epoch counter per slot (read / written only by this rank)
//   [64 KB, ..)  the stage: one float per gradient float (the gradient region's layout)
// One bucket [lo, hi) of the gradient region is exchanged as
//   copy grad[lo, hi) -> stage[lo, hi)                   (local, D2D)
//   barrier (slot 2k): every rank's stage holds its bucket
//   rank r sums elements [lo + r*n/W, lo + (r+1)*n/W) over the W stages in rank order
//     0, 1, ..., W-1 and stores the sum into all W stages (reduce-scatter and all-gather in one
//     pass: 1x the bucket read and 1x written per rank, over NVLink)
//   barrier (slot 2k+1): every chunk is summed everywhere
//   copy stage[lo, hi) -> grad[lo, hi)                   (local)
// Each element's sum is formed by exactly one rank in a fixed order, so every rank ends with
// the same bits, independent of W's ring / tree choices (NCCL's sum order varies with its
// algorithm). All of it is kernels and memcpys on the comm stream: it is captured into the
// step's CUDA graph with the rest of the step. The epoch of a barrier lives in device memory
// (the counter above), so replays of a captured graph advance it.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>

#include "common.h"
#include "ctx.h"

namespace pooch {

constexpr int kMaxWorld = 16;
constexpr size_t kFlagsOff = 0, kCountOff = 32 << 10, kStageOff = 64 << 10;
constexpr int kMaxSlots = (32 << 10) / (4 * kMaxWorld);  // 512

struct PeerArgs {
  char* base[kMaxWorld];  // exchange buffers of ranks 0..W-1 (own one included)
  int rank, world;
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One thread: advance this slot's epoch, announce it to every rank, wait until every rank has
// announced it. A rank that never arrives (a dead peer) traps after 120 s instead of hanging.
__global__ void peer_barrier_kernel(PeerArgs a, int slot) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  char* own = a.base[a.rank];
  uint32_t* cnt = reinterpret_cast<uint32_t*>(own + kCountOff) + slot;
  const uint32_t e = *cnt + 1;
  *cnt = e;
  __threadfence_system();
  for (int p = 0; p < a.world; ++p)
    st_release_sys(reinterpret_cast<uint32_t*>(a.base[p] + kFlagsOff) + slot * kMaxWorld + a.rank, e);
  const uint32_t* mine = reinterpret_cast<const uint32_t*>(own + kFlagsOff) + slot * kMaxWorld;
  const uint64_t t0 = globaltimer();
  for (int p = 0; p < a.world; ++p) {
    // epochs only grow, and a peer cannot pass this slot's next barrier before this rank
    // arrives at it, so ">= e" is exact
    while ((int32_t)(ld_acquire_sys(mine + p) - e) < 0) {
      if (globaltimer() - t0 > 120ull * 1000000000ull) __trap();
      __nanosleep(256);
    }
  }
  __threadfence_system();
}

// Elements [c0, c1) (float4 units from the stage start) of the bucket: sum over the W stages
// in rank order, store the sum into every stage.
__global__ void __launch_bounds__(256) peer_sum_kernel(PeerArgs a, size_t c0, size_t c1) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = c0 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < c1; i += stride) {
    float4 s = __ldcg(reinterpret_cast<const float4*>(a.base[0] + kStageOff) + i);
    for (int p = 1; p < a.world; ++p) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(a.base[p] + kStageOff) + i);
      s.x += v.x;
      s.y += v.y;
      s.z += v.z;
      s.w += v.w;
    }
    for (int p = 0; p < a.world; ++p) __stcg(reinterpret_cast<float4*>(a.base[p] + kStageOff) + i, s);
  }
  __threadfence_system();
}

static PeerArgs peer_args(const pooch_ctx* c) {
  PeerArgs a{};
  for (int p = 0; p < c->world; ++p) a.base[p] = static_cast<char*>(c->peer_base[p]);
  a.rank = c->rank;
  a.world = c->world;
  return a;
}

// Allreduce (sum) of src[0, n) (n = hi - lo floats, lo / hi multiples of 4) through the stage
// range [lo, hi); the result replaces src. `slot` selects the barrier pair (2 slot, 2 slot + 1).
pooch_status peer_allreduce(pooch_ctx* c, float* src, size_t lo, size_t hi, int slot, cudaStream_t st) {
  if (!c->peer_own || (int)c->peer_base.size() != c->world)
    return fail(POOCH_EUSAGE, "peer allreduce without pooch_set_peers");
  if (2 * slot + 1 >= kMaxSlots) return fail(POOCH_EUSAGE, "too many allreduce buckets (%d)", slot);
  if (lo % 4 || hi % 4 || hi > c->peer_floats) return fail(POOCH_EUSAGE, "bad allreduce range [%zu, %zu)", lo, hi);
  float* stage = reinterpret_cast<float*>(static_cast<char*>(c->peer_own) + kStageOff) + lo;
  const size_t n = hi - lo;
  const PeerArgs a = peer_args(c);
  POOCH_CUDA(cudaMemcpyAsync(stage, src, n * 4, cudaMemcpyDeviceToDevice, st));
  peer_barrier_kernel<<<1, 32, 0, st>>>(a, 2 * slot);
  POOCH_CUDA(cudaGetLastError());
  const size_t n4 = n / 4, lo4 = lo / 4;
  const size_t c0 = lo4 + n4 * c->rank / c->world, c1 = lo4 + n4 * (c->rank + 1) / c->world;
  if (c1 > c0) {
    const int blocks = (int)std::min<size_t>((size_t)c->sm_count * 4, (c1 - c0 + 255) / 256);
    peer_sum_kernel<<<blocks, 256, 0, st>>>(a, c0, c1);
    POOCH_CUDA(cudaGetLastError());
  }
  peer_barrier_kernel<<<1, 32, 0, st>>>(a, 2 * slot + 1);
  POOCH_CUDA(cudaGetLastError());
  POOCH_CUDA(cudaMemcpyAsync(src, stage, n * 4, cudaMemcpyDeviceToDevice, st));
  return POOCH_OK;
}

int peer_max_slots() { return kMaxSlots / 2; }

static pooch_status ctx_fail(pooch_ctx* c, pooch_status st) {
  if (c) c->err = tls_error();
  return st;
}

void peer_close(pooch_ctx* c) {
  for (int p = 0; p < (int)c->peer_base.size(); ++p)
    if (c->peer_base[p] && c->peer_base[p] != c->peer_own) cudaIpcCloseMemHandle(c->peer_base[p]);
  c->peer_base.clear();
  if (c->peer_own) cudaFree(c->peer_own);
  c->peer_own = nullptr;
  c->peer_floats = 0;
}

}  // namespace pooch

using namespace pooch;

extern "C" pooch_status pooch_peer_open(pooch_ctx* c, int32_t rank, int32_t world, void* handle64,
                                        uint64_t* bytes) {
  if (!c || !handle64) return fail(POOCH_EUSAGE, "null argument");
  if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world)
    return ctx_fail(c, fail(POOCH_EUSAGE, "bad rank %d / world %d (world <= %d)", rank, world, kMaxWorld));
  if (c->nccl) return ctx_fail(c, fail(POOCH_EUSAGE, "context already has an NCCL communicator"));
  POOCH_CUDA(cudaSetDevice(c->device));
  peer_close(c);
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, c->device);
  const size_t floats = ((size_t)c->param_floats + 3) / 4 * 4;
  const size_t total = kStageOff + floats * 4;
  void* p = nullptr;
  if (cudaMalloc(&p, total) != cudaSuccess) {
    cudaGetLastError();
    return ctx_fail(c, fail(POOCH_ECUDA, "cudaMalloc of the %zu-byte peer exchange buffer failed", total));
  }
  POOCH_CUDA(cudaMemset(p, 0, kStageOff));
  POOCH_CUDA(cudaDeviceSynchronize());
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, p) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(p);
    return ctx_fail(c, fail(POOCH_ECUDA, "cudaIpcGetMemHandle failed"));
  }
  std::memcpy(handle64, &h, sizeof(h));
  c->peer_own = p;
  c->peer_floats = floats;
  c->rank = rank;
  c->world = world;
  if (bytes) *bytes = total;
  return POOCH_OK;
}

extern "C" pooch_status pooch_set_peers(pooch_ctx* c, const void* handles) {
  if (!c || !handles) return fail(POOCH_EUSAGE, "null argument");
  if (!c->peer_own) return ctx_fail(c, fail(POOCH_EUSAGE, "pooch_set_peers before pooch_peer_open"));
  POOCH_CUDA(cudaSetDevice(c->device));
  for (int p = 0; p < (int)c->peer_base.size(); ++p)
    if (c->peer_base[p] && c->peer_base[p] != c->peer_own) cudaIpcCloseMemHandle(c->peer_base[p]);
  c->peer_base.assign(c->world, nullptr);
  for (int p = 0; p < c->world; ++p) {
    if (p == c->rank) {
      c->peer_base[p] = c->peer_own;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + 64 * p, sizeof(h));
    void* q = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaGetLastError();
      // leave no half-mapped peer set behind (has_comm() would route the step through it)
      for (int r = 0; r < p; ++r)
        if (c->peer_base[r] && c->peer_base[r] != c->peer_own) cudaIpcCloseMemHandle(c->peer_base[r]);
      c->peer_base.clear();
      return ctx_fail(c, fail(POOCH_ECUDA, "cudaIpcOpenMemHandle (rank %d): %s", p, cudaGetErrorString(e)));
    }
    c->peer_base[p] = q;
  }
  c->have_plan = false;
  peer_setup_buckets(c);
  if ((int)c->buckets.size() + 1 > peer_max_slots()) {
    for (int r = 0; r < c->world; ++r)
      if (c->peer_base[r] && c->peer_base[r] != c->peer_own) cudaIpcCloseMemHandle(c->peer_base[r]);
    c->peer_base.clear();
    return ctx_fail(c, fail(POOCH_EUSAGE, "%zu allreduce buckets exceed the %d barrier slots", c->buckets.size(),
                            peer_max_slots() - 1));
  }
  return POOCH_OK;
}
