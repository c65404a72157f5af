// mmaprobe.cu -- raw tcgen05.mma kind::tf32 issue throughput on this B200 by tile width N and
// by where A comes from (shared memory descriptor vs TMEM): one CTA per SM, one thread issues
// `iters` back-to-back M=128 x N x K=8 MMAs into one accumulator (operands are zeroed smem /
// TMEM; only the timing matters). Answers whether BN = 64 tiles can reach the per-flop rate of
// BN = 128 / 256 at all.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -shared -Xcompiler -fPIC -o mmaprobe.so mmaprobe.cu
#include <cuda_runtime.h>

#include <cstdint>

#include "../../paper_1907_05013_b200/csrc/ptx.cuh"

using namespace pooch::ptx;

template <int N, bool TS>
__global__ void probe(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x;
  for (int i = tid; i < (128 + 256) * 32; i += blockDim.x) ((float*)smem)[i] = 0.f;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (tid < 32) tmem_alloc(&tmem_base, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t sa = smem_u32(smem), sb = sa + 128 * 128;
    const uint32_t idesc = idesc_tf32(128, N, false, false);
    const uint64_t ad = smem_desc(sa, 16, 1024, 2), bd = smem_desc(sb, 16, 1024, 2);
    const uint32_t acc = tmem_base, ta = tmem_base + 256;
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (TS) mma_tf32_ts(acc, ta + 8 * (i & 3), bd, idesc, 1u);
      else mma_tf32(acc, ad + 2 * (i & 3), bd, idesc, 1u);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

// The igemm 3xTF32 AT k-block pattern: per k-step kk (of 4) lo*B, hi*Bs, hi*B with A hi / lo in
// one of 6 TMEM stages (64 columns each) and B / Bs two SW128 tiles (k-step = +32 B), plus one
// tcgen05.commit per k-block (12 MMAs), as the MMA warp of igemm_kernel issues them.
template <int N, int V = 0>
__global__ void probe_kblock(int kblocks, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar, bar2, bar0, rot[6];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x;
  for (int i = tid; i < 2 * 256 * 32; i += blockDim.x) ((float*)smem)[i] = 0.f;
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    mbar_init(&bar0, 1);
    mbar_arrive(&bar0);
    for (int i = 0; i < 6; ++i) mbar_init(&rot[i], 1);
    fence_mbar_init();
  }
  if (tid < 32) tmem_alloc(&tmem_base, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t sb = smem_u32(smem), sbs = sb + N * 128;
    const uint32_t idesc = idesc_tf32(128, N, false, false);
    const uint32_t acc = tmem_base, a0 = tmem_base + 2 * N;
    unsigned long long t0 = clock64();
    for (int k = 0; k < kblocks; ++k) {
      if (V & 1) mbar_wait(&bar0, 0);  // V bit 0: a (satisfied) try_wait per k-block
      if (V & 8) {                     // V bit 3: a (satisfied) test_wait per k-block
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(smem_u32(&bar0)), "r"(0u) : "memory");
      }
      if (V & 16) {                    // V bit 4: the barrier word read with a plain ld.shared
        uint64_t w;
        asm volatile("ld.shared.b64 %0, [%1];" : "=l"(w) : "r"(smem_u32(&bar0)) : "memory");
        if (w == 0x123456789ull) cycles[0] = w;
      }
      if (V & 4) tc_fence_after();     // V bit 2: tcgen05.fence::after_thread_sync per k-block
      const uint32_t ta = (V & 64) ? acc + 4 * N + 64u * (k % ((512 - 4 * N) / 64)) : a0 + 64u * (k % ((512 - 2 * N) / 64));
      if (V & 64) {  // V bit 6: hi * [B; Bs] as one N = 2 * 64 MMA + lo * B (N = 64) into the small half
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t bd = smem_desc(sb + kk * 32, 16, 1024, 2);
          const uint32_t d = acc + (k / 7 % 2) * 2 * N;
          mma_tf32_ts(d, ta + 8 * kk, bd, idesc_tf32(128, 2 * N, false, false), 1u);
          if (V & 128) mma_tf32_ts(d, ta + 8 * kk + 32, bd, idesc_tf32(128, 2 * N, false, false), 1u);  // lo * [B; Bs]
          else mma_tf32_ts(d + N, ta + 8 * kk + 32, bd, idesc, 1u);
        }
        mma_commit(&bar2);
        continue;
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t bd = smem_desc(sb + kk * 32, 16, 1024, 2), bsd = smem_desc(sbs + kk * 32, 16, 1024, 2);
        mma_tf32_ts(acc + (k / 7 % 2) * N, ta + 8 * kk + 32, bd, idesc, 1u);
        mma_tf32_ts(acc + (k / 7 % 2) * N, ta + 8 * kk, bsd, idesc, 1u);
        mma_tf32_ts(acc + (k / 7 % 2) * N, ta + 8 * kk, bd, idesc, 1u);
        if ((V & 32) && kk == 1) mbar_wait(&bar0, 0);  // V bit 5: the try_wait mid-k-block
      }
      mma_commit((V & 2) ? &rot[k % 6] : &bar2);  // V bit 1: commit to 6 rotating barriers
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

// The same k-block pattern driven through igemm's stage ring: NS TMEM stages, the MMA thread
// waits full[s] (ARR arrivals from the consumer warps) and commits empty[s]; the consumer warps
// wait empty[s] and arrive on full[s] -- no data work at all, so the time is the MMAs plus
// whatever bubbles the ring's mbarrier round trip leaves.
__device__ __forceinline__ void wait_hint(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 32;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

template <int N, int NS, int ARR, int V = 0>
__global__ void probe_ring(int kblocks, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[8], empty[8], bar, bar0;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 2 * 256 * 32; i += blockDim.x) ((float*)smem)[i] = 0.f;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], ARR);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&bar, 1);
    mbar_init(&bar0, 1);
    mbar_arrive(&bar0);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tmem_base, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  unsigned long long t0 = clock64();
  if (warp == 0) {
    const uint32_t sb = smem_u32(smem), sbs = sb + N * 128;
    const uint32_t idesc = idesc_tf32(128, N, false, false);
    const uint32_t acc = tmem_base, a0 = tmem_base + 2 * N;
    for (int k = 0; k < kblocks; ++k) {
      const int s = k % NS;
      // V bit 0: no tcgen05.fence::after_thread_sync; bit 1: only the issuing lane waits; bit 2:
      // wait on an always-complete barrier instead; bit 3: try_wait with a 32-ns suspend hint
      if (V & 4) mbar_wait(&bar0, 0);
      else if (V & 8) wait_hint(&full[s], (k / NS) & 1);
      else if (!(V & 2) || tid == 0) mbar_wait(&full[s], (k / NS) & 1);
      if (!(V & 1)) tc_fence_after();
      if (tid == 0) {
        const uint32_t ta = a0 + 64u * s;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t bd = smem_desc(sb + kk * 32, 16, 1024, 2), bsd = smem_desc(sbs + kk * 32, 16, 1024, 2);
          mma_tf32_ts(acc + (k / 7 % 2) * N, ta + 8 * kk + 32, bd, idesc, 1u);
          mma_tf32_ts(acc + (k / 7 % 2) * N, ta + 8 * kk, bsd, idesc, 1u);
          mma_tf32_ts(acc + (k / 7 % 2) * N, ta + 8 * kk, bd, idesc, 1u);
        }
        mma_commit(&empty[s]);
      }
      if (!(V & 2) && !(V & 32)) __syncwarp();  // V bit 5: no __syncwarp
    }
    if (tid == 0) {
      mma_commit(&bar);
      mbar_wait(&bar, 0);
      cycles[blockIdx.x] = clock64() - t0;
    }
  } else if (warp <= 4 && !(V & 16)) {  // V bit 4: the consumer warps sit idle
    for (int k = 0; k < kblocks; ++k) {
      const int s = k % NS;
      if (k >= NS) {
        if (V & 8) wait_hint(&empty[s], ((k / NS) - 1) & 1);
        else mbar_wait(&empty[s], ((k / NS) - 1) & 1);
      }
      tc_fence_before();
      if (ARR == 128 || tid == 32) mbar_arrive(&full[s]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

template <int N, int NS, int ARR, int V = 0>
static float run_ring(int kblocks, unsigned long long* cyc) {
  const int smem = 2 * 256 * 128 + 2048;
  cudaFuncSetAttribute(probe_ring<N, NS, ARR, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  probe_ring<N, NS, ARR, V><<<148, 160, smem>>>(kblocks, cyc);
  cudaEventRecord(e0);
  probe_ring<N, NS, ARR, V><<<148, 160, smem>>>(kblocks, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

template <int N, int V = 0>
static float run_kb(int kblocks, unsigned long long* cyc) {
  const int smem = 2 * 256 * 128 + 2048;
  cudaFuncSetAttribute(probe_kblock<N, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  probe_kblock<N, V><<<148, 128, smem>>>(kblocks, cyc);
  cudaEventRecord(e0);
  probe_kblock<N, V><<<148, 128, smem>>>(kblocks, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

template <int N, bool TS>
static float run(int iters, unsigned long long* cyc) {
  const int smem = (128 + 256) * 128 + 2048;
  cudaFuncSetAttribute(probe<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  probe<N, TS><<<148, 128, smem>>>(iters, cyc);
  cudaEventRecord(e0);
  probe<N, TS><<<148, 128, smem>>>(iters, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

// which: 0..5 = N 64 / 128 / 256 with A in smem, then the same with A in TMEM; returns ms
extern "C" float mmaprobe_run(int which, int iters, unsigned long long* cyc) {
  switch (which) {
    case 0: return run<64, false>(iters, cyc);
    case 1: return run<128, false>(iters, cyc);
    case 2: return run<256, false>(iters, cyc);
    case 3: return run<64, true>(iters, cyc);
    case 4: return run<128, true>(iters, cyc);
    case 5: return run<256, true>(iters, cyc);
    case 6: return run_kb<64>(iters / 12, cyc);
    case 7: return run_kb<128>(iters / 12, cyc);
    case 8: return run_ring<64, 6, 128>(iters / 12, cyc);
    case 9: return run_ring<64, 6, 1>(iters / 12, cyc);
    case 10: return run_ring<64, 3, 128>(iters / 12, cyc);
    case 11: return run_ring<128, 3, 128>(iters / 12, cyc);
    case 12: return run_ring<64, 2, 128>(iters / 12, cyc);
    case 13: return run_ring<64, 6, 128, 1>(iters / 12, cyc);
    case 14: return run_ring<64, 6, 128, 2>(iters / 12, cyc);
    case 15: return run_ring<64, 6, 128, 3>(iters / 12, cyc);
    case 16: return run_ring<64, 6, 128, 4>(iters / 12, cyc);
    case 17: return run_ring<64, 6, 128, 8>(iters / 12, cyc);
    case 18: return run_ring<128, 3, 128, 4>(iters / 12, cyc);
    case 19: return run_ring<64, 6, 128, 4 + 16>(iters / 12, cyc);
    case 20: return run_ring<64, 6, 128, 4 + 16 + 1>(iters / 12, cyc);
    case 21: return run_ring<64, 6, 128, 4 + 16 + 1 + 32>(iters / 12, cyc);
    case 22: return run_ring<64, 6, 128, 4 + 32>(iters / 12, cyc);
    case 23: return run_kb<64, 1>(iters / 12, cyc);
    case 24: return run_kb<64, 2>(iters / 12, cyc);
    case 25: return run_kb<64, 4>(iters / 12, cyc);
    case 26: return run_kb<64, 7>(iters / 12, cyc);
    case 27: return run_kb<64, 8>(iters / 12, cyc);
    case 28: return run_kb<64, 16>(iters / 12, cyc);
    case 29: return run_kb<64, 32>(iters / 12, cyc);
    case 30: return run_kb<128, 1>(iters / 12, cyc);
    case 31: return run_kb<128, 0>(iters / 12, cyc);
    case 32: return run_kb<64, 64>(iters / 12, cyc);
    case 33: return run_kb<64, 65>(iters / 12, cyc);
    case 34: return run_kb<64, 64 + 128>(iters / 12, cyc);
    case 35: return run_kb<64, 65 + 128>(iters / 12, cyc);
  }
  return -1.f;
}
