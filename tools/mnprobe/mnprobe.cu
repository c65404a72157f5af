// mnprobe.cu -- does tcgen05.mma kind::tf32 read MN-major shared-memory operands on this B200?
// One CTA: D[M=128][N=128] = A * B^T over K = 32 with A given MN-major (global [K][M], row k
// holds the M values) and B MN-major (global [K][N]); TMA loads 32-column boxes with
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B and the smem descriptors use layout type
// SWIZZLE_128B_BASE32B (1), the layout CUTLASS requires for MN-major tf32 (sm100_smem_selector:
// "for mn-major tf32 operands, SW128_32B is the only available smem layout"); LBO = byte stride
// between 32-element MN chunks, SBO = byte stride between 4-row K groups.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o mnprobe.so mnprobe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../paper_1907_05013_b200/csrc/ptx.cuh"

using namespace pooch::ptx;

constexpr int M = 128, N = 128, K = 32;

__global__ void probe_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, float* d,
                             uint32_t lbo_a, uint32_t sbo_a, uint32_t lbo_b, uint32_t sbo_b, uint32_t layout,
                             int variant) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  float* sa = (float*)smem;                 // 4 chunks x [32 rows][32] = 16 KB
  float* sb = (float*)(smem + 16384);       // 16 KB
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    fence_mbar_init();
  }
  if (tid < 32) tmem_alloc(&tmem_base, 128);
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    mbar_arrive_expect_tx(&bar_load, 32768);
    for (int c = 0; c < 4; ++c) {
      tma_load_2d(smem_u32(sa) + c * 4096, &ta, &bar_load, c * 32, 0);
      tma_load_2d(smem_u32(sb) + c * 4096, &tb, &bar_load, c * 32, 0);
    }
  }
  mbar_wait(&bar_load, 0);
  if (tid == 0) {
    tc_fence_after();
    const uint32_t idesc = idesc_tf32(M, N, true, true);
    for (int kk = 0; kk < K / 8; ++kk) {
      // k-step of 8 rows = 2 four-row K groups: advance the start address by 8 rows of 128 B
      const uint32_t koff = kk * 8 * 128;
      const uint64_t da = smem_desc(smem_u32(sa) + koff, lbo_a, sbo_a, layout);
      const uint64_t db = smem_desc(smem_u32(sb) + koff, lbo_b, sbo_b, layout);
      mma_tf32(tmem_base, da, db, idesc, kk > 0 ? 1u : 0u);
    }
    mma_commit(&bar_mma);
  }
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  // 4 warps x 32 lanes = 128 rows; 4 x 32 columns
  const int warp = tid / 32, lane = tid % 32;
  for (int cb = 0; cb < N / 32; ++cb) {
    float v[32];
    tmem_ld32(tmem_base + ((warp * 32) << 16) + cb * 32, v);
    for (int j = 0; j < 32; ++j) d[(warp * 32 + lane) * N + cb * 32 + j] = v[j];
  }
  __syncthreads();
  if (tid < 32) tmem_dealloc(tmem_base, 128);
}

// Probe 2 (halo reuse): A is ONE 32-channel block of K + 4 rows (a halo strip); A's four MN
// chunks are that block shifted by q = 0..3 rows (chunk stride LBO = 128 B = one row), i.e.
// A[q*32 + c][k] = halo[k + q][c] -- the 3x3 wgrad's tap shift along W as a descriptor offset.
__global__ void probe2_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, float* d,
                              uint32_t lbo_a, uint32_t start_rows) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  float* sa = (float*)smem;                 // 40 rows x 128 B (halo) = 5 KB
  float* sb = (float*)(smem + 8192);        // B: 4 chunks x [32 rows][32] = 16 KB
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    fence_mbar_init();
  }
  if (tid < 32) tmem_alloc(&tmem_base, 128);
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    mbar_arrive_expect_tx(&bar_load, 40 * 128 + 16384);
    tma_load_2d(smem_u32(sa), &ta, &bar_load, 0, 0);
    for (int c = 0; c < 4; ++c) tma_load_2d(smem_u32(sb) + c * 4096, &tb, &bar_load, c * 32, 0);
  }
  mbar_wait(&bar_load, 0);
  if (tid == 0) {
    tc_fence_after();
    const uint32_t idesc = idesc_tf32(M, N, true, true);
    for (int kk = 0; kk < K / 8; ++kk) {
      const uint32_t koff = kk * 8 * 128;
      const uint64_t da = smem_desc(smem_u32(sa) + start_rows * 128 + koff, lbo_a, 512, 1);
      const uint64_t db = smem_desc(smem_u32(sb) + koff, 4096, 512, 1);
      mma_tf32(tmem_base, da, db, idesc, kk > 0 ? 1u : 0u);
    }
    mma_commit(&bar_mma);
  }
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  const int warp = tid / 32, lane = tid % 32;
  for (int cb = 0; cb < N / 32; ++cb) {
    float v[32];
    tmem_ld32(tmem_base + ((warp * 32) << 16) + cb * 32, v);
    for (int j = 0; j < 32; ++j) d[(warp * 32 + lane) * N + cb * 32 + j] = v[j];
  }
  __syncthreads();
  if (tid < 32) tmem_dealloc(tmem_base, 128);
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  return (PFN_cuTensorMapEncodeTiled_v12000)f;
}

// global [K rows][cols] row-major; box {32 cols, K rows}
static int make_map(CUtensorMap* m, const float* g, int cols, int swz) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)K};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)K};
  cuuint32_t es[2] = {1, 1};
  return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)g, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, (CUtensorMapSwizzle)swz, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

// halo [40 rows][32] row-major; box {32, 40}
static int make_halo_map(CUtensorMap* m, const float* g) {
  cuuint64_t dims[2] = {32, 40};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {32, 40};
  cuuint32_t es[2] = {1, 1};
  return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)g, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

extern "C" int mnprobe_halo(const float* halo, const float* b_kxn, float* d, uint32_t lbo_a, uint32_t start_rows) {
  CUtensorMap ta, tb;
  if (make_halo_map(&ta, halo) != 0 || make_map(&tb, b_kxn, N, 4) != 0) return 100;
  const int smem = 8192 + 16384 + 1024;
  cudaFuncSetAttribute(probe2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe2_kernel<<<1, 128, smem>>>(ta, tb, d, lbo_a, start_rows);
  return (int)cudaDeviceSynchronize();
}

extern "C" int mnprobe_run(const float* a_kxm, const float* b_kxn, float* d, uint32_t lbo_a, uint32_t sbo_a,
                           uint32_t lbo_b, uint32_t sbo_b, int layout, int swz) {
  CUtensorMap ta, tb;
  if (make_map(&ta, a_kxm, M, swz) != 0 || make_map(&tb, b_kxn, N, swz) != 0) return 100;
  const int smem = 32768 + 1024;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_kernel<<<1, 128, smem>>>(ta, tb, d, lbo_a, sbo_a, lbo_b, sbo_b, (uint32_t)layout, 0);
  cudaError_t e = cudaDeviceSynchronize();
  return (int)e;
}
