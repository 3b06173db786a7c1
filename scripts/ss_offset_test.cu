// Experiment: can a K-major SWIZZLE_128B shared-memory descriptor start at a row that is not a
// multiple of 8 (i.e. not 1024-byte aligned)?  A 256 x 32 fp32 tile is written in the TMA SW128
// layout (row R, 16-byte chunk q at R*128 + ((q ^ (R & 7)) << 4)); D = A[s .. s+127] . B^T is
// computed with 4 tf32 K steps for several row offsets s and two choices of the descriptor's
// base-offset field (bits 49-51), and compared with the exact host product (small integers).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o ss_offset_test ss_offset_test.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../paper_2604_23265_b200/csrc/tc_common.cuh"

using namespace rte::tc;

constexpr int kRowsA = 256, kN = 32, kK = 32;

__host__ __device__ inline float aval(int r, int k) { return (float)(((r * 7 + k * 3) % 17) - 8); }
__host__ __device__ inline float bval(int n, int k) { return (float)(((n * 5 + k * 11) % 13) - 6); }

__device__ inline uint32_t sw_off(int r, int k) { return r * 128 + ((((k >> 2) ^ (r & 7))) << 4) + (k & 3) * 4; }

__global__ void ss_offset(float* out, int s, int bo_mode) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* A = sm;
  uint8_t* B = sm + kRowsA * 128;
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < kRowsA * kK; i += blockDim.x) {
    const int r = i / kK, k = i % kK;
    *reinterpret_cast<float*>(A + sw_off(r, k)) = aval(r, k);
  }
  for (int i = threadIdx.x; i < kN * kK; i += blockDim.x) {
    const int n = i / kK, k = i % kK;
    *reinterpret_cast<float*>(B + sw_off(n, k)) = bval(n, k);
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x < 32) tmem_alloc(&slot, 32);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x < 32) {
    constexpr uint32_t idesc = idesc_tf32(128, kN);
    const uint32_t a_addr = smem_u32(A) + (uint32_t)s * 128u;
    uint64_t da = sdesc_sw128(a_addr);
    if (bo_mode == 1) da |= (uint64_t)((a_addr >> 7) & 7) << 49;
    const uint64_t db = sdesc_sw128(smem_u32(B));
#pragma unroll
    for (int k = 0; k < 4; ++k) mma_tf32_elect(tmem, da + 2 * k, db + 2 * k, idesc, k > 0);
    mma_commit_elect(&bar);
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  tc_fence_after();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float v[32];
  tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), v);
  const int row = warp * 32 + lane;
  for (int n = 0; n < kN; ++n) out[row * kN + n] = v[n];
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 32);
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * kN * sizeof(float));
  float* h = (float*)malloc(128 * kN * sizeof(float));
  const int smem = kRowsA * 128 + kN * 128 + 1024;
  cudaFuncSetAttribute(ss_offset, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int offs[] = {0, 1, 2, 3, 5, 7, 8, 9, 32, 33, 34, 66, 127};
  for (int bo = 0; bo < 2; ++bo) {
    for (int s : offs) {
      ss_offset<<<1, 128, smem>>>(d, s, bo);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, 128 * kN * sizeof(float), cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int r = 0; r < 128; ++r)
        for (int n = 0; n < kN; ++n) {
          double ref = 0;
          for (int k = 0; k < kK; ++k) ref += (double)aval(s + r, k) * bval(n, k);
          if (h[r * kN + n] != (float)ref) ++bad;
        }
      printf("base_offset_mode=%d s=%3d: %s, %d / %d wrong\n", bo, s, cudaGetErrorString(e), bad, 128 * kN);
    }
  }
  return 0;
}
