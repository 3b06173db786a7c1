// Microbenchmark (experiments only): cycles per tcgen05.mma.kind::tf32 (M = 128, K = 8) as a
// function of N, with A from shared memory (SS) or TMEM (TS), B from shared memory; back-to-back
// MMAs into one accumulator issued by one elected thread, timed with clock64 around a commit wait.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../include -o mma_bench mma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2604_23265_b200/csrc/tc_common.cuh"

using namespace rte::tc;

template <int N, bool TS>
__global__ void bench(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  // zero the operand tiles (A: 128 x 32 fp32 = 16 KB, B: 256 x 32 fp32 = 32 KB)
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x < 32) {
    constexpr uint32_t idesc = idesc_tf32(128, N);
    const uint64_t da = sdesc_sw128(smem_u32(sm)), db = sdesc_sw128(smem_u32(sm + 16384));
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (TS)
          mma_tf32_ts_elect(tmem, tmem + 256 + 8 * k, db + 2 * k, idesc, 1);
        else
          mma_tf32_elect(tmem, da + 2 * k, db + 2 * k, idesc, 1);
      }
    }
    mma_commit_elect(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int N, bool TS>
void run(int blocks) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * blocks);
  const int iters = 2000;
  auto k = bench<N, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
  k<<<blocks, 128, 50 * 1024>>>(d, 10);
  k<<<blocks, 128, 50 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += h[i];
  avg /= blocks;
  const double per = avg / (iters * 4.0);
  const double flops = 2.0 * 128 * N * 8;
  printf("%s N=%3d blocks=%3d: %7.1f cycles/MMA  %7.0f flop/cycle/SM  (%s)\n", TS ? "TS" : "SS", N, blocks, per,
         flops / per, cudaGetErrorString(e));
  cudaFree(d);
}

int main_kblock();
int main() {
  main_kblock();
  for (int blocks : {148}) {
    run<32, false>(blocks); run<64, false>(blocks); run<128, false>(blocks); run<256, false>(blocks);
    run<32, true>(blocks); run<64, true>(blocks); run<128, true>(blocks); run<256, true>(blocks);
  }
  return 0;
}

// (appended) The fused 3xTF32 K-block of the conv kernel (BN = 32): per K block, 4 K steps of
// [TS N=64 hi.[Bhi;Blo] -> D0, TS N=32 lo.Bhi -> D1], A alternating between two TMEM buffers, then
// commits (bempty, afree); optionally a converter-like warp group writing the other A buffer with
// tcgen05.st while the MMAs run, to expose TMEM port contention.
template <bool STORES>
__global__ void kblock(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[2];
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    constexpr uint32_t id64 = idesc_tf32(128, 64), id32 = idesc_tf32(128, 32);
    const uint64_t db = sdesc_sw128(smem_u32(sm));
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t a = tmem + 384 + 64 * (i & 1);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        mma_tf32_ts_elect(tmem, a + 8 * k, db + 2 * k, id64, 1);
        mma_tf32_ts_elect(tmem + 32, a + 32 + 8 * k, db + 2 * k, id32, 1);
      }
      mma_commit_elect(&bar[0]);
      mma_commit_elect(&bar[1]);
    }
    mbar_wait(&bar[0], (iters - 1) & 1);
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  } else if (STORES && warp >= 2 && warp < 6) {
    float v[32];
    for (int j = 0; j < 32; ++j) v[j] = 0.f;
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    for (int i = 0; i < iters; ++i) {
      const uint32_t a = tmem + 384 + 64 * ((i + 1) & 1) + lane_base;
      tmem_st32(a, v);
      tmem_st32(a + 32, v);
      tmem_wait_st();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <bool STORES>
void run_kblock(int blocks) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * blocks);
  const int iters = 2000;
  auto k = kblock<STORES>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 20 * 1024);
  k<<<blocks, 192, 20 * 1024>>>(d, 10);
  k<<<blocks, 192, 20 * 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += h[i];
  printf("K block (4x [TS N=64 + TS N=32]) %s, blocks=%d: %.1f cycles (%s)\n", STORES ? "with concurrent tcgen05.st" : "alone",
         blocks, avg / blocks / iters, cudaGetErrorString(e));
  cudaFree(d);
}

int main_kblock() {
  run_kblock<false>(1);
  run_kblock<false>(148);
  run_kblock<true>(1);
  run_kblock<true>(148);
  return 0;
}
