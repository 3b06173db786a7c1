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

int main() {
  for (int blocks : {1, 148}) {
    run<32, false>(blocks); run<64, false>(blocks); run<128, false>(blocks); run<256, false>(blocks);
    run<32, true>(blocks); run<64, true>(blocks); run<128, true>(blocks); run<256, true>(blocks);
  }
  return 0;
}
