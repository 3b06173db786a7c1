// Microbenchmark (experiments only): latency of the synchronisation primitives the GEMM pipeline
// uses -- mbarrier arrive -> try_wait hand-off between two warps, and tcgen05.commit -> mbarrier
// with no MMA in flight.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o sync_bench sync_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2604_23265_b200/csrc/tc_common.cuh"

using namespace rte::tc;

__global__ void pingpong(long long* out, int iters) {
  __shared__ uint64_t ping, pong;
  if (threadIdx.x == 0) {
    mbar_init(&ping, 1);
    mbar_init(&pong, 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const uint32_t ph = i & 1;
    if (warp == 0) {
      if (lane == 0) mbar_arrive(&ping);
      mbar_wait(&pong, ph);
    } else if (warp == 1) {
      mbar_wait(&ping, ph);
      if (lane == 0) mbar_arrive(&pong);
    }
  }
  if (threadIdx.x == 0) out[0] = (clock64() - t0) / iters;
}

__global__ void commit_lat(long long* out, int iters) {
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_alloc(&slot, 32);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      mma_commit_elect(&bar);
      mbar_wait(&bar, i & 1);
    }
    if (threadIdx.x == 0) out[1] = (clock64() - t0) / iters;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) mma_commit_elect(&bar);
    if (threadIdx.x == 0) out[2] = (clock64() - t0) / iters;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(slot, 32);
}

// 4-warp "converter" hand-off: 4 warps arrive (lane 0 each) on a count-4 barrier, one waiter.
__global__ void fanin(long long* out, int iters) {
  __shared__ uint64_t full, back;
  if (threadIdx.x == 0) {
    mbar_init(&full, 4);
    mbar_init(&back, 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const uint32_t ph = i & 1;
    if (warp >= 1 && warp <= 4) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&full);
      mbar_wait(&back, ph);
    } else if (warp == 0) {
      mbar_wait(&full, ph);
      if (lane == 0) mbar_arrive(&back);
    }
  }
  if (threadIdx.x == 0) out[3] = (clock64() - t0) / iters;
}

int main1() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  cudaMemset(d, 0, 8 * sizeof(long long));
  pingpong<<<1, 64>>>(d, 10000);
  commit_lat<<<1, 128>>>(d, 10000);
  fanin<<<1, 160>>>(d, 10000);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[8];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("mbarrier ping-pong round trip (2 hand-offs): %lld cycles (%s)\n", h[0], cudaGetErrorString(e));
  printf("tcgen05.commit -> mbarrier wait (nothing in flight): %lld cycles\n", h[1]);
  printf("tcgen05.commit issue only: %lld cycles\n", h[2]);
  printf("4-warp fan-in + reply round trip: %lld cycles\n", h[3]);
  return 0;
}
// (appended) costs of per-K-block instructions: tcgen05 fences, clock64, tcgen05.st + wait::st
__global__ void misc_costs(long long* out, int iters) {
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) tmem_alloc(&slot, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  float v[32];
  for (int i = 0; i < 32; ++i) v[i] = (float)i;
  if (threadIdx.x < 32) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) tc_fence_after();
    long long t1 = clock64();
    for (int i = 0; i < iters; ++i) tc_fence_before();
    long long t2 = clock64();
    long long acc = 0;
    for (int i = 0; i < iters; ++i) acc += clock64();
    long long t3 = clock64();
    for (int i = 0; i < iters; ++i) {
      tmem_st32(tm, v);
      tmem_wait_st();
    }
    long long t4 = clock64();
    for (int i = 0; i < iters; ++i) {
      tmem_st32(tm, v);
      tmem_st32(tm + 32, v);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
    }
    long long t5 = clock64();
    float w[32];
    for (int i = 0; i < iters; ++i) tmem_ld32(tm, w);
    long long t6 = clock64();
    if (threadIdx.x == 0) {
      out[4] = (t1 - t0) / iters;
      out[5] = (t2 - t1) / iters;
      out[6] = (t3 - t2) / iters + (acc == 42);
      out[7] = (t4 - t3) / iters;
      out[8] = (t5 - t4) / iters;
      out[9] = (t6 - t5) / iters + (w[3] == 1234.f);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tm, 128);
}

int main2() {
  long long* d;
  cudaMalloc(&d, 16 * sizeof(long long));
  misc_costs<<<1, 128>>>(d, 1000);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[16];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("tcgen05.fence::after_thread_sync: %lld cycles (%s)\n", h[4], cudaGetErrorString(e));
  printf("tcgen05.fence::before_thread_sync: %lld cycles\n", h[5]);
  printf("clock64: %lld cycles\n", h[6]);
  printf("tcgen05.st x32 + wait::st: %lld cycles\n", h[7]);
  printf("2x tcgen05.st x32 + wait::st + fence + syncwarp: %lld cycles\n", h[8]);
  printf("tcgen05.ld x32 + wait::ld: %lld cycles\n", h[9]);
  return 0;
}
int main() {
  main1();
  return main2();
}
