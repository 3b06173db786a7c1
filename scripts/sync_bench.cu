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

int main() {
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
