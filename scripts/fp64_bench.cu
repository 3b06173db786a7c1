// Microbenchmark (experiments only): B200 fp64 throughput, SIMT DFMA vs mma.sync m8n8k4 f64 (DMMA).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_bench fp64_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a[8], b = 1.0000001, c = 0.9999999;
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double acc[8][2];
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1])
                   : "d"(a), "d"(b));
  double s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000, blocks = sms * 4, threads = 256;
  float ms;
  dfma_kernel<<<blocks, threads>>>(d, 100);
  cudaEventRecord(e0);
  dfma_kernel<<<blocks, threads>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("SIMT DFMA: %.1f TFLOP/s\n", 2.0 * 8 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12);
  dmma_kernel<<<blocks, threads>>>(d, 100);
  cudaEventRecord(e0);
  dmma_kernel<<<blocks, threads>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  // per warp per mma: 8x8x4 MACs = 256 FMA = 512 flop
  printf("DMMA m8n8k4: %.1f TFLOP/s (%s)\n", 512.0 * 8 * iters * (double)blocks * (threads / 32) / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
