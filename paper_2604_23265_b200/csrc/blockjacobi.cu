// Block-Jacobi preconditioner (NEXT-2; "the standard Block Jacobi preconditioner";
// DESIGN.md R35): P r = A_cc^{-1} r_c per cell, A_cc = diag((|c_m| + |s_m|)/h + sigma_t) - sigma_s S
// (the restriction of A to the cell's M ordinates).  The inverse blocks are built once per problem
// (lazily, on the first use) in fp64 by in-place Gauss-Jordan elimination with partial pivoting,
// one thread block per cell, and kept in fp64 and fp32; applying P is a batched M x M matvec.
#include <algorithm>
#include <string>

#include "common.h"

namespace rte {
namespace {

// In-place Gauss-Jordan inversion of the cell block in shared memory (fp64, partial pivoting).
__global__ void bj_invert_kernel(int N, int M, const double* __restrict__ sig_t, const double* __restrict__ sig_s,
                                 const double* __restrict__ St, const double* __restrict__ ax,
                                 const double* __restrict__ ay, double* __restrict__ inv64, float* __restrict__ inv32) {
  extern __shared__ double sm[];
  double* A = sm;                                       // [M][M]
  int* perm = reinterpret_cast<int*>(sm + (size_t)M * M);  // [M]
  __shared__ int piv;
  const int64_t cell = blockIdx.x;                      // global cell index b*N*N + j*N + i
  const int b = (int)(cell / ((int64_t)N * N));
  const double st = sig_t[cell], ss = sig_s[cell];
  const double* Stb = St + (int64_t)b * M * M;          // S^T[n][m]
  for (int e = threadIdx.x; e < M * M; e += blockDim.x) {
    const int m = e / M, n = e % M;
    A[e] = (m == n ? ax[m] + ay[m] + st : 0.0) - ss * Stb[(int64_t)n * M + m];
  }
  __syncthreads();
  for (int k = 0; k < M; ++k) {
    if (threadIdx.x == 0) {  // pivot: largest |A[i][k]|, i >= k
      int p = k;
      double best = fabs(A[k * M + k]);
      for (int i = k + 1; i < M; ++i)
        if (fabs(A[i * M + k]) > best) {
          best = fabs(A[i * M + k]);
          p = i;
        }
      piv = p;
      perm[k] = p;
    }
    __syncthreads();
    const int p = piv;
    if (p != k)
      for (int c = threadIdx.x; c < M; c += blockDim.x) {
        const double t = A[k * M + c];
        A[k * M + c] = A[p * M + c];
        A[p * M + c] = t;
      }
    __syncthreads();
    const double inv_piv = 1.0 / A[k * M + k];
    __syncthreads();
    for (int c = threadIdx.x; c < M; c += blockDim.x) A[k * M + c] = (c == k ? 1.0 : A[k * M + c]) * inv_piv;
    __syncthreads();
    for (int e = threadIdx.x; e < M * M; e += blockDim.x) {
      const int i = e / M, c = e % M;
      if (i == k) continue;
      const double f = A[i * M + k];  // (column k of row i, read before this row's update below)
      if (c == k) continue;
      A[e] -= f * A[k * M + c];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < M; i += blockDim.x)
      if (i != k) A[i * M + k] = -A[i * M + k] * inv_piv;
    __syncthreads();
  }
  // undo the row interchanges as column interchanges, in reverse order
  for (int k = M - 1; k >= 0; --k) {
    const int p = perm[k];
    if (p != k)
      for (int i = threadIdx.x; i < M; i += blockDim.x) {
        const double t = A[i * M + k];
        A[i * M + k] = A[i * M + p];
        A[i * M + p] = t;
      }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < M * M; e += blockDim.x) {
    inv64[cell * M * M + e] = A[e];
    inv32[cell * M * M + e] = (float)A[e];
  }
}

// y[cell][m] = alpha_b sum_n Binv[cell][m][n] x[cell][n]   (alpha scales the input, may be NULL)
template <typename T>
__global__ void bj_apply_kernel(const T* __restrict__ Binv, const T* __restrict__ x, T* __restrict__ y, int M,
                                int64_t ncell, int64_t cells_per_sample, const double* __restrict__ alpha,
                                int alpha_stride) {
  const int64_t n = ncell * M;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cell = e / M;
    const int m = (int)(e - cell * M);
    const T* row = Binv + (cell * M + m) * M;
    const T* xc = x + cell * M;
    T acc = T(0);
    for (int k = 0; k < M; ++k) acc = fma(row[k], xc[k], acc);
    const T al = alpha ? (T)alpha[(cell / cells_per_sample) * alpha_stride] : T(1);
    y[e] = al * acc;
  }
}

}  // namespace

void bj_prepare(const rte_problem* p) {
  if (p->bj64) return;
  RTE_REQUIRE(p->kind == 0, "block Jacobi: defined for the psi-space DO operator (not the (A)TFPS alpha-space systems)");
  const size_t blk = (size_t)p->M * p->M;
  const double gib = (double)p->ncell * blk * 12.0 / (1 << 30);
  RTE_REQUIRE(gib <= 24.0, "block Jacobi: the inverse cell blocks would need " + std::to_string(gib) +
                               " GiB (cells x M^2 x 12 B > 24 GiB)");
  const size_t smem = sizeof(double) * blk + sizeof(int) * p->M;
  RTE_REQUIRE(smem <= 200 * 1024, "block Jacobi: M too large for the in-shared-memory inversion (M <= 128)");
  p->bj64 = dalloc<double>(p->ncell * blk);
  p->bj32 = dalloc<float>(p->ncell * blk);
  if (smem > 48 * 1024)
    RTE_CHECK_CUDA(cudaFuncSetAttribute(bj_invert_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  prof_begin(nullptr, "bj_invert");
  bj_invert_kernel<<<(unsigned)p->ncell, 128, smem>>>(p->N, p->M, p->sig_t64, p->sig_s64, p->St64, p->ax64, p->ay64,
                                                       p->bj64, p->bj32);
  after_launch("bj_invert", nullptr, (double)p->ncell * 2.0 * blk * p->M, 12.0 * (double)p->ncell * blk, 3);
  RTE_CHECK_CUDA(cudaDeviceSynchronize());
}

template <typename T>
void bj_apply(const rte_problem* p, const T* x, T* y, const double* alpha, int alpha_stride, cudaStream_t st) {
  bj_prepare(p);
  const int64_t n = p->n;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
  const T* Binv;
  if constexpr (sizeof(T) == 4) Binv = p->bj32;
  else Binv = p->bj64;
  prof_begin(st, sizeof(T) == 4 ? "bj_apply" : "bj_apply_f64");
  bj_apply_kernel<T><<<blocks, 256, 0, st>>>(Binv, x, y, p->M, p->ncell, (int64_t)p->N * p->N, alpha, alpha_stride);
  after_launch(sizeof(T) == 4 ? "bj_apply" : "bj_apply_f64", st, 2.0 * (double)n * p->M,
               (double)sizeof(T) * ((double)n * 2 + (double)p->ncell * p->M * p->M), 0);
}
template void bj_apply<float>(const rte_problem*, const float*, float*, const double*, int, cudaStream_t);
template void bj_apply<double>(const rte_problem*, const double*, double*, const double*, int, cudaStream_t);

}  // namespace rte

using namespace rte;

rte_status rte_blockjacobi_apply(const rte_problem* p, const float* r_dev, float* z_dev, void* stream) {
  try {
    RTE_REQUIRE(p && r_dev && z_dev, "rte_blockjacobi_apply: NULL argument");
    RTE_REQUIRE((const void*)r_dev != (const void*)z_dev, "rte_blockjacobi_apply: r and z must not alias");
    bj_apply<float>(p, r_dev, z_dev, nullptr, 0, as_stream(stream));
    return RTE_OK;
  } catch (const Fail& f) {
    return f.st;
  }
}

rte_status rte_blockjacobi_apply_f64(const rte_problem* p, const double* r_dev, double* z_dev, void* stream) {
  try {
    RTE_REQUIRE(p && r_dev && z_dev, "rte_blockjacobi_apply_f64: NULL argument");
    RTE_REQUIRE((const void*)r_dev != (const void*)z_dev, "rte_blockjacobi_apply_f64: r and z must not alias");
    bj_apply<double>(p, r_dev, z_dev, nullptr, 0, as_stream(stream));
    return RTE_OK;
  } catch (const Fail& f) {
    return f.st;
  }
}
