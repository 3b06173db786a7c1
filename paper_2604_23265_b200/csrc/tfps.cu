// TFPS alpha-space operator kernels (NEXT-3; §2.2; readings R37-R39).
//
// Unknowns alpha[b][j][i][k], k < 2 Md (x-modes, then y-modes of the cell's material).  A cell's
// solution at the midpoint of its face f is F_C(f) = L_mat (fac_mat[f] (.) alpha_C) (+ chi^s), with the
// material's eigenvectors L (columns) and basis factors fac (tfps_setup.cpp).  The equation rows a cell
// owns (R39):
//   rows [0, Md):   the face x = i h:  i > 0: F_(j,i-1)(R) - F_(j,i)(L)            (midpoint continuity)
//                                      i = 0: c_m > 0: F_(j,0)(L)_m, c_m < 0: F_(j,N-1)(R)_m (inflow rows)
//   rows [Md, 2Md): the face y = j h:  j > 0: F_(j-1,i)(T) - F_(j,i)(B)
//                                      j = 0: s_m > 0: F_(0,i)(B)_m, s_m < 0: F_(N-1,i)(T)_m
// (eq:2DTFPS_continuity_cond, eq:2DTFPS_boundary_cond; the particular-solution and inflow terms are
// the right-hand side, eq:2DTFPS_linear_sys).  Every row is two small dense contractions
// [2Md] -> [Md] with per-material matrices: a grouped GEMV per face, one warp per cell, the four
// scaled coefficient vectors staged in shared memory, L stored k-major so a warp's loads of one k
// row are coalesced over the output directions.
#include "common.h"

namespace rte {
namespace {

constexpr int kWarps = 8;

template <typename T>
__global__ void __launch_bounds__(32 * kWarps) tfps_apply_kernel(
    int B, int N, int Md, const int* __restrict__ mat, const T* __restrict__ LT, const T* __restrict__ fac,
    const T* __restrict__ x, T* __restrict__ y, const double* __restrict__ alpha, int alpha_stride,
    const float* __restrict__ bvec, const int8_t* __restrict__ sgx, const int8_t* __restrict__ sgy) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int K = 2 * Md;
  T* u = reinterpret_cast<T*>(smem_raw) + (size_t)warp * 4 * K;
  const int64_t cells = (int64_t)B * N * N;
  const int64_t cell = (int64_t)blockIdx.x * kWarps + warp;
  if (cell >= cells) return;
  const int i = (int)(cell % N), j = (int)((cell / N) % N);
  const int64_t base = cell - ((int64_t)j * N + i);  // first cell of the sample
  const int b = (int)(base / ((int64_t)N * N));
  const T al = alpha ? (T)alpha[(int64_t)b * alpha_stride] : T(1);
  // the four (cell, face) sources: 0 = (left or row-end cell, R), 1 = (C, L), 2 = (below or column-top, T), 3 = (C, B)
  int64_t src[4];
  src[0] = base + (int64_t)j * N + (i > 0 ? i - 1 : N - 1);
  src[1] = cell;
  src[2] = base + (int64_t)(j > 0 ? j - 1 : N - 1) * N + i;
  src[3] = cell;
  const int face[4] = {1, 0, 3, 2};  // R, L, T, B (fac rows: L, R, B, T, C)
  int ms[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    ms[s] = mat[src[s]];
    const T* f = fac + ((size_t)ms[s] * 5 + face[s]) * K;
    const T* a = x + src[s] * K;
    for (int k = lane; k < K; k += 32) u[s * K + k] = f[k] * a[k] * al;
  }
  __syncwarp();
  for (int m = lane; m < Md; m += 32) {
    T F[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const T* Lm = LT + (size_t)ms[s] * K * Md + m;
      const T* us = u + s * K;
      T acc = T(0);
      for (int k = 0; k < K; ++k) acc = fma(Lm[(size_t)k * Md], us[k], acc);
      F[s] = acc;
    }
    T ox = i > 0 ? F[0] - F[1] : (sgx[m] > 0 ? F[1] : F[0]);
    T oy = j > 0 ? F[2] - F[3] : (sgy[m] > 0 ? F[3] : F[2]);
    T* yo = y + cell * K;
    if (bvec) {
      const float* bo = bvec + cell * K;
      ox = (T)bo[m] - ox;
      oy = (T)bo[Md + m] - oy;
    }
    yo[m] = ox;
    yo[Md + m] = oy;
  }
}

// b: particular-solution jumps on interior faces, inflow minus the particular solution on boundary rows.
__global__ void tfps_rhs_kernel(int B, int N, int Md, const float* __restrict__ chis, const float* __restrict__ inflow,
                                const int8_t* __restrict__ sgx, const int8_t* __restrict__ sgy, float* __restrict__ bv) {
  const int K = 2 * Md;
  const int64_t n = (int64_t)B * N * N * K;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e % K);
    const int64_t cell = e / K;
    const int i = (int)(cell % N), j = (int)((cell / N) % N);
    const int b = (int)(cell / ((int64_t)N * N));
    const int64_t base = (int64_t)b * N * N;
    const float* inf = inflow ? inflow + (int64_t)b * 4 * N * Md : nullptr;
    double v;
    if (r < Md) {
      const int m = r;
      if (i > 0) {
        v = (double)chis[cell] - (double)chis[cell - 1];
      } else if (sgx[m] > 0) {
        v = (inf ? (double)inf[(0 * N + j) * Md + m] : 0.0) - (double)chis[cell];
      } else {
        v = (inf ? (double)inf[(1 * N + j) * Md + m] : 0.0) - (double)chis[base + (int64_t)j * N + N - 1];
      }
    } else {
      const int m = r - Md;
      if (j > 0) {
        v = (double)chis[cell] - (double)chis[cell - N];
      } else if (sgy[m] > 0) {
        v = (inf ? (double)inf[(2 * N + i) * Md + m] : 0.0) - (double)chis[cell];
      } else {
        v = (inf ? (double)inf[(3 * N + i) * Md + m] : 0.0) - (double)chis[base + (int64_t)(N - 1) * N + i];
      }
    }
    bv[e] = (float)v;
  }
}

// psi at the cell centres (eq:2DTFPS_sol): psi_m = sum_k L[m][k] fac[C][k] alpha_k + chi^s.
template <typename T>
__global__ void __launch_bounds__(32 * kWarps) tfps_reconstruct_kernel(int64_t cells, int Md,
                                                                       const int* __restrict__ mat,
                                                                       const T* __restrict__ LT,
                                                                       const T* __restrict__ fac,
                                                                       const T* __restrict__ chis,
                                                                       const T* __restrict__ x, T* __restrict__ psi) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int K = 2 * Md;
  T* u = reinterpret_cast<T*>(smem_raw) + (size_t)warp * K;
  const int64_t cell = (int64_t)blockIdx.x * kWarps + warp;
  if (cell >= cells) return;
  const int mt = mat[cell];
  const T* f = fac + ((size_t)mt * 5 + 4) * K;
  for (int k = lane; k < K; k += 32) u[k] = f[k] * x[cell * K + k];
  __syncwarp();
  for (int m = lane; m < Md; m += 32) {
    const T* Lm = LT + (size_t)mt * K * Md + m;
    T acc = T(0);
    for (int k = 0; k < K; ++k) acc = fma(Lm[(size_t)k * Md], u[k], acc);
    psi[cell * Md + m] = acc + chis[cell];
  }
}

}  // namespace

template <typename T>
void launch_tfps_apply(const rte_problem* p, const T* x, T* y, const double* alpha, int alpha_stride, const float* b,
                       cudaStream_t st) {
  const bool f64 = sizeof(T) == 8;
  const char* cls = f64 ? "tfps_apply_f64" : "tfps_apply_f32";
  prof_begin(st, cls);
  const int64_t cells = p->ncell;
  const size_t smem = sizeof(T) * kWarps * 4 * 2 * p->Md;
  auto kern = tfps_apply_kernel<T>;
  if (smem > 48 * 1024) RTE_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<(unsigned)((cells + kWarps - 1) / kWarps), 32 * kWarps, smem, st>>>(
      p->B, p->N, p->Md, p->tf_mat, f64 ? (const T*)p->tf_L64 : (const T*)p->tf_L32,
      f64 ? (const T*)p->tf_fac64 : (const T*)p->tf_fac32, x, y, alpha, alpha_stride, b, p->sgx, p->sgy);
  // 4 contractions [2Md] -> [Md] per cell; bytes: alpha read once (neighbours from cache), y written
  // (+ b read), the per-cell material index
  const double K = 2.0 * p->Md;
  after_launch(cls, st, (double)cells * 4.0 * 2.0 * K * p->Md,
               (double)cells * (K * sizeof(T) * 2 + (b ? K * 4 : 0) + 4), f64 ? 3 : 2);
}
template void launch_tfps_apply<float>(const rte_problem*, const float*, float*, const double*, int, const float*,
                                       cudaStream_t);
template void launch_tfps_apply<double>(const rte_problem*, const double*, double*, const double*, int, const float*,
                                        cudaStream_t);

void launch_tfps_rhs(const rte_problem* p, float* b, cudaStream_t st) {
  const int64_t n = p->n;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
  prof_begin(st, "tfps_rhs");
  tfps_rhs_kernel<<<blocks, 256, 0, st>>>(p->B, p->N, p->Md, p->tf_chis32, p->inflow, p->sgx, p->sgy, b);
  after_launch("tfps_rhs", st, 0.0, 4.0 * (double)n + 4.0 * p->ncell, 0);
}

template <typename T>
void launch_tfps_reconstruct(const rte_problem* p, const T* alpha, T* psi, cudaStream_t st) {
  const bool f64 = sizeof(T) == 8;
  const size_t smem = sizeof(T) * kWarps * 2 * p->Md;
  prof_begin(st, "tfps_reconstruct");
  tfps_reconstruct_kernel<T><<<(unsigned)((p->ncell + kWarps - 1) / kWarps), 32 * kWarps, smem, st>>>(
      p->ncell, p->Md, p->tf_mat, f64 ? (const T*)p->tf_L64 : (const T*)p->tf_L32,
      f64 ? (const T*)p->tf_fac64 : (const T*)p->tf_fac32, f64 ? (const T*)p->tf_chis64 : (const T*)p->tf_chis32,
      alpha, psi);
  after_launch("tfps_reconstruct", st, (double)p->ncell * 2.0 * 2.0 * p->Md * p->Md,
               (double)p->ncell * sizeof(T) * 3.0 * p->Md, 0);
}
template void launch_tfps_reconstruct<float>(const rte_problem*, const float*, float*, cudaStream_t);
template void launch_tfps_reconstruct<double>(const rte_problem*, const double*, double*, cudaStream_t);

}  // namespace rte
