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
#include <type_traits>

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

// ---- ATFPS compressed system (NEXT-3b, readings R40-R42) ------------------------
// Padded layout [cells][2 Md]: the row of a selected mode k of cell C sits at slot (C, k); dropped modes
// carry the identity row.  Mode k is centred at face k / (Md/2) in L, R, B, T.  Per cell (one warp): the
// selected-mode traces of the cell at its 4 faces and of the 4 neighbours at the shared faces, the jump
// vector of each face, then each selected mode's row = its P-row (interface type: the material pair, or
// the boundary face and material) dotted with the jump of its face.
//   MODE 0 (A x):  jumps of the selected traces, y = x on dropped slots (y = b - A x with b);
//   MODE 1 (b):    particular-solution jumps / inflow minus the particular solution; 0 on dropped slots;
//   MODE 2 (layer, eq:2DAdaptive_TFPS_layer1/2): the full coefficients -- selected = x, dropped = the
//                  projected jump of the smooth solution psi_bar = sum_sel x chi + chi^s.
template <typename T, int MODE>
__global__ void __launch_bounds__(32 * kWarps) atfps_kernel(
    int B, int N, int Md, int nmat, const int* __restrict__ mat, const uint8_t* __restrict__ sel,
    const T* __restrict__ LT, const T* __restrict__ fac, const T* __restrict__ chis, const float* __restrict__ inflow,
    const T* __restrict__ P, const int* __restrict__ row, const int* __restrict__ dirs, const T* __restrict__ x,
    T* __restrict__ y, const double* __restrict__ alpha, int alpha_stride, const float* __restrict__ bvec) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int K = 2 * Md, H = Md / 2;
  T* u = reinterpret_cast<T*>(smem_raw) + (size_t)warp * (8 * K + 4 * Md);  // 8 scaled coefficient vectors
  T* v = u + 8 * K;                                                          // 4 jump vectors (L, R, B, T)
  const int64_t cells = (int64_t)B * N * N;
  const int64_t cell = (int64_t)blockIdx.x * kWarps + warp;
  if (cell >= cells) return;
  const int i = (int)(cell % N), j = (int)((cell / N) % N);
  const int64_t base = cell - ((int64_t)j * N + i);
  const int b = (int)(base / ((int64_t)N * N));
  const T al = alpha ? (T)alpha[(int64_t)b * alpha_stride] : T(1);
  const int mC = mat[cell];
  // neighbours across L, R, B, T (-1 outside the grid)
  const int64_t nb[4] = {i > 0 ? cell - 1 : -1, i < N - 1 ? cell + 1 : -1, j > 0 ? cell - N : -1,
                         j < N - 1 ? cell + N : -1};
  // traces: s = 0..3 the cell at its faces L, R, B, T; s = 4..7 the neighbour across face s-4 at the
  // shared face (R, L, T, B of the neighbour)
  int tm[8];
  int64_t tc[8];
  int tf[8];
  const int opp[4] = {1, 0, 3, 2};
  for (int s = 0; s < 8; ++s) {
    tc[s] = s < 4 ? cell : nb[s - 4];
    tf[s] = s < 4 ? s : opp[s - 4];
    tm[s] = tc[s] >= 0 ? mat[tc[s]] : 0;
  }
  if (MODE != 1) {
    for (int s = 0; s < 8; ++s) {
      if (tc[s] < 0) continue;
      const T* f = fac + ((size_t)tm[s] * 5 + tf[s]) * K;
      const uint8_t* sl = sel + (size_t)tm[s] * K;
      const T* a = x + tc[s] * K;
      for (int k = lane; k < K; k += 32) u[s * K + k] = sl[k] ? f[k] * a[k] * al : T(0);
    }
    __syncwarp();
  }
  // the jump vector of each face (the component list of boundary faces is dirs[face])
  for (int fa = 0; fa < 4; ++fa) {
    const bool interior = nb[fa] >= 0;
    const int d = interior ? Md : H;
    const bool low = fa == 0 || fa == 2;  // L or B: the cell is C+ (the neighbour is C-)
    for (int q = lane; q < d; q += 32) {
      const int m = interior ? q : dirs[fa * H + q];
      T tC = T(0), tN = T(0);
      if (MODE != 1) {
        const T* Lm = LT + m;
        for (int s2 = 0; s2 < 2; ++s2) {
          const int s = s2 == 0 ? fa : 4 + fa;
          if (tc[s] < 0) continue;
          const T* Lms = Lm + (size_t)tm[s] * K * Md;
          const T* us = u + s * K;
          T acc = T(0);
          for (int k = 0; k < K; ++k) acc = fma(Lms[(size_t)k * Md], us[k], acc);
          (s2 == 0 ? tC : tN) = acc;
        }
      }
      T val;
      if (interior) {
        const T cC = chis[cell], cN = chis[nb[fa]];
        const T tm_ = low ? tN : tC, tp_ = low ? tC : tN;         // traces of C- and C+
        const T cm_ = low ? cN : cC, cp_ = low ? cC : cN;
        if (MODE == 0) val = tm_ - tp_;
        else if (MODE == 1) val = cp_ - cm_;
        else val = low ? (tm_ + cm_) - (tp_ + cp_) : (tp_ + cp_) - (tm_ + cm_);  // P^k(other) - P^k(own)
      } else {
        const int pos = (fa < 2) ? j : i;
        const T psi_in = inflow ? (T)inflow[(((int64_t)b * 4 + fa) * N + pos) * Md + m] : T(0);
        if (MODE == 0) val = tC;
        else if (MODE == 1) val = psi_in - chis[cell];
        else val = psi_in - (tC + chis[cell]);
      }
      v[fa * Md + q] = val;
    }
  }
  __syncwarp();
  const uint8_t* slC = sel + (size_t)mC * K;
  const size_t nint = (size_t)2 * nmat * nmat;
  for (int k = lane; k < K; k += 32) {
    const int fa = k / H;
    const bool keep = slC[k] != 0;
    T out;
    if ((MODE == 2) == keep) {
      out = MODE == 0 ? x[cell * K + k] * al : MODE == 1 ? T(0) : x[cell * K + k];
    } else {
      const bool interior = nb[fa] >= 0;
      const T* Pr;
      int r, d;
      if (interior) {
        const bool low = fa == 0 || fa == 2;
        const int o = fa < 2 ? 0 : 1;
        const int mm = low ? mat[nb[fa]] : mC, mp = low ? mC : mat[nb[fa]];
        const size_t t = ((size_t)o * nmat + mm) * nmat + mp;
        d = Md;
        r = row[t * 2 * K + (low ? 1 : 0) * K + k];
        Pr = P + t * Md * Md + (size_t)r * Md;
      } else {
        const size_t t = (size_t)fa * nmat + mC;
        d = H;
        r = row[(nint + t) * 2 * K + k];
        Pr = P + nint * Md * Md + t * H * H + (size_t)r * H;
      }
      T acc = T(0);
      const T* vf = v + fa * Md;
      for (int q = 0; q < d; ++q) acc = fma(Pr[q], vf[q], acc);
      out = acc;
    }
    if (MODE == 0 && bvec) out = (T)bvec[cell * K + k] - out;
    y[cell * K + k] = out;
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

template <typename T>
void launch_atfps(const rte_problem* p, int mode, const T* x, T* y, const double* alpha, int alpha_stride,
                  const float* b, cudaStream_t st) {
  const bool f64 = sizeof(T) == 8;
  const char* cls = mode == 1 ? "atfps_rhs" : mode == 2 ? "atfps_layer" : f64 ? "atfps_apply_f64" : "atfps_apply_f32";
  prof_begin(st, cls);
  const int64_t cells = p->ncell;
  const int K = 2 * p->Md;
  const size_t smem = sizeof(T) * kWarps * (8 * K + 4 * p->Md);
  auto go = [&](auto mode_tag) {
    constexpr int MODE = decltype(mode_tag)::value;
    auto kern = atfps_kernel<T, MODE>;
    if (smem > 48 * 1024) RTE_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)((cells + kWarps - 1) / kWarps), 32 * kWarps, smem, st>>>(
        p->B, p->N, p->Md, p->nmat, p->tf_mat, p->at_sel, f64 ? (const T*)p->tf_L64 : (const T*)p->tf_L32,
        f64 ? (const T*)p->tf_fac64 : (const T*)p->tf_fac32, f64 ? (const T*)p->tf_chis64 : (const T*)p->tf_chis32,
        p->inflow, f64 ? (const T*)p->at_P64 : (const T*)p->at_P32, p->at_row, p->at_dirs, x, y, alpha,
        alpha_stride, b);
  };
  if (mode == 0) go(std::integral_constant<int, 0>{});
  else if (mode == 1) go(std::integral_constant<int, 1>{});
  else go(std::integral_constant<int, 2>{});
  // 8 trace contractions [2Md] -> [Md] and 2Md projections of length Md per cell
  const double Kd = 2.0 * p->Md;
  after_launch(cls, st, (double)cells * (8.0 * 2.0 * Kd * p->Md + 2.0 * Kd * p->Md),
               (double)cells * (Kd * sizeof(T) * 2 + (b ? Kd * 4 : 0) + 4), f64 ? 3 : 2);
}
template void launch_atfps<float>(const rte_problem*, int, const float*, float*, const double*, int, const float*,
                                  cudaStream_t);
template void launch_atfps<double>(const rte_problem*, int, const double*, double*, const double*, int,
                                   const float*, cudaStream_t);

}  // namespace rte
