// The filtered loss of the training objective (NEXT-4, eq:loss / eq:loss_delta;
// readings R43-R45) on an ATFPS problem (rte_setup_atfps):
//
//   loss_delta = || b_bar_delta - A_bar_delta D_delta psi_d ||_2    (per sample)
//
// * D_delta (R43): per cell, the samples of psi_d at the centre and the four face midpoints (the average
//   of the two adjacent cell-centre values; the cell's own value at a boundary face) minus chi^s, times the
//   material's minimum-norm least-squares fit operator Dp [2Md][5Md] (tfps_setup.cpp atfps_fit_pinv; rows
//   of dropped modes 0).  fit_kernel: one warp per cell, the 5 Md samples staged in shared memory.
// * A_bar, b_bar: the compressed operator and right-hand side of tfps.cu (launch_atfps modes 0 and 1).
// * The gradient with respect to psi_d (what training back-propagates, R45):
//   g = D_lin^T A_bar^T w, w = -r / ||r|| per sample: atfps_adjoint_kernel applies A_bar^T (per cell: the
//   rows of each face -- the cell's own modes centred there and the neighbour's modes centred at the
//   opposite face -- projected back with their P-rows into a direction vector, then L^T and the face
//   factor of the cell's trace, with the sign of the cell's side of the jump; the identity on dropped
//   slots), fit_adjoint_kernel applies Dp^T per cell and scatter_kernel the transpose of the sampling
//   (centre, half of each interior face sample to either cell, all of a boundary face sample).
// fp32 and fp64 instantiations; reductions in fp64, fixed order (deterministic).
#include <cmath>
#include <type_traits>
#include <vector>

#include "common.h"

namespace rte {
namespace {

constexpr int kWarps = 8;

template <typename T>
__global__ void __launch_bounds__(32 * kWarps) fit_kernel(int B, int N, int Md, const int* __restrict__ mat,
                                                          const T* __restrict__ Dp, const T* __restrict__ chis,
                                                          const T* __restrict__ psi, T* __restrict__ alpha) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int K = 2 * Md, R = 5 * Md;
  T* y = reinterpret_cast<T*>(smem_raw) + (size_t)warp * R;
  const int64_t cells = (int64_t)B * N * N;
  const int64_t cell = (int64_t)blockIdx.x * kWarps + warp;
  if (cell >= cells) return;
  const int i = (int)(cell % N), j = (int)((cell / N) % N);
  const int64_t nb[4] = {i > 0 ? cell - 1 : -1, i < N - 1 ? cell + 1 : -1, j > 0 ? cell - N : -1,
                         j < N - 1 ? cell + N : -1};  // L, R, B, T
  const T cs = chis[cell];
  for (int m = lane; m < Md; m += 32) {
    const T c = psi[cell * Md + m];
    y[m] = c - cs;
    for (int f = 0; f < 4; ++f) y[(1 + f) * Md + m] = (nb[f] >= 0 ? T(0.5) * (c + psi[nb[f] * Md + m]) : c) - cs;
  }
  __syncwarp();
  const T* D = Dp + (size_t)mat[cell] * K * R;
  for (int k = lane; k < K; k += 32) {
    const T* Dk = D + (size_t)k * R;
    T acc = T(0);
    for (int q = 0; q < R; ++q) acc = fma(Dk[q], y[q], acc);
    alpha[cell * K + k] = acc;
  }
}

// r = b_bar - r (r holds A_bar alpha on entry); norm2[b] = sum of r^2 over sample b (one block per
// sample, fp64, fixed-order tree: deterministic)
template <typename T>
__global__ void __launch_bounds__(1024) residual_norm_kernel(int64_t per, const T* __restrict__ bbar, T* __restrict__ r,
                                                             double* __restrict__ norm2) {
  __shared__ double red[1024];
  const int64_t base = (int64_t)blockIdx.x * per;
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < per; e += blockDim.x) {
    const T v = bbar[base + e] - r[base + e];
    r[base + e] = v;
    s += (double)v * (double)v;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) norm2[blockIdx.x] = red[0];
}

// ga = A_bar^T (-r / ||r||)  (see the file header; tfps.cu atfps_kernel MODE 0 is the forward)
template <typename T>
__global__ void __launch_bounds__(32 * kWarps) atfps_adjoint_kernel(
    int B, int N, int Md, int nmat, const int* __restrict__ mat, const uint8_t* __restrict__ sel,
    const T* __restrict__ LT, const T* __restrict__ fac, const T* __restrict__ P, const int* __restrict__ row,
    const int* __restrict__ dirs, const T* __restrict__ r, const double* __restrict__ norm2, T* __restrict__ ga) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int K = 2 * Md, H = Md / 2;
  T* wf = reinterpret_cast<T*>(smem_raw) + (size_t)warp * 4 * Md;  // per face: sum of P-rows x row weights
  const int64_t cells = (int64_t)B * N * N;
  const int64_t cell = (int64_t)blockIdx.x * kWarps + warp;
  if (cell >= cells) return;
  const int i = (int)(cell % N), j = (int)((cell / N) % N);
  const int b = (int)(cell / ((int64_t)N * N));
  const double n2 = norm2[b];
  const T scale = n2 > 0.0 ? (T)(-1.0 / sqrt(n2)) : T(0);
  const int mC = mat[cell];
  const int64_t nb[4] = {i > 0 ? cell - 1 : -1, i < N - 1 ? cell + 1 : -1, j > 0 ? cell - N : -1,
                         j < N - 1 ? cell + N : -1};
  const int opp[4] = {1, 0, 3, 2};
  const size_t nint = (size_t)2 * nmat * nmat;
  const uint8_t* slC = sel + (size_t)mC * K;
  for (int fa = 0; fa < 4; ++fa) {
    T* w = wf + fa * Md;
    if (nb[fa] >= 0) {
      const bool low = fa == 0 || fa == 2;  // the cell is C+ at its L / B faces
      const int o = fa < 2 ? 0 : 1;
      const int mN = mat[nb[fa]];
      const int mm = low ? mN : mC, mp = low ? mC : mN;
      const size_t t = ((size_t)o * nmat + mm) * nmat + mp;
      const T* Pt = P + t * Md * Md;
      const uint8_t* slN = sel + (size_t)mN * K;
      const int fo = opp[fa];
      for (int m = lane; m < Md; m += 32) {
        T acc = T(0);
        for (int kk = 0; kk < H; ++kk) {  // the rows of this face: the cell's modes centred at fa ...
          const int k = fa * H + kk;
          if (slC[k]) acc = fma(r[cell * K + k], Pt[(size_t)row[t * 2 * K + (low ? 1 : 0) * K + k] * Md + m], acc);
        }
        for (int kk = 0; kk < H; ++kk) {  // ... and the neighbour's modes centred at the opposite face
          const int k = fo * H + kk;
          if (slN[k]) acc = fma(r[nb[fa] * K + k], Pt[(size_t)row[t * 2 * K + (low ? 0 : 1) * K + k] * Md + m], acc);
        }
        w[m] = low ? -acc : acc;  // jump = trace(C-) - trace(C+)
      }
    } else {
      const size_t t = (size_t)fa * nmat + mC;
      const T* Pb = P + nint * Md * Md + t * H * H;
      for (int m = lane; m < Md; m += 32) w[m] = T(0);
      __syncwarp();
      for (int q = lane; q < H; q += 32) {
        T acc = T(0);
        for (int kk = 0; kk < H; ++kk) {
          const int k = fa * H + kk;
          if (slC[k]) acc = fma(r[cell * K + k], Pb[(size_t)row[(nint + t) * 2 * K + k] * H + q], acc);
        }
        w[dirs[fa * H + q]] = acc;  // boundary row = P-row . trace restricted to the incoming directions
      }
    }
  }
  __syncwarp();
  const T* Lc = LT + (size_t)mC * K * Md;
  const T* fc = fac + (size_t)mC * 5 * K;
  for (int k = lane; k < K; k += 32) {
    T out;
    if (slC[k]) {
      const T* Lk = Lc + (size_t)k * Md;
      T acc = T(0);
      for (int fa = 0; fa < 4; ++fa) {
        T s = T(0);
        for (int m = 0; m < Md; ++m) s = fma(Lk[m], wf[fa * Md + m], s);
        acc = fma(fc[(size_t)fa * K + k], s, acc);
      }
      out = acc;
    } else {
      out = r[cell * K + k];  // identity row of a dropped slot
    }
    ga[cell * K + k] = out * scale;
  }
}

// u[C] = Dp^T ga[C]  ([5Md] per cell)
template <typename T>
__global__ void __launch_bounds__(32 * kWarps) fit_adjoint_kernel(int64_t cells, int Md, const int* __restrict__ mat,
                                                                  const T* __restrict__ Dp, const T* __restrict__ ga,
                                                                  T* __restrict__ u) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int K = 2 * Md, R = 5 * Md;
  const int64_t cell = (int64_t)blockIdx.x * kWarps + warp;
  if (cell >= cells) return;
  const T* D = Dp + (size_t)mat[cell] * K * R;
  const T* g = ga + cell * K;
  for (int q = lane; q < R; q += 32) {
    T acc = T(0);
    for (int k = 0; k < K; ++k) acc = fma(D[(size_t)k * R + q], g[k], acc);
    u[cell * R + q] = acc;
  }
}

// g_psi[C][m] = u[C][centre] + sum_f (interior ? 1/2 : 1) u[C][f] + sum_f interior 1/2 u[nb_f][opposite f]
template <typename T>
__global__ void scatter_kernel(int B, int N, int Md, const T* __restrict__ u, T* __restrict__ g) {
  const int64_t n = (int64_t)B * N * N * Md;
  const int R = 5 * Md;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(e % Md);
    const int64_t cell = e / Md;
    const int i = (int)(cell % N), j = (int)((cell / N) % N);
    const int64_t nb[4] = {i > 0 ? cell - 1 : -1, i < N - 1 ? cell + 1 : -1, j > 0 ? cell - N : -1,
                           j < N - 1 ? cell + N : -1};
    const int opp[4] = {1, 0, 3, 2};
    const T* uc = u + cell * R;
    T acc = uc[m];
    for (int f = 0; f < 4; ++f) {
      if (nb[f] >= 0) {
        acc += T(0.5) * uc[(1 + f) * Md + m];
        acc += T(0.5) * u[nb[f] * R + (1 + opp[f]) * Md + m];
      } else {
        acc += uc[(1 + f) * Md + m];
      }
    }
    g[e] = acc;
  }
}

// the fit operators on the device (built on first use; fp64 and fp32 copies)
void prepare(const rte_problem* p) {
  if (p->ls_Dp64) return;
  RTE_REQUIRE(p->kind == 2, "filtered loss: not an ATFPS problem (rte_setup_atfps)");
  const int Md = p->Md, K = 2 * Md, R = 5 * Md, nmat = p->nmat;
  std::vector<uint8_t> sel((size_t)nmat * K);
  std::vector<double> fac((size_t)nmat * 5 * K);
  RTE_CHECK_CUDA(cudaMemcpy(sel.data(), p->at_sel, sel.size(), cudaMemcpyDeviceToHost));
  RTE_CHECK_CUDA(cudaMemcpy(fac.data(), p->tf_fac64, sizeof(double) * fac.size(), cudaMemcpyDeviceToHost));
  std::vector<double> Dp((size_t)nmat * K * R);
  for (int m = 0; m < nmat; ++m)
    atfps_fit_pinv(p->tf_Lh.data() + (size_t)m * Md * K, fac.data() + (size_t)m * 5 * K, sel.data() + (size_t)m * K,
                   Md, Dp.data() + (size_t)m * K * R);
  std::vector<float> Dp32(Dp.begin(), Dp.end());
  p->ls_Dp64 = dalloc<double>(Dp.size());
  upload(p->ls_Dp64, Dp.data(), Dp.size());
  p->ls_Dp32 = dalloc<float>(Dp.size());
  upload(p->ls_Dp32, Dp32.data(), Dp.size());
  p->ls_ws_bytes = sizeof(double) * ((size_t)3 * p->n + (size_t)p->ncell * R);
  p->ls_ws = dalloc<unsigned char>(p->ls_ws_bytes);
  p->ls_norm = dalloc<double>(p->B);
}

template <typename T>
const T* dp_of(const rte_problem* p) {
  return std::is_same<T, double>::value ? (const T*)p->ls_Dp64 : (const T*)p->ls_Dp32;
}

}  // namespace

template <typename T>
void atfps_fit(const rte_problem* p, const T* psi, T* alpha, cudaStream_t st) {
  prepare(p);
  const bool f64 = sizeof(T) == 8;
  const int64_t cells = p->ncell;
  const int Md = p->Md;
  prof_begin(st, "loss_fit");
  fit_kernel<T><<<(unsigned)((cells + kWarps - 1) / kWarps), 32 * kWarps, sizeof(T) * kWarps * 5 * Md, st>>>(
      p->B, p->N, Md, p->tf_mat, dp_of<T>(p), f64 ? (const T*)p->tf_chis64 : (const T*)p->tf_chis32, psi, alpha);
  after_launch("loss_fit", st, (double)cells * 2.0 * 2.0 * Md * 5.0 * Md, (double)cells * sizeof(T) * 3.0 * Md, 0);
}

template <typename T>
void atfps_loss(const rte_problem* p, const T* psi, double* loss_host, T* grad, cudaStream_t st) {
  prepare(p);
  const bool f64 = sizeof(T) == 8;
  const int64_t n = p->n, cells = p->ncell;
  const int Md = p->Md, K = 2 * Md;
  T* alpha = reinterpret_cast<T*>(p->ls_ws);
  T* r = alpha + n;
  T* bbar = r + n;
  T* u = bbar + n;
  atfps_fit<T>(p, psi, alpha, st);
  launch_atfps<T>(p, 1, nullptr, bbar, nullptr, 0, nullptr, st);  // b_bar
  launch_atfps<T>(p, 0, alpha, r, nullptr, 0, nullptr, st);       // A_bar alpha
  prof_begin(st, "loss_norm");
  residual_norm_kernel<T><<<p->B, 1024, 0, st>>>((int64_t)p->N * p->N * K, bbar, r, p->ls_norm);
  after_launch("loss_norm", st, 2.0 * n, (double)n * sizeof(T) * 3.0, 0);
  if (grad) {
    const unsigned blocks = (unsigned)((cells + kWarps - 1) / kWarps);
    prof_begin(st, "loss_adjoint");
    atfps_adjoint_kernel<T><<<blocks, 32 * kWarps, sizeof(T) * kWarps * 4 * Md, st>>>(
        p->B, p->N, Md, p->nmat, p->tf_mat, p->at_sel, f64 ? (const T*)p->tf_L64 : (const T*)p->tf_L32,
        f64 ? (const T*)p->tf_fac64 : (const T*)p->tf_fac32, f64 ? (const T*)p->at_P64 : (const T*)p->at_P32,
        p->at_row, p->at_dirs, r, p->ls_norm, alpha);  // (alpha is dead: reused for the coefficient gradient)
    after_launch("loss_adjoint", st, (double)cells * (4.0 * 2.0 * K * Md + 2.0 * K * Md), (double)n * sizeof(T) * 2.0, 0);
    prof_begin(st, "loss_fit_adjoint");
    fit_adjoint_kernel<T><<<blocks, 32 * kWarps, 0, st>>>(cells, Md, p->tf_mat, dp_of<T>(p), alpha, u);
    after_launch("loss_fit_adjoint", st, (double)cells * 2.0 * K * 5.0 * Md, (double)cells * sizeof(T) * 7.0 * Md, 0);
    prof_begin(st, "loss_scatter");
    const int64_t ne = cells * Md;
    scatter_kernel<T><<<(unsigned)std::min<int64_t>((ne + 255) / 256, (int64_t)num_sms() * 16), 256, 0, st>>>(
        p->B, p->N, Md, u, grad);
    after_launch("loss_scatter", st, 0.0, (double)ne * sizeof(T) * 6.0, 0);
  }
  std::vector<double> n2(p->B);
  RTE_CHECK_CUDA(cudaMemcpyAsync(n2.data(), p->ls_norm, sizeof(double) * p->B, cudaMemcpyDeviceToHost, st));
  RTE_CHECK_CUDA(cudaStreamSynchronize(st));
  for (int b = 0; b < p->B; ++b) loss_host[b] = sqrt(n2[b]);
}

template void atfps_fit<float>(const rte_problem*, const float*, float*, cudaStream_t);
template void atfps_fit<double>(const rte_problem*, const double*, double*, cudaStream_t);
template void atfps_loss<float>(const rte_problem*, const float*, double*, float*, cudaStream_t);
template void atfps_loss<double>(const rte_problem*, const double*, double*, double*, cudaStream_t);

}  // namespace rte
