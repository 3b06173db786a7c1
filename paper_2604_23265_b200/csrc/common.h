// Internal declarations shared by the library's translation units (NOT part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/rte.h"

namespace rte {

// ---- error handling -------------------------------------------------------
void set_error(const std::string& msg);
struct Fail {
  rte_status st;
};
#define RTE_CHECK_CUDA(expr)                                                     \
  do {                                                                           \
    cudaError_t e__ = (expr);                                                    \
    if (e__ != cudaSuccess) {                                                    \
      ::rte::set_error(std::string(#expr) + ": " + cudaGetErrorString(e__));     \
      throw ::rte::Fail{RTE_ECUDA};                                              \
    }                                                                            \
  } while (0)
#define RTE_REQUIRE(cond, msg)                                                   \
  do {                                                                           \
    if (!(cond)) {                                                               \
      ::rte::set_error(msg);                                                     \
      throw ::rte::Fail{RTE_EINVAL};                                             \
    }                                                                            \
  } while (0)
// Launch bookkeeping.  prof_begin(st) goes right before a kernel launch, after_launch right
// after it: it checks the launch, counts it and -- when per-launch timing is on
// (rte_timing_enable) -- records a CUDA-event pair on the launching stream together with the
// launch's ALGORITHMIC flops and bytes (DESIGN.md §5 gives the per-unit figures).
// kind: 0 HBM-bound streaming, 1 3xTF32 tensor-core contraction, 2 fp32 SIMT contraction,
//       3 fp64 SIMT, 4 tiny/latency (Givens etc.).
// cls = the launch's timing class (the name after_launch will book); with a class filter set
// (rte_timing_filter), only launches whose class starts with it are timed.
void prof_begin(cudaStream_t st, const char* cls = nullptr);
void after_launch(const char* what, cudaStream_t st = 0, double flops = 0.0, double bytes = 0.0, int kind = 4);

template <typename T>
T* dalloc(size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  cudaError_t e = cudaMalloc(&p, n * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error(std::string("cudaMalloc failed: ") + cudaGetErrorString(e));
    throw Fail{RTE_ENOMEM};
  }
  return static_cast<T*>(p);
}
void dfree(void* p);
template <typename T>
void upload(T* d, const T* h, size_t n) {
  RTE_CHECK_CUDA(cudaMemcpy(d, h, n * sizeof(T), cudaMemcpyHostToDevice));
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int num_sms();

#ifdef __CUDACC__
// One output of the operator (PAPER.md:91-93 eq:DORTE_2d, upwind stencil R9) from the cell's psi,
// its two upwind neighbours nx, ny (0 outside the grid), the centre c = psi_{cell, 0} and the
// centred contraction v = [S (psi - c)]_m (S row-stochastic, R5):
//   (A psi)_m = a_x (psi - nx) + a_y (psi - ny) + (sigma_t - sigma_s) psi + sigma_s ((psi - c) - v)
// This is eq:DORTE_2d rearranged exactly (sigma_t psi - sigma_s S psi = (sigma_t - sigma_s) psi +
// sigma_s (psi - S psi), S psi = c + v), with sigma_t - sigma_s = eps sigma_a (sd) taken from the
// host in fp64.  Written this way no product of sigma_t ~ 1/eps with psi is ever formed, so in the
// diffusive regime (sigma_t ~ 1e2..1e6, eps sigma_a ~ 1e-3) nothing cancels at the scale of
// sigma_t psi; the rounding error scales with the terms that survive.
template <typename T>
__host__ __device__ __forceinline__ T stencil_diag(T ax, T ay, T sd, T ss, T psi, T nx, T ny, T c, T v) {
  return fma(ax, psi - nx, fma(ay, psi - ny, fma(sd, psi, ss * ((psi - c) - v))));
}
#endif

}  // namespace rte

// ---- problem ----------------------------------------------------------------
struct rte_problem {
  int B, N, M;        // M: unknowns per cell (directions; 2 x directions for a TFPS problem)
  int64_t ncell;      // B*N*N
  int64_t n;          // ncell*M
  // host copies (fp64)
  std::vector<double> c, s, zeta, w;
  std::vector<double> S;   // [B][M][M] row-stochastic K W
  std::vector<float> h_eps, h_sa;  // [B][N][N] eps and sigma_a as given (rte_set_source)
  // device
  float* sig_t = nullptr;   // [B][N][N]  sigma_T / eps
  float* sig_s = nullptr;   //            sigma_T / eps - eps sigma_a
  float* sig_d = nullptr;   //            sigma_t - sigma_s = eps sigma_a (stencil_diag)
  double* sig_d64 = nullptr;
  float* f = nullptr;
  double* sig_t64 = nullptr;
  double* sig_s64 = nullptr;
  float* S32 = nullptr;     // [B][M][M]  S[m][n]   (row m, n contiguous)  = GEMM B operand N x K, K-major
  float* St32 = nullptr;    // [B][M][M]  S^T[n][m] (for the SIMT path)
  double* St64 = nullptr;   // [B][M][M]  S^T fp64
  float* S_hi = nullptr;    // [B][M][M]  tf32 hi of S[m][n]
  float* S_lo = nullptr;    // [B][M][M]  tf32 lo
  float* ax = nullptr;      // [M]  |c_m|/h  (fp32)
  float* ay = nullptr;      // [M]  |s_m|/h
  double* ax64 = nullptr;
  double* ay64 = nullptr;
  int8_t* sgx = nullptr;    // [M]  sign(c_m)
  int8_t* sgy = nullptr;    // [M]  sign(s_m)
  float* inflow = nullptr;  // [B][4][N][M]
  bool tc_apply = false;    // tensor-core apply path available for this M
  mutable void* tc_state = nullptr;  // lazily created TMA descriptors etc.
  mutable double* scratch64 = nullptr;  // small device scratch
  // block-Jacobi inverse cell blocks [ncell][M][M] (blockjacobi.cu; built on first use)
  mutable double* bj64 = nullptr;
  mutable float* bj32 = nullptr;
  // ---- TFPS alpha-space problem (kind 1, rte_setup_tfps; tfps.cu).  Md = directions, M = 2 Md.
  int kind = 0;             // 0: psi-space DO operator, 1: TFPS alpha-space operator
  int Md = 0;
  int nmat = 0;
  int* tf_mat = nullptr;    // [B][N][N] material index
  float* tf_L32 = nullptr;  // [nmat][Md][2Md] eigenvectors (columns)
  double* tf_L64 = nullptr;
  float* tf_fac32 = nullptr;  // [nmat][5][2Md] basis factors at faces L, R, B, T and the centre
  double* tf_fac64 = nullptr;
  float* tf_chis32 = nullptr;  // [B][N][N] particular solution f / (sigma_t - sigma_s)
  double* tf_chis64 = nullptr;
  std::vector<double> tf_xi;   // host copies: [nmat][2Md], [nmat][Md][2Md]
  std::vector<double> tf_Lh;
  // ---- ATFPS compressed system (kind 2, rte_setup_atfps; tfps.cu).  Padded [cells][2Md] layout.
  double at_delta = 0.0;
  int64_t at_dim = 0;           // selected unknowns (the compressed dimension)
  uint8_t* at_sel = nullptr;    // [nmat][2Md] mode kept (eq:def_V_delta)
  float* at_P32 = nullptr;      // interface projections: interior [2][nmat][nmat][Md][Md], then
  double* at_P64 = nullptr;     //   boundary [4][nmat][Md/2][Md/2]
  int* at_row = nullptr;        // P-row of each (side, mode): interior [2][nmat][nmat][2][2Md], boundary [4][nmat][2][2Md]
  int* at_dirs = nullptr;       // [4][Md/2] incoming directions of the faces L, R, B, T
  float* at_tmp32 = nullptr;    // [n] full coefficients (layer reconstruction scratch)
  double* at_tmp64 = nullptr;
  // ---- filtered loss (NEXT-4, loss.cu; built on the first rte_atfps_loss / rte_atfps_fit call)
  mutable float* ls_Dp32 = nullptr;   // [nmat][2Md][5Md] D_delta fit operators (R43)
  mutable double* ls_Dp64 = nullptr;
  mutable void* ls_ws = nullptr;      // scratch: alpha, residual, b_bar (n each), fit adjoint [cells][5Md]
  mutable size_t ls_ws_bytes = 0;
  mutable double* ls_norm = nullptr;  // [B] ||r||^2 per sample
};

// ---- kernel launchers (apply.cu) --------------------------------------------
namespace rte {
void launch_rhs(const rte_problem* p, float* b, cudaStream_t st);
// y = alpha * A x  (alpha scales the input, i.e. A(alpha x)); alpha_dev may be NULL (1).
void launch_apply_f32(const rte_problem* p, const float* x, float* y, const double* alpha_dev,
                      int alpha_stride, cudaStream_t st);
// y = A x (fp64); if b != NULL: y = b - A x.
void launch_apply_f64(const rte_problem* p, const double* x, double* y, const float* b, cudaStream_t st);
bool apply_tc_supported(int M);
// block Jacobi (blockjacobi.cu): y = A_cc^{-1} (alpha x) per cell; builds the blocks on first use
void bj_prepare(const rte_problem* p);
template <typename T>
void bj_apply(const rte_problem* p, const T* x, T* y, const double* alpha, int alpha_stride, cudaStream_t st);
double apply_flops(const rte_problem* p);
double apply_bytes(const rte_problem* p, int elt, int b_elt);
void free_tc_state(rte_problem* p);
void free_gmres_work(const rte_problem* p);
// CUDA-graph capture support (krylov.cu caches one graph per Arnoldi step): while capturing,
// prof_begin records nothing and marks the capture unusable if it would have timed a launch.
void capture_begin();
bool capture_end();
int64_t launches_now();
void launches_add(int64_t d);
std::vector<std::string> capture_classes();                      // timing classes captured so far
bool prof_wants_any(const std::vector<std::string>& classes);    // timing would record one of them
void drop_net_graphs(const struct ::mgnet_net* net);  // (krylov.cu) forget graphs using `net`
void launch_apply_tc(const rte_problem* p, const float* x, float* y, const double* alpha_dev,
                     int alpha_stride, cudaStream_t st);
// TFPS alpha-space operator (tfps.cu, tfps_setup.cpp)
template <typename T>
void launch_tfps_apply(const rte_problem* p, const T* x, T* y, const double* alpha_dev, int alpha_stride,
                       const float* b, cudaStream_t st);
void launch_tfps_rhs(const rte_problem* p, float* b, cudaStream_t st);
template <typename T>
void launch_tfps_reconstruct(const rte_problem* p, const T* alpha, T* psi, cudaStream_t st);
void tfps_local_modes(const double* S, const std::vector<double>& c, const std::vector<double>& s, double gamma,
                      std::vector<double>& xi, std::vector<double>& L);
void tfps_face_factors(const std::vector<double>& xi, int M, double sigma_t, double h, double* fac);
void atfps_interface(const std::vector<double>& Lh, const std::vector<uint8_t>& sel, int M, int a, int b, int fm,
                     int fp, const std::vector<int>& dirs, std::vector<double>& P, int* rowmap);
template <typename T>
void launch_atfps(const rte_problem* p, int mode, const T* x, T* y, const double* alpha_dev, int alpha_stride,
                  const float* b, cudaStream_t st);  // mode 0: A x (y = b - A x if b), 1: rhs (T = float), 2: layer
// filtered loss (NEXT-4, loss.cu, tfps_setup.cpp)
void atfps_fit_pinv(const double* L, const double* fac, const uint8_t* sel, int M, double* Dp);
template <typename T>
void atfps_fit(const rte_problem* p, const T* psi, T* alpha, cudaStream_t st);
template <typename T>
void atfps_loss(const rte_problem* p, const T* psi, double* loss_host, T* grad, cudaStream_t st);
}  // namespace rte
