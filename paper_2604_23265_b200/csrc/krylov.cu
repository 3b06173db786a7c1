// Restarted right-preconditioned GMRES(m) on the device (
// DESIGN.md R21, R22).  Host C++ drives the loop; every vector operation runs in the kernels
// below.  Design:
//  - Krylov basis V in float32, stored UNNORMALISED: column i holds alpha_i^{-1} v_i, with the
//    per-sample scale alpha_i kept in fp64 on the device.  Consumers (V-cycle lift, apply input,
//    dots, updates, combination) fold alpha_i in, so no separate normalisation pass is needed.
//  - Classical Gram-Schmidt with re-orthogonalisation (CGS2) in three fused streaming passes:
//      A: h1 = alpha V^T w;   B: v' = w - V (alpha h1) and h2 = alpha V^T v', ||v'||^2;
//      C: v'' = v' - V (alpha h2) and ||v''||^2.
//    Every dot product accumulates in fp64 with a deterministic (fixed-order) two-level reduction
//    (warp shuffles -> per-block partials -> last-block finalisation).
//  - Givens rotations, least squares and the convergence decision run in tiny per-sample device
//    kernels; the host reads one 32-byte status record per sample per iteration.
//  - The iterate x is float64 and every restart recomputes r = b - A x in float64.
#include <math.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <type_traits>
#include <vector>

#include "common.h"
#include "mgnet.h"

namespace rte {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxRestart = 64;     // array bound of the per-sample device scratch
constexpr int kMaxRestartApi = 32;  // restart range accepted by the API (the fused CGS kernels' NV)

struct RedArgs {
  double* partials;   // [B][nblk][nq]
  unsigned* counters; // [B]
  double* out;        // [B][out_ld]
  int out_ld;
  int nblk;
};

// Block-reduce NQ doubles per thread, write partials, last block finalises (fixed order).
// scale_q (may be NULL) multiplies quantity q at finalisation.
template <int NQ>
__device__ void reduce_finalize(double (&acc)[NQ], const RedArgs& ra, int b, const double* scale, int nscale) {
  __shared__ double red[kThreads / 32][NQ > 0 ? NQ : 1];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    double v = acc[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][q] = v;
  }
  __syncthreads();
  double* part = ra.partials + ((int64_t)b * ra.nblk + blockIdx.x) * NQ;
  for (int q = threadIdx.x; q < NQ; q += blockDim.x) {
    double v = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) v += red[w][q];
    part[q] = v;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned prev = atomicAdd(ra.counters + b, 1u);
    last = (prev == (unsigned)ra.nblk - 1);
  }
  __syncthreads();
  if (last) {
    __threadfence();
    const double* pb = ra.partials + (int64_t)b * ra.nblk * NQ;
    for (int q = threadIdx.x; q < NQ; q += blockDim.x) {
      double v = 0.0;
      for (int k = 0; k < ra.nblk; ++k) v += ((volatile const double*)pb)[(int64_t)k * NQ + q];
      if (scale && q < nscale) v *= scale[q];
      ra.out[(int64_t)b * ra.out_ld + q] = v;
    }
    if (threadIdx.x == 0) ra.counters[b] = 0u;
  }
}

// 16-byte vector of the basis element type (float4 for the fp32 basis, double2 for fp64).
template <typename T> struct Vec16;
template <> struct Vec16<float> { using type = float4; };
template <> struct Vec16<double> { using type = double2; };

// One CGS pass over NV basis vectors (see file header).  T = basis element type.
//  UPDATE: dst = src - sum_i (hin_i alpha_i) V_i   (else dst = src, not written)
//  DOTS  : out[i] = alpha_i <V_i, dst>, i < NV ;  always out[NV] = ||dst||^2
template <typename T, int NV, bool UPDATE, bool DOTS>
__global__ void __launch_bounds__(kThreads, 1) cgs_kernel(
    const T* __restrict__ V, int64_t vld, const double* __restrict__ alpha, int alpha_ld,
    const double* __restrict__ hin, int hin_ld, const T* src, T* dst, int64_t ns,
    const int* __restrict__ active, RedArgs ra, const double* __restrict__ sel_w2,
    const double* __restrict__ sel_v2) {
  using VT = typename Vec16<T>::type;
  constexpr int W = (int)(sizeof(VT) / sizeof(T));
  constexpr int NQ = (DOTS ? NV : 0) + 1;
  const int b = blockIdx.y;
  if (active && !active[b]) return;
  // selective re-orthogonalisation (DGKS, "twice is enough"): this second pass runs only when
  // ||v'||^2 < ||w||^2 / 2 (both from the previous passes); otherwise v' already is v_{j+1}
  if (sel_w2 && !(sel_v2[(int64_t)b * hin_ld] < 0.5 * sel_w2[(int64_t)b * hin_ld])) return;
  __shared__ T coef[NV > 0 ? NV : 1];
  if (UPDATE) {
    for (int i = threadIdx.x; i < NV; i += blockDim.x)
      coef[i] = (T)(hin[(int64_t)b * hin_ld + i] * alpha[(int64_t)b * alpha_ld + i]);
    __syncthreads();
  }
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  const int64_t nv = ns / W;
  const VT* s4 = reinterpret_cast<const VT*>(src + (int64_t)b * ns);
  VT* d4 = reinterpret_cast<VT*>(dst + (int64_t)b * ns);
  const T* Vb = V + (int64_t)b * ns;
  for (int64_t q = (int64_t)blockIdx.x * kThreads + threadIdx.x; q < nv; q += (int64_t)ra.nblk * kThreads) {
    VT sv = s4[q];
    T* s = reinterpret_cast<T*>(&sv);
    VT vv[NV > 0 ? NV : 1];
#pragma unroll
    for (int i = 0; i < NV; ++i) vv[i] = reinterpret_cast<const VT*>(Vb + (int64_t)i * vld)[q];
    if (UPDATE) {
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const T* v = reinterpret_cast<const T*>(&vv[i]);
#pragma unroll
        for (int e = 0; e < W; ++e) s[e] = fma(-coef[i], v[e], s[e]);
      }
      __stcs(d4 + q, sv);  // streaming store: the 256 MiB result cannot stay in L2 for its next reader,
                           // and evict-first keeps it from displacing the read stream (0.92 -> 0.95 of HBM)
    }
    if (DOTS) {
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const T* v = reinterpret_cast<const T*>(&vv[i]);
#pragma unroll
        for (int e = 0; e < W; ++e) acc[i] += (double)v[e] * (double)s[e];
      }
    }
#pragma unroll
    for (int e = 0; e < W; ++e) acc[NQ - 1] += (double)s[e] * (double)s[e];
  }
  reduce_finalize<NQ>(acc, ra, b, DOTS ? alpha + (int64_t)b * alpha_ld : nullptr, DOTS ? NV : 0);
}

// DCGS2 (reorth = 3; delayed classical Gram-Schmidt with re-orthogonalisation): the
// second CGS pass of the candidate q~_j is delayed to step j and fused with the first pass of the new
// vector, so every Arnoldi step streams the basis twice (pass 1: dots; this pass: both updates) --
// CGS1's traffic -- with CGS2's orthogonality.  With NV = j final vectors V_0..V_{j-1}, the
// candidate V_j (first-pass projected at step j-1, not yet re-orthogonalised) and w = A P(q~_j):
//   V_j     <- V_j - sum_{i<j} cA_i V_i                  (the delayed second pass: q_j = alpha_j V_j)
//   V_{j+1} <- w - sum_{i<j} cB_i V_i - cB_j V_j(old)     (first pass of the new vector, times r_j)
// and the next step's re-orthogonalisation dots: out[i] = alpha_i <V_i, V_{j+1}> for i <= j (V_j the
// corrected one, alpha_j its final scale), out[j+1] = ||V_{j+1}||^2.  Coefficients: dcgs_coef_kernel.
template <typename T, int NV>
__global__ void __launch_bounds__(kThreads, 1) dcgs_update_kernel(
    T* V, int64_t vld, const double* __restrict__ alpha, int alpha_ld, const double* __restrict__ cA,
    const double* __restrict__ cB, int c_ld, const T* __restrict__ w, int64_t ns, const int* __restrict__ active,
    RedArgs ra) {
  using VT = typename Vec16<T>::type;
  constexpr int W = (int)(sizeof(VT) / sizeof(T));
  constexpr int NQ = NV + 2;
  const int b = blockIdx.y;
  if (active && !active[b]) return;
  __shared__ T sA[NV > 0 ? NV : 1];
  __shared__ T sB[NV + 1];
  for (int i = threadIdx.x; i <= NV; i += blockDim.x) {
    if (i < NV) sA[i] = (T)cA[(int64_t)b * c_ld + i];
    sB[i] = (T)cB[(int64_t)b * c_ld + i];
  }
  __syncthreads();
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  const int64_t nv = ns / W;
  T* Vb = V + (int64_t)b * ns;
  VT* vj4 = reinterpret_cast<VT*>(Vb + (int64_t)NV * vld);
  VT* vn4 = reinterpret_cast<VT*>(Vb + (int64_t)(NV + 1) * vld);
  const VT* w4 = reinterpret_cast<const VT*>(w + (int64_t)b * ns);
  for (int64_t q = (int64_t)blockIdx.x * kThreads + threadIdx.x; q < nv; q += (int64_t)ra.nblk * kThreads) {
    VT wv = w4[q];
    VT jv = vj4[q];
    VT vv[NV > 0 ? NV : 1];
#pragma unroll
    for (int i = 0; i < NV; ++i) vv[i] = reinterpret_cast<const VT*>(Vb + (int64_t)i * vld)[q];
    T* wn = reinterpret_cast<T*>(&wv);
    T* jn = reinterpret_cast<T*>(&jv);
#pragma unroll
    for (int e = 0; e < W; ++e) wn[e] = fma(-sB[NV], jn[e], wn[e]);  // (uses the candidate before its correction)
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const T* v = reinterpret_cast<const T*>(&vv[i]);
#pragma unroll
      for (int e = 0; e < W; ++e) {
        jn[e] = fma(-sA[i], v[e], jn[e]);
        wn[e] = fma(-sB[i], v[e], wn[e]);
      }
    }
    if (NV > 0) vj4[q] = jv;
    __stcs(vn4 + q, wv);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const T* v = reinterpret_cast<const T*>(&vv[i]);
#pragma unroll
      for (int e = 0; e < W; ++e) acc[i] += (double)v[e] * (double)wn[e];
    }
#pragma unroll
    for (int e = 0; e < W; ++e) {
      acc[NV] += (double)jn[e] * (double)wn[e];
      acc[NV + 1] += (double)wn[e] * (double)wn[e];
    }
  }
  reduce_finalize<NQ>(acc, ra, b, alpha + (int64_t)b * alpha_ld, NV + 1);
}

// DCGS2 step-j coefficients (per sample, fp64), between pass 1 and dcgs_update_kernel.  Inputs:
//   a[i] = alpha_i <V_i, V_j>, i < j  (q_i . V_j, from the previous step's update pass; a[j] = ||V_j||^2)
//   z[i] = alpha_i <V_i, w>, i <= j   (pass 1; alpha_j = alpha~_j = 1/||V_j||, so z_j = q~_j . w)
// With s_i = q_i . q~_j = a_i alpha~_j and r = ||q~_j - sum s_i q_i|| = sqrt(1 - |s|^2):
//   q_j = (q~_j - sum_{i<j} s_i q_i) / r                       (the delayed re-orthogonalisation)
//   column j-1 of H becomes exact for q_j: h_{i,j-1} += h_{j,j-1} s_i, h_{j,j-1} *= r
//   A P q_j = (w - Q_j c) / r with c = H[0..j][0..j-1] s      (Arnoldi relation A P Q_{j-1} = Q_j H)
//   h_{i,j} = (z_i - c_i) / r (i < j),  h_{j,j} = ((z_j - s.z) / r - c_j) / r
//   V_{j+1} = r w~ = w - Q_j d,  d = c + r h_{.,j}               (w~: first-pass projection of A P q_j)
// expressed on the stored vectors (cA: V_j's correction, cB: V_{j+1}'s projection).  Writes the final
// alpha_j = alpha~_j / r, column j of the unrotated H (Hc, also hcol for the Givens kernel) and r.
__global__ void __launch_bounds__(32) dcgs_coef_kernel(int B, int j, int m, const double* __restrict__ a,
                                                       const double* __restrict__ z, int hld, double* Hc,
                                                       double* alpha, int alpha_ld, double* cA, double* cB,
                                                       double* hcol, double* rbuf, const int* __restrict__ active) {
  // one warp per sample; lane i owns row i of the column (j <= 31 < 32 lanes, restart <= 32)
  const int b = blockIdx.x, i = threadIdx.x;
  if (b >= B || !active[b]) return;
  __shared__ double s_sh[32];
  double* H = Hc + (int64_t)b * (m + 1) * m;  // [m+1][m]
  double* al = alpha + (int64_t)b * alpha_ld;
  const double* ab = a + (int64_t)b * hld;
  const double* zb = z + (int64_t)b * hld;
  const double at = al[j];
  const double si = i < j ? ab[i] * at : 0.0;
  const double zi = i <= j ? zb[i] : 0.0;
  const double ali = i < j ? al[i] : 0.0;
  s_sh[i] = si;
  double ss = si * si, sz = si * zi;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    sz += __shfl_xor_sync(0xffffffffu, sz, o);
  }
  const double r = sqrt(fmax(1.0 - ss, 1e-300));
  if (j > 0) {
    const double hl = H[j * m + (j - 1)];
    if (i < j) H[i * m + (j - 1)] += hl * si;
    __syncwarp();
    if (i == j) H[j * m + (j - 1)] = hl * r;
  }
  __syncwarp();
  double ci = 0.0;
  if (i <= j)
    for (int k = (i > 0 ? i - 1 : 0); k < j; ++k) ci += H[i * m + k] * s_sh[k];  // (upper Hessenberg)
  const double cj = __shfl_sync(0xffffffffu, ci, j);
  const double zj = __shfl_sync(0xffffffffu, zi, j);
  const double hj = ((zj - sz) / r - cj) / r;
  const double dj = cj + r * hj;
  const double hi_ = i < j ? (zi - ci) / r : hj;
  double* cAb = cA + (int64_t)b * hld;
  double* cBb = cB + (int64_t)b * hld;
  if (i < j) {
    const double di = ci + r * hi_;
    cAb[i] = si * ali / at;
    cBb[i] = (di - dj * si / r) * ali;
  }
  if (i <= j) {
    hcol[(int64_t)b * hld + i] = hi_;
    H[i * m + j] = hi_;
  }
  if (i == j) {
    cBb[j] = dj * at / r;
    al[j] = at / r;
    rbuf[b] = r;
  }
}

// DCGS2 cycle end (per sample): finalise the last column k-1 with the re-orthogonalisation dots of the
// candidate q~_k (the last update pass computed them), then QR of the unrotated H[0..k][0..k-1] by
// Givens rotations, y = R^{-1} (beta e_1) and coef_i = y_i alpha_i.
__global__ void dcgs_backsolve_kernel(int B, int m, double* Hc, const double* __restrict__ a, int hld,
                                      const double* __restrict__ alpha, int alpha_ld, const int* __restrict__ kcols,
                                      const int* __restrict__ brk, double* coef, int coef_ld) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int k = kcols[b];
  if (k <= 0) return;
  double* H = Hc + (int64_t)b * (m + 1) * m;
  const double* al = alpha + (int64_t)b * alpha_ld;
  const double* ab = a + (int64_t)b * hld;
  const double n2 = ab[k];
  if (!brk[b] && n2 > 0.0) {
    const double at = 1.0 / sqrt(n2);
    double ss = 0.0, s[kMaxRestart + 1];
    for (int i = 0; i < k; ++i) {
      s[i] = ab[i] * at;
      ss += s[i] * s[i];
    }
    const double hl = H[k * m + (k - 1)];
    for (int i = 0; i < k; ++i) H[i * m + (k - 1)] += hl * s[i];
    H[k * m + (k - 1)] = hl * sqrt(fmax(1.0 - ss, 1e-300));
  }
  double R[kMaxRestart + 1][kMaxRestart];
  double g[kMaxRestart + 1];
  for (int i = 0; i <= k; ++i) {
    g[i] = 0.0;
    for (int l = 0; l < k; ++l) R[i][l] = H[i * m + l];
  }
  g[0] = 1.0 / al[0];  // beta = ||r|| (alpha_0 = 1/beta; r_0 = 1 keeps it)
  for (int l = 0; l < k; ++l) {
    const double x = R[l][l], yv = R[l + 1][l];
    const double den = hypot(x, yv);
    const double cs = den > 0 ? x / den : 1.0, sn = den > 0 ? yv / den : 0.0;
    for (int q = l; q < k; ++q) {
      const double t = cs * R[l][q] + sn * R[l + 1][q];
      R[l + 1][q] = -sn * R[l][q] + cs * R[l + 1][q];
      R[l][q] = t;
    }
    g[l + 1] = -sn * g[l];
    g[l] = cs * g[l];
  }
  double y[kMaxRestart];
  for (int i = k - 1; i >= 0; --i) {
    double t = g[i];
    for (int l = i + 1; l < k; ++l) t -= R[i][l] * y[l];
    y[i] = t / R[i][i];
  }
  for (int i = 0; i < k; ++i) coef[(int64_t)b * coef_ld + i] = y[i] * al[i];
}

// ||x||^2 per sample (x fp32 or fp64); optionally writes xo = (TO)x.
template <typename T, typename TO>
__global__ void __launch_bounds__(kThreads) norm_kernel(const T* __restrict__ x, TO* __restrict__ xo, int64_t ns,
                                                         RedArgs ra) {
  // 4 elements per thread per trip, all loads issued first (bytes in flight for the HBM stream;
  // ns % 4 == 0 since M % 4 == 0)
  const int b = blockIdx.y;
  double acc[1] = {0.0};
  const T* xb = x + (int64_t)b * ns;
  TO* xob = xo ? xo + (int64_t)b * ns : nullptr;
  const int64_t n4 = ns / 4;
  for (int64_t q = (int64_t)blockIdx.x * kThreads + threadIdx.x; q < n4; q += (int64_t)ra.nblk * kThreads) {
    double v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = (double)xb[4 * q + i];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[0] += v[i] * v[i];
    if (xob)
#pragma unroll
      for (int i = 0; i < 4; ++i) xob[4 * q + i] = (TO)v[i];
  }
  reduce_finalize<1>(acc, ra, b, nullptr, 0);
}

// acc += sum_{u < U} cs[i+u] V_{i+u}[q]: all U 16-byte loads issued before the first FMA.
template <int U, typename T, typename VT, int W>
__device__ __forceinline__ void combine_cols(double (&acc)[W], const T* __restrict__ Vb, int64_t vld, int64_t q,
                                             const double* cs, int i) {
  VT v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) v[u] = __ldg(reinterpret_cast<const VT*>(Vb + (int64_t)(i + u) * vld) + q);
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const T* x = reinterpret_cast<const T*>(&v[u]);
#pragma unroll
    for (int e = 0; e < W; ++e) acc[e] += cs[i + u] * (double)x[e];
  }
}

// dst = sum_{i < k_b} coef_i V_i   (coef already includes alpha), fp64 accumulation; 16-byte
// vector loads of every basis column (the k_b columns stream once at HBM rate).
template <typename T, typename TO>
__global__ void __launch_bounds__(kThreads) combine_kernel(const T* __restrict__ V, int64_t vld,
                                                            const double* __restrict__ coef, int coef_ld,
                                                            const int* __restrict__ kcols, TO* __restrict__ dst,
                                                            int64_t ns, int nblk) {
  static_assert(sizeof(TO) == sizeof(T), "combine stores in the basis type");
  using VT = typename Vec16<T>::type;
  constexpr int W = (int)(sizeof(VT) / sizeof(T));
  const int b = blockIdx.y;
  const int k = kcols[b];
  __shared__ double cs[kMaxRestart + 1];
  for (int i = threadIdx.x; i < k; i += blockDim.x) cs[i] = coef[(int64_t)b * coef_ld + i];
  __syncthreads();
  const T* Vb = V + (int64_t)b * ns;
  const int64_t nv = ns / W;
  for (int64_t q = (int64_t)blockIdx.x * kThreads + threadIdx.x; q < nv; q += (int64_t)nblk * kThreads) {
    double acc[W];
#pragma unroll
    for (int e = 0; e < W; ++e) acc[e] = 0.0;
    int i = 0;
    for (; i + 8 <= k; i += 8) combine_cols<8, T, VT, W>(acc, Vb, vld, q, cs, i);  // 8 columns in flight
    if (i + 4 <= k) {
      combine_cols<4, T, VT, W>(acc, Vb, vld, q, cs, i);
      i += 4;
    }
    for (; i < k; ++i) combine_cols<1, T, VT, W>(acc, Vb, vld, q, cs, i);
    VT o;  // TO == T at every call site: one 16-byte store
    T* ov = reinterpret_cast<T*>(&o);
#pragma unroll
    for (int e = 0; e < W; ++e) ov[e] = (T)acc[e];
    reinterpret_cast<VT*>(dst + (int64_t)b * ns)[q] = o;
  }
}

// x += z (+ q)  for samples with kcols > 0 (z fp32 or fp64; q optional fp32).
template <typename TZ>
__global__ void axpy64_kernel(double* __restrict__ x, const TZ* __restrict__ z, const float* __restrict__ q,
                              const int* __restrict__ kcols, int64_t ns, int nblk) {
  const int b = blockIdx.y;
  if (kcols[b] <= 0) return;
  const int64_t n4 = ns / 4;  // 4 elements per thread per trip, loads first
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n4; e += (int64_t)nblk * blockDim.x) {
    const int64_t o = (int64_t)b * ns + 4 * e;
    double xv[4], zv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      xv[i] = x[o + i];
      zv[i] = (double)z[o + i] + (q ? (double)q[o + i] : 0.0);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) x[o + i] = xv[i] + zv[i];
  }
}

// fp64 mode: z64 = alpha_j V64_j and z32 = (float) z64 (the V-cycle's input).
__global__ void scale_f64_kernel(const double* __restrict__ v, const double* __restrict__ alpha, int alpha_ld,
                                 double* __restrict__ z64, float* __restrict__ z32, int64_t ns, int nblk) {
  const int b = blockIdx.y;
  const double a = alpha[(int64_t)b * alpha_ld];
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ns; e += (int64_t)nblk * blockDim.x) {
    const int64_t o = (int64_t)b * ns + e;
    const double t = a * v[o];
    z64[o] = t;
    if (z32) z32[o] = (float)t;
  }
}

// fp64 mode: z64 += q32 (the V-cycle's correction V(z)); z32 = (float) z64 when `to32`.
__global__ void add_f32_to_f64_kernel(double* __restrict__ z64, const float* __restrict__ q, float* __restrict__ z32,
                                      int64_t n) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    if (q) z64[e] += (double)q[e];
    if (z32) z32[e] = (float)z64[e];
  }
}

struct Status {      // per-sample record read by the host each iteration (32 bytes)
  double est;        // |g_{j+1}| / ||b||   (or true relres at cycle start)
  int active;        // still iterating in this cycle
  int breakdown;     // lucky breakdown happened at this step
  int kcols;         // Krylov columns usable at cycle end
  int converged;     // (cycle start) true residual <= rtol ||b||
  int pad[2];
};

// Cycle start: beta = ||r||, alpha_0 = 1/beta, g = beta e_1, convergence by the true residual.
__global__ void cycle_init_kernel(int B, const double* __restrict__ rnorm2, const double* __restrict__ bnorm,
                                  double rtol, int stop_all, double* alpha, int alpha_ld, double* g, int g_ld,
                                  int* active, int* kcols, const int* done, Status* st) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  double beta = sqrt(fmax(rnorm2[b], 0.0));
  double rel = bnorm[b] > 0 ? beta / bnorm[b] : 0.0;
  int conv = (beta <= rtol * bnorm[b]);
  int act = (!conv && !stop_all && !done[b]) ? 1 : 0;
  active[b] = act;
  kcols[b] = 0;
  alpha[(int64_t)b * alpha_ld] = beta > 0 ? 1.0 / beta : 0.0;
  for (int i = 0; i < g_ld; ++i) g[(int64_t)b * g_ld + i] = 0.0;
  g[(int64_t)b * g_ld] = beta;
  st[b].est = rel;
  st[b].active = act;
  st[b].breakdown = 0;
  st[b].kcols = 0;
  st[b].converged = conv;
}

// Givens update of column j (per sample).  h1/h2: pass outputs ([.., j] dots, [j+1] = ||.||^2).
__global__ void givens_kernel(int B, int j, int m, const double* __restrict__ h1, const double* __restrict__ h2,
                              int h_ld, const double* __restrict__ nrm2, int nrm_ld, int selective, double* Hr, double* Hraw,
                              int save_raw, double* cs, double* sn, double* g, double* alpha, int alpha_ld,
                              const double* __restrict__ bnorm, double rtol, int last, int* active, int* kcols,
                              Status* st, const double* __restrict__ hcol, const double* __restrict__ rbuf,
                              int* brkd) {
  // hcol != NULL: DCGS2 (reorth = 3): column j comes from dcgs_coef_kernel, h2[j+1] = ||V_{j+1}||^2 from
  // the update pass, and h_{j+1,j} = ||V_{j+1}|| / r_j (V_{j+1} = r_j w~)
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  if (!active[b]) {
    st[b].active = 0;
    st[b].breakdown = 0;
    return;
  }
  // selective mode: the re-orthogonalisation pass ran iff ||v'||^2 < ||w||^2 / 2 (h1[j+1] = ||w||^2,
  // h2[j+1] = ||v'||^2); without it the column is h1 and h_{j+1,j} = ||v'||
  bool use_h2 = h2 != nullptr;
  const double* nr = nrm2 + (int64_t)b * nrm_ld;
  if (selective) {
    use_h2 = h2[(int64_t)b * h_ld + j + 1] < 0.5 * h1[(int64_t)b * h_ld + j + 1];
    if (!use_h2) nr = h2 + (int64_t)b * h_ld + j + 1;
  }
  double col[kMaxRestart + 1];
  double dc_r = 1.0;
  if (hcol) {
    nr = h2 + (int64_t)b * h_ld + j + 1;
    dc_r = rbuf[b];
    use_h2 = false;
  }
  bool finite = isfinite(*nr) && isfinite(dc_r);
  for (int i = 0; i <= j; ++i) {
    col[i] = hcol ? hcol[(int64_t)b * h_ld + i]
                  : h1[(int64_t)b * h_ld + i] + (use_h2 ? h2[(int64_t)b * h_ld + i] : 0.0);
    finite = finite && isfinite(col[i]);
  }
  if (!finite) {
    // NaN/Inf guard: a non-finite Arnoldi column (an operator or preconditioner that produced
    // NaN/Inf) stops the sample before anything of this step is applied; the cycle-end update
    // uses the j finite columns before it (breakdown = 2, gmres_solve returns RTE_ENUMERIC)
    active[b] = 0;
    kcols[b] = j;
    brkd[b] = 2;
    st[b].est = NAN;
    st[b].active = 0;
    st[b].breakdown = 2;
    st[b].kcols = j;
    return;
  }
  const double vn = sqrt(fmax(*nr, 0.0));
  double hj1 = vn / dc_r;
  const int ldh = m;  // H stored [B][m+1][m]
  double* Hb = Hr + (int64_t)b * (m + 1) * m;
  if (hcol) {
    Hraw[(int64_t)b * (m + 1) * m + (j + 1) * ldh + j] = hj1;  // (rows 0..j: dcgs_coef_kernel)
  } else if (save_raw) {
    double* R = Hraw + (int64_t)b * (m + 1) * m;
    for (int i = 0; i <= j; ++i) R[i * ldh + j] = col[i];
    R[(j + 1) * ldh + j] = hj1;
  }
  double* csb = cs + (int64_t)b * m;
  double* snb = sn + (int64_t)b * m;
  for (int i = 0; i < j; ++i) {
    double t = csb[i] * col[i] + snb[i] * col[i + 1];
    col[i + 1] = -snb[i] * col[i] + csb[i] * col[i + 1];
    col[i] = t;
  }
  double den = hypot(col[j], hj1);
  double c = den > 0 ? col[j] / den : 1.0, s = den > 0 ? hj1 / den : 0.0;
  csb[j] = c;
  snb[j] = s;
  for (int i = 0; i < j; ++i) Hb[i * ldh + j] = col[i];
  Hb[j * ldh + j] = den;
  double* gb = g + (int64_t)b * (m + 1);
  gb[j + 1] = -s * gb[j];
  gb[j] = c * gb[j];
  double est = fabs(gb[j + 1]) / bnorm[b];
  int brk = (hj1 <= 1e-14 * den) ? 1 : 0;
  alpha[(int64_t)b * alpha_ld + j + 1] = brk ? 0.0 : 1.0 / (hcol ? vn : hj1);
  int stop = brk || (fabs(gb[j + 1]) <= rtol * bnorm[b]) || last || (j + 1 == m);
  if (stop) {
    active[b] = 0;
    kcols[b] = j + 1;
    brkd[b] = brk;  // (how the cycle ended, for the DCGS2 back-solve)
  }
  st[b].est = est;
  st[b].active = !stop;
  st[b].breakdown = brk;
  st[b].kcols = stop ? j + 1 : 0;
}

// y = R^{-1} g (k_b columns) and coef_i = y_i alpha_i.
__global__ void backsolve_kernel(int B, int m, const double* __restrict__ Hr, const double* __restrict__ g,
                                 const double* __restrict__ alpha, int alpha_ld, const int* __restrict__ kcols,
                                 double* coef, int coef_ld) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  int k = kcols[b];
  const double* Hb = Hr + (int64_t)b * (m + 1) * m;
  const double* gb = g + (int64_t)b * (m + 1);
  double y[kMaxRestart];
  for (int i = k - 1; i >= 0; --i) {
    double s = gb[i];
    for (int l = i + 1; l < k; ++l) s -= Hb[i * m + l] * y[l];
    y[i] = s / Hb[i * m + i];
  }
  for (int i = 0; i < k; ++i) coef[(int64_t)b * coef_ld + i] = y[i] * alpha[(int64_t)b * alpha_ld + i];
}

}  // namespace

// ---------------------------------------------------------------------------------------
struct GmresWork {
  int B = 0, m = 0;
  int64_t ns = 0;
  int nblk = 0;
  float* V = nullptr;      // (m+1) x n
  float* w = nullptr;      // n
  float* z = nullptr;      // n
  double* r64 = nullptr;   // n
  double *Hr = nullptr, *Hraw = nullptr, *cs = nullptr, *sn = nullptr, *g = nullptr, *alpha = nullptr;
  double *h1 = nullptr, *h2 = nullptr, *h3 = nullptr, *coef = nullptr, *bnorm = nullptr, *rn2 = nullptr;
  double *cA = nullptr, *cB = nullptr, *hcol = nullptr, *rbuf = nullptr;  // DCGS2 step coefficients
  double* partials = nullptr;
  unsigned* counters = nullptr;
  int *active = nullptr, *kcols = nullptr, *done = nullptr, *brkd = nullptr;
  Status* st_dev = nullptr;
  Status* st_host = nullptr;  // pinned, 2 slots of B (the step statuses are read one step late)
  cudaEvent_t st_ev[2] = {nullptr, nullptr};  // slot copies done
  // fp64-basis mode (gmres_opts.precision = 1), allocated on first use
  double* V64 = nullptr;   // (m+1) x n
  double* w64 = nullptr;
  double* z64 = nullptr;
  float* q32 = nullptr;    // V-cycle output
  // gmres_solve_host, allocated on first use: device copies of b and x, a copy stream, and the
  // events ordering the early device->host copy of x against the solve stream
  float* bh = nullptr;     // n
  double* xh = nullptr;    // n
  cudaStream_t cp = nullptr;
  cudaEvent_t ev_x = nullptr, ev_cp = nullptr;
  // CUDA graphs of the fp32 Arnoldi step's operator part, w = A P(alpha_j V_j) (the preconditioner
  // and the apply: ~90 launches at config 5), one per (net, net epoch, j, precond); every input and
  // output pointer of that part is fixed per j because this workspace is cached per problem
  struct StepGraph {
    cudaGraphExec_t exec = nullptr;  // nullptr: seen once (kernels warmed), not captured yet
    int64_t launches = 0;
    std::vector<std::string> classes;  // timing classes inside
  };
  std::map<std::tuple<const mgnet_net*, uint64_t, int, int>, StepGraph> graphs;
  void drop_graphs(const mgnet_net* only = nullptr) {
    for (auto it = graphs.begin(); it != graphs.end();) {
      if (only && std::get<0>(it->first) != only) {
        ++it;
        continue;
      }
      if (it->second.exec) cudaGraphExecDestroy(it->second.exec);
      it = graphs.erase(it);
    }
  }
  void release() {
    drop_graphs();
    void* ps[] = {V, w, z, r64, Hr, Hraw, cs, sn, g, alpha, h1, h2, h3, coef, bnorm, rn2, cA, cB, hcol, rbuf, partials, counters,
                  active, kcols, done, brkd, st_dev, V64, w64, z64, q32, bh, xh};
    for (void* p : ps) dfree(p);
    if (cp) cudaStreamDestroy(cp);
    if (ev_x) cudaEventDestroy(ev_x);
    if (ev_cp) cudaEventDestroy(ev_cp);
    if (st_host) cudaFreeHost(st_host);
    for (auto& e : st_ev)
      if (e) cudaEventDestroy(e);
    *this = GmresWork();
  }
};

template <typename TB>
static void launch_cgs(const GmresWork& W, const TB* V, int nv, bool update, bool dots, const double* hin,
                       const TB* src, TB* dst, double* out, cudaStream_t st, const double* sel_w2 = nullptr,
                       const double* sel_v2 = nullptr) {
  RedArgs ra{W.partials, W.counters, out, kMaxRestart + 2, W.nblk};
  dim3 grid(W.nblk, W.B);
  const int64_t vld = W.ns * W.B;
  const char* cls = sel_w2 ? "cgs_reorth_selective" : update ? (dots ? "cgs_update_dots" : "cgs_update") : "cgs_dots";
  prof_begin(st, cls);
  auto go = [&](auto nv_tag, auto up_tag, auto dot_tag) {
    constexpr int NV = decltype(nv_tag)::value;
    constexpr bool UP = decltype(up_tag)::value;
    constexpr bool DT = decltype(dot_tag)::value;
    cgs_kernel<TB, NV, UP, DT><<<grid, kThreads, 0, st>>>(V, vld, W.alpha, W.m + 1, hin, kMaxRestart + 2, src,
                                                          dst, W.ns, W.active, ra, sel_w2, sel_v2);
  };
  using T = std::true_type;
  using F = std::false_type;
  auto pick = [&](auto nv_tag) {
    if (update && dots) go(nv_tag, T{}, T{});
    else if (update) go(nv_tag, T{}, F{});
    else go(nv_tag, F{}, T{});
  };
  switch (nv) {
#define RTE_NV_CASE(K) case K: pick(std::integral_constant<int, K>{}); break;
    RTE_NV_CASE(1) RTE_NV_CASE(2) RTE_NV_CASE(3) RTE_NV_CASE(4) RTE_NV_CASE(5) RTE_NV_CASE(6) RTE_NV_CASE(7)
    RTE_NV_CASE(8) RTE_NV_CASE(9) RTE_NV_CASE(10) RTE_NV_CASE(11) RTE_NV_CASE(12) RTE_NV_CASE(13)
    RTE_NV_CASE(14) RTE_NV_CASE(15) RTE_NV_CASE(16) RTE_NV_CASE(17) RTE_NV_CASE(18) RTE_NV_CASE(19)
    RTE_NV_CASE(20) RTE_NV_CASE(21) RTE_NV_CASE(22) RTE_NV_CASE(23) RTE_NV_CASE(24) RTE_NV_CASE(25)
    RTE_NV_CASE(26) RTE_NV_CASE(27) RTE_NV_CASE(28) RTE_NV_CASE(29) RTE_NV_CASE(30) RTE_NV_CASE(31)
    RTE_NV_CASE(32)
#undef RTE_NV_CASE
    default:
      set_error("gmres: restart > 32 is not supported by the fused CGS kernels");
      throw Fail{RTE_EINVAL};
  }
  // bytes: NV basis vectors + src read, dst written if updating; flops: 2 per (vector, element)
  // for each of the update and the dots, + 2 per element for the norm.
  const double ne = (double)W.ns * W.B;
  const double bytes = (double)sizeof(TB) * ne * (nv + 1 + (update ? 1 : 0));
  const double flops = ne * (2.0 * nv * ((update ? 1 : 0) + (dots ? 1 : 0)) + 2.0);
  // (selective pass: whether it streamed is decided on the device, so no bytes are booked)
  if (sel_w2)
    after_launch(cls, st, 0.0, 0.0, 0);
  else
    after_launch(cls, st, flops, bytes, 0);
}

// DCGS2 update pass at step j (NV = j final vectors before the candidate V_j).
template <typename TB>
static void launch_dcgs_update(const GmresWork& W, TB* V, int j, const TB* w, cudaStream_t st) {
  RedArgs ra{W.partials, W.counters, W.h2, kMaxRestart + 2, W.nblk};
  dim3 grid(W.nblk, W.B);
  const int64_t vld = W.ns * W.B;
  prof_begin(st, "dcgs_update");
  auto go = [&](auto nv_tag) {
    constexpr int NV = decltype(nv_tag)::value;
    dcgs_update_kernel<TB, NV><<<grid, kThreads, 0, st>>>(V, vld, W.alpha, W.m + 1, W.cA, W.cB, kMaxRestart + 2, w,
                                                          W.ns, W.active, ra);
  };
  switch (j) {
#define RTE_NV_CASE(K) case K: go(std::integral_constant<int, K>{}); break;
    RTE_NV_CASE(0) RTE_NV_CASE(1) RTE_NV_CASE(2) RTE_NV_CASE(3) RTE_NV_CASE(4) RTE_NV_CASE(5) RTE_NV_CASE(6)
    RTE_NV_CASE(7) RTE_NV_CASE(8) RTE_NV_CASE(9) RTE_NV_CASE(10) RTE_NV_CASE(11) RTE_NV_CASE(12) RTE_NV_CASE(13)
    RTE_NV_CASE(14) RTE_NV_CASE(15) RTE_NV_CASE(16) RTE_NV_CASE(17) RTE_NV_CASE(18) RTE_NV_CASE(19)
    RTE_NV_CASE(20) RTE_NV_CASE(21) RTE_NV_CASE(22) RTE_NV_CASE(23) RTE_NV_CASE(24) RTE_NV_CASE(25)
    RTE_NV_CASE(26) RTE_NV_CASE(27) RTE_NV_CASE(28) RTE_NV_CASE(29) RTE_NV_CASE(30) RTE_NV_CASE(31)
#undef RTE_NV_CASE
    default:
      set_error("gmres: restart > 32 is not supported by the fused DCGS2 kernels");
      throw Fail{RTE_EINVAL};
  }
  // bytes: j final vectors + the candidate + w read, the candidate and the new vector written;
  // flops: 2 per (vector, element) for the two updates and the dots, + 2 per element for the norm
  const double ne = (double)W.ns * W.B;
  after_launch("dcgs_update", st, ne * (2.0 * j + 2.0 * (j + 1) + 2.0 * (j + 1) + 2.0),
               (double)sizeof(TB) * ne * (j + 4), 0);
}

template <typename T, typename TO>
static void launch_norm(const GmresWork& W, const T* x, TO* xo, double* out, cudaStream_t st) {
  RedArgs ra{W.partials, W.counters, out, 1, W.nblk};
  prof_begin(st, "norm");
  norm_kernel<T, TO><<<dim3(W.nblk, W.B), kThreads, 0, st>>>(x, xo, W.ns, ra);
  const double ne = (double)W.ns * W.B;
  after_launch("norm", st, 2.0 * ne, ne * (sizeof(T) + (xo ? sizeof(TO) : 0.0)), 0);
}

}  // namespace rte

using namespace rte;

// Workspace cache keyed by problem (freed by rte_destroy through free_gmres_work).
static std::mutex g_wmu;
static std::map<const rte_problem*, GmresWork> g_work;

void rte::free_gmres_work(const rte_problem* p) {
  std::lock_guard<std::mutex> lk(g_wmu);
  auto it = g_work.find(p);
  if (it != g_work.end()) {
    it->second.release();
    g_work.erase(it);
  }
}

void rte::drop_net_graphs(const mgnet_net* net) {
  std::lock_guard<std::mutex> lk(g_wmu);
  for (auto& kv : g_work) kv.second.drop_graphs(net);
}

static bool graphs_enabled() {
  static const bool on = getenv("RTE_NO_GRAPHS") == nullptr;
  return on;
}

// w = A P(alpha_j V_j) in fp32 (precond 0 none, 1 MgNet, 2 block Jacobi): the operator part of
// Arnoldi step j
static void step_operator(const rte_problem* p, const mgnet_net* net, const GmresWork& W, int precond, int j,
                          cudaStream_t st) {
  const int m = W.m;
  const float* vj = W.V + (size_t)j * p->n;
  if (precond == 1) {
    vcycle_run(net, vj, W.z, true, W.alpha + j, m + 1, st);
    launch_apply_f32(p, W.z, W.w, nullptr, 0, st);
  } else if (precond == 2) {
    bj_apply<float>(p, vj, W.z, W.alpha + j, m + 1, st);
    launch_apply_f32(p, W.z, W.w, nullptr, 0, st);
  } else {
    launch_apply_f32(p, vj, W.w, W.alpha + j, m + 1, st);
  }
}

// Captures step j's operator part into a graph (on a private stream; nothing runs).  Returns
// nullptr (and caches nothing) when capture is unavailable or per-launch timing would have to be
// recorded inside it.
static GmresWork::StepGraph* capture_step(const rte_problem* p, const mgnet_net* net, GmresWork& W, int precond,
                                          int j) {
  static thread_local cudaStream_t cap = nullptr;
  if (!cap && cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  if (cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  capture_begin();
  const int64_t l0 = launches_now();
  bool ok = true;
  try {
    step_operator(p, net, W, precond, j, cap);
  } catch (...) {
    ok = false;
  }
  ok = capture_end() && ok;
  const int64_t nl = launches_now() - l0;
  launches_add(-nl);  // captured, not run
  cudaGraph_t g = nullptr;
  const cudaError_t e = cudaStreamEndCapture(cap, &g);
  cudaGraphExec_t exec = nullptr;
  if (ok && e == cudaSuccess && g && cudaGraphInstantiate(&exec, g, 0) == cudaSuccess) {
    cudaGraphDestroy(g);
    auto& sg = W.graphs[{net, net ? net->graph_epoch : 0, j, precond}];
    sg.exec = exec;
    sg.launches = nl;
    sg.classes = capture_classes();
    return &sg;
  }
  if (g) cudaGraphDestroy(g);
  (void)cudaGetLastError();
  return nullptr;
}

static void run_step_operator(const rte_problem* p, const mgnet_net* net, GmresWork& W, int precond, int j,
                              cudaStream_t st, bool capture_now = false) {
  if (graphs_enabled()) {
    const auto key = std::make_tuple(net, net ? net->graph_epoch : (uint64_t)0, j, precond);
    auto it = W.graphs.find(key);
    if (it == W.graphs.end()) {
      if (!capture_now) {  // first sight: run eagerly (warms kernels and lazy allocations), remember
        W.graphs[key];
        step_operator(p, net, W, precond, j, st);
        return;
      }
    } else if (it->second.exec) {
      if (!prof_wants_any(it->second.classes)) {  // (per-launch timing of an inner class: eager)
        RTE_CHECK_CUDA(cudaGraphLaunch(it->second.exec, st));
        launches_add(it->second.launches);
        return;
      }
      step_operator(p, net, W, precond, j, st);
      return;
    }
    if (!prof_wants_any({})) {  // (timing every class: a capture would be discarded anyway)
      W.graphs.erase(key);
      GmresWork::StepGraph* sg = capture_step(p, net, W, precond, j);
      if (sg) {
        RTE_CHECK_CUDA(cudaGraphLaunch(sg->exec, st));
        launches_add(sg->launches);
        return;
      }
      W.graphs[key];  // capture unavailable: keep running eagerly, retry next time
    }
  }
  step_operator(p, net, W, precond, j, st);
}

static GmresWork& get_work(const rte_problem* p, int m) {
  std::lock_guard<std::mutex> lk(g_wmu);
  GmresWork& W = g_work[p];
  // exact match only: every per-sample array (alpha, g, coef, H, the fp64 basis) is laid out with
  // stride m + 1 and captured graphs bake W.m in, so a different restart re-allocates
  if (W.V && W.m == m) return W;
  W.release();
  W.B = p->B;
  W.m = m;
  W.ns = p->n / p->B;
  int64_t n4 = W.ns / 4;
  int want = std::max(1, (2 * num_sms() + W.B - 1) / W.B);
  W.nblk = (int)std::max<int64_t>(1, std::min<int64_t>(want, (n4 + kThreads - 1) / kThreads));
  const int64_t n = p->n;
  const int B = p->B;
  W.V = dalloc<float>((size_t)(m + 1) * n);
  W.w = dalloc<float>(n);
  W.z = dalloc<float>(n);
  W.r64 = dalloc<double>(n);
  W.Hr = dalloc<double>((size_t)B * (m + 1) * m);
  W.Hraw = dalloc<double>((size_t)B * (m + 1) * m);
  W.cs = dalloc<double>((size_t)B * m);
  W.sn = dalloc<double>((size_t)B * m);
  W.g = dalloc<double>((size_t)B * (m + 1));
  W.alpha = dalloc<double>((size_t)B * (m + 1));
  W.h1 = dalloc<double>((size_t)B * (kMaxRestart + 2));
  W.h2 = dalloc<double>((size_t)B * (kMaxRestart + 2));
  W.h3 = dalloc<double>((size_t)B * (kMaxRestart + 2));
  W.cA = dalloc<double>((size_t)B * (kMaxRestart + 2));
  W.cB = dalloc<double>((size_t)B * (kMaxRestart + 2));
  W.hcol = dalloc<double>((size_t)B * (kMaxRestart + 2));
  W.rbuf = dalloc<double>(B);
  W.coef = dalloc<double>((size_t)B * (m + 1));
  W.bnorm = dalloc<double>(B);
  W.rn2 = dalloc<double>(B);
  W.partials = dalloc<double>((size_t)B * W.nblk * (kMaxRestart + 2));
  W.counters = dalloc<unsigned>(B);
  W.active = dalloc<int>(B);
  W.kcols = dalloc<int>(B);
  W.done = dalloc<int>(B);
  W.brkd = dalloc<int>(B);
  W.st_dev = dalloc<Status>(B);
  RTE_CHECK_CUDA(cudaMemset(W.counters, 0, sizeof(unsigned) * B));
  RTE_CHECK_CUDA(cudaMemset(W.Hraw, 0, sizeof(double) * B * (m + 1) * m));
  RTE_CHECK_CUDA(cudaHostAlloc(&W.st_host, sizeof(Status) * 2 * B, cudaHostAllocDefault));
  for (auto& e : W.st_ev) RTE_CHECK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return W;
}

extern "C" rte_status gmres_prepare(const rte_problem* p, const mgnet_net* net, const gmres_opts* opts, void* stream) {
  try {
    RTE_REQUIRE(p && opts, "gmres_prepare: NULL argument");
    RTE_REQUIRE(opts->restart >= 1 && opts->restart <= kMaxRestartApi, "gmres_prepare: restart must be in [1, 32]");
    RTE_REQUIRE(opts->precond == 0 || opts->precond == 2 || (opts->precond == 1 && net),
                "gmres_prepare: precond must be 0, 1 (with a net) or 2");
    if (!graphs_enabled() || opts->precision == 1) return RTE_OK;  // (the fp64 mode runs eagerly)
    const int m = opts->restart;
    GmresWork& W = get_work(p, m);
    if (opts->precond == 2) bj_prepare(p);
    cudaStream_t st = as_stream(stream);
    step_operator(p, net, W, opts->precond, 0, st);  // warm every kernel (results discarded)
    RTE_CHECK_CUDA(cudaStreamSynchronize(st));
    for (int j = 0; j < m; ++j) {
      auto it = W.graphs.find({net, net ? net->graph_epoch : (uint64_t)0, j, opts->precond});
      if (it != W.graphs.end() && it->second.exec) continue;
      if (it != W.graphs.end()) W.graphs.erase(it);
      if (!capture_step(p, net, W, opts->precond, j)) W.graphs[{net, net ? net->graph_epoch : (uint64_t)0, j, opts->precond}];
    }
    return RTE_OK;
  } catch (const Fail& f) {
    return f.st;
  } catch (const std::exception& e) {
    set_error(std::string("internal: ") + e.what());
    return RTE_EINTERNAL;
  }
}

// Host side of gmres_solve_host: where x goes when the solve has (probably) finished.
struct HostOut {
  double* x_host;
  bool copied = false;  // the early copy of the final x is in flight / done
};

static rte_status solve_impl(const rte_problem* p, const mgnet_net* net, const float* b_dev, double* x_dev,
                             const gmres_opts* opts, gmres_report* rep, cudaStream_t st, GmresWork* Wh,
                             HostOut* ho) {
  try {
    RTE_REQUIRE(p && b_dev && x_dev && opts && rep, "gmres_solve: NULL argument");
    const int m = opts->restart;
    RTE_REQUIRE(m >= 1 && m <= kMaxRestartApi, "gmres_solve: restart must be in [1, 32]");
    RTE_REQUIRE(opts->maxit >= 0, "gmres_solve: maxit must be >= 0");
    RTE_REQUIRE(opts->rtol > 0.0, "gmres_solve: rtol must be > 0");
    RTE_REQUIRE(opts->precond == 0 || opts->precond == 2 || (opts->precond == 1 && net),
                "gmres_solve: precond must be 0 (none), 1 (MgNet, requires a net) or 2 (block Jacobi)");
    RTE_REQUIRE(opts->x0_zero == 0 || opts->x0_zero == 1, "gmres_solve: x0_zero must be 0 or 1");
    if (opts->precond == 2) bj_prepare(p);  // (NEXT-2; builds the inverse cell blocks once)
    RTE_REQUIRE(!net || net->prob == p, "gmres_solve: net was created for another problem");
    GmresWork& W = Wh ? *Wh : get_work(p, m);
    const int B = p->B;
    const int64_t n = p->n;
    const int hld = kMaxRestart + 2;
    const int reorth = opts->reorth;  // 0 CGS2, 1 CGS1, 2 selective (DGKS), 3 DCGS2 (delayed CGS2)
    RTE_REQUIRE(reorth >= 0 && reorth <= 3, "gmres_solve: reorth must be 0, 1, 2 or 3");
    RTE_REQUIRE(opts->precision == 0 || opts->precision == 1, "gmres_solve: precision must be 0 or 1");
    const bool f64 = opts->precision == 1;
    if (f64 && !W.V64) {
      W.V64 = dalloc<double>((size_t)(m + 1) * n);
      W.w64 = dalloc<double>(n);
      W.z64 = dalloc<double>(n);
      W.q32 = dalloc<float>(n);
    }
    std::vector<int> total(B, 0), restarts(B, 0), brk(B, 0), conv(B, 0), done(B, 0);
    std::vector<double> est_last(B, 0.0), relres(B, 0.0);
    for (int b = 0; b < B; ++b) {
      rep[b].iterations = 0;
      rep[b].restarts = 0;
      rep[b].converged = 0;
      rep[b].breakdown = 0;
      rep[b].relres_true = 0;
      rep[b].relres_est = 0;
    }
    RTE_CHECK_CUDA(cudaMemsetAsync(W.done, 0, sizeof(int) * B, st));
    if (opts->x0_zero) RTE_CHECK_CUDA(cudaMemsetAsync(x_dev, 0, sizeof(double) * n, st));
    // ||b|| per sample
    launch_norm<float, float>(W, b_dev, nullptr, W.rn2, st);
    {
      std::vector<double> bn2(B);
      RTE_CHECK_CUDA(cudaMemcpyAsync(bn2.data(), W.rn2, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
      RTE_CHECK_CUDA(cudaStreamSynchronize(st));
      for (double& v : bn2) v = sqrt(v);
      RTE_CHECK_CUDA(cudaMemcpyAsync(W.bnorm, bn2.data(), sizeof(double) * B, cudaMemcpyHostToDevice, st));
      RTE_CHECK_CUDA(cudaStreamSynchronize(st));
    }
    bool first_cycle = true;
    int total_all = 0;  // lockstep inner iterations
    while (true) {
      // r = b - A x (fp64), v0 = r (basis precision, unnormalised), ||r||^2.  With x0 = 0 the first
      // residual is b itself (A 0 = 0 and b - 0 = b exactly in fp64): no apply, same bits.
      if (first_cycle && opts->x0_zero) {
        if (f64)
          launch_norm<float, double>(W, b_dev, W.V64, W.rn2, st);
        else
          launch_norm<float, float>(W, b_dev, W.V, W.rn2, st);
      } else {
        launch_apply_f64(p, x_dev, W.r64, b_dev, st);
        if (f64)
          launch_norm<double, double>(W, W.r64, W.V64, W.rn2, st);
        else
          launch_norm<double, float>(W, W.r64, W.V, W.rn2, st);
      }
      int stop_all = (total_all >= opts->maxit) ? 1 : 0;
      prof_begin(st, "cycle_init");
      cycle_init_kernel<<<(B + 63) / 64, 64, 0, st>>>(B, W.rn2, W.bnorm, opts->rtol, stop_all, W.alpha, m + 1, W.g,
                                                      m + 1, W.active, W.kcols, W.done, W.st_dev);
      after_launch("cycle_init", st);
      RTE_CHECK_CUDA(cudaMemcpyAsync(W.st_host, W.st_dev, sizeof(Status) * B, cudaMemcpyDeviceToHost, st));
      RTE_CHECK_CUDA(cudaStreamSynchronize(st));
      int n_active = 0;
      for (int b = 0; b < B; ++b) {
        relres[b] = W.st_host[b].est;
        conv[b] = W.st_host[b].converged;
        if (W.st_host[b].active) {
          ++n_active;
          ++restarts[b];
        }
      }
      if (n_active == 0) break;
      int pending = -1;  // step whose status has not been read yet
      // read step k's statuses (slot k & 1): history, counts, breakdown; returns the active count
      auto process_step = [&](int k) -> int {
        RTE_CHECK_CUDA(cudaEventSynchronize(W.st_ev[k & 1]));
        const Status* slot = W.st_host + (size_t)(k & 1) * B;
        int still = 0;
        for (int b = 0; b < B; ++b) {
          const Status& s = slot[b];
          bool was_active = (s.active || s.kcols == k + 1 || (s.breakdown == 2 && s.kcols == k));
          if (!was_active) continue;
          if (rep[b].history) rep[b].history[total[b]] = s.est;
          ++total[b];
          est_last[b] = s.est;
          if (s.breakdown) brk[b] = s.breakdown;
          if (s.active) ++still;
        }
        return still;
      };
      for (int j = 0; j < m; ++j) {
        // Arnoldi step j: w = A P(alpha_j V_j), then CGS passes against V_0..V_j (basis type TB)
        const double* h2 = nullptr;
        const double* nrm = nullptr;
        auto cgs_passes = [&](auto* V, auto* wv) {
          using TB = std::remove_pointer_t<decltype(V)>;
          TB* vnext = V + (size_t)(j + 1) * n;
          launch_cgs<TB>(W, V, j + 1, false, true, nullptr, wv, nullptr, W.h1, st);      // pass A
          if (reorth == 3) {  // DCGS2: coefficients, then one fused update pass (V_j corrected, V_{j+1})
            prof_begin(st, "dcgs_coef");
            dcgs_coef_kernel<<<B, 32, 0, st>>>(B, j, m, W.h2, W.h1, hld, W.Hraw, W.alpha, m + 1, W.cA, W.cB,
                                               W.hcol, W.rbuf, W.active);
            after_launch("dcgs_coef", st);
            launch_dcgs_update<TB>(W, V, j, wv, st);
            h2 = W.h2;
            nrm = W.h2;
          } else if (reorth != 1) {
            launch_cgs<TB>(W, V, j + 1, true, true, W.h1, wv, vnext, W.h2, st);          // pass B
            if (reorth == 2)                                                          // pass C (selective)
              launch_cgs<TB>(W, V, j + 1, true, false, W.h2, vnext, vnext, W.h3, st, W.h1 + (j + 1), W.h2 + (j + 1));
            else
              launch_cgs<TB>(W, V, j + 1, true, false, W.h2, vnext, vnext, W.h3, st);     // pass C
            h2 = W.h2;
            nrm = W.h3;  // update-only passes put ||.||^2 at index 0
          } else {
            launch_cgs<TB>(W, V, j + 1, true, false, W.h1, wv, vnext, W.h2, st);         // CGS1 only
            h2 = nullptr;
            nrm = W.h2;
          }
        };
        if (f64) {
          // fp64 basis: z = P(alpha_j V_j) with the fp64 V-cycle, w = A z in fp64 (W.r64 is free
          // inside a cycle and holds P z)
          const double* vj = W.V64 + (size_t)j * n;
          prof_begin(st, "scale_f64");
          scale_f64_kernel<<<dim3(W.nblk, B), kThreads, 0, st>>>(vj, W.alpha + j, m + 1, W.z64, nullptr, W.ns,
                                                                  W.nblk);
          after_launch("scale_f64", st, 0.0, 16.0 * (double)n, 0);
          const double* zin = W.z64;
          if (opts->precond == 1) {
            vcycle_run_f64(net, W.z64, W.r64, true, st);
            zin = W.r64;
          } else if (opts->precond == 2) {
            bj_apply<double>(p, W.z64, W.r64, nullptr, 0, st);
            zin = W.r64;
          }
          launch_apply_f64(p, zin, W.w64, nullptr, st);
          cgs_passes(W.V64, W.w64);
        } else {
          // fp32 basis: z = P(alpha_j V_j) or alpha_j V_j, w = A z in fp32 (a cached CUDA graph per j
          // when available), then the CGS passes
          run_step_operator(p, net, W, opts->precond, j, st);
          cgs_passes(W.V, W.w);
        }
        ++total_all;
        int last = (total_all >= opts->maxit) ? 1 : 0;
        prof_begin(st, "givens");
        givens_kernel<<<(B + 63) / 64, 64, 0, st>>>(B, j, m, W.h1, h2, hld, nrm, hld, reorth == 2 ? 1 : 0, W.Hr, W.Hraw,
                                                    first_cycle ? 1 : 0, W.cs, W.sn, W.g, W.alpha, m + 1, W.bnorm,
                                                    opts->rtol, last, W.active, W.kcols, W.st_dev,
                                                    reorth == 3 ? W.hcol : nullptr, W.rbuf, W.brkd);
        after_launch("givens", st);
        // The step's status is read one step late: step j + 1 is enqueued before the host waits for
        // step j, so the GPU never idles on the host round trip.  When step j turns out to have
        // stopped every sample, the already queued step j + 1 is gated out on the device (its CGS
        // passes and Givens rotation skip inactive samples; the operator part writes scratch only).
        RTE_CHECK_CUDA(cudaMemcpyAsync(W.st_host + (size_t)(j & 1) * B, W.st_dev, sizeof(Status) * B,
                                       cudaMemcpyDeviceToHost, st));
        RTE_CHECK_CUDA(cudaEventRecord(W.st_ev[j & 1], st));
        if (pending >= 0 && process_step(pending) == 0) {
          pending = -1;
          --total_all;  // (step j was queued but did no work: it does not count toward maxit)
          break;
        }
        pending = j;
        if (last) {  // the budget ends here: nothing more to enqueue, read this step now
          process_step(j);
          pending = -1;
          break;
        }
      }
      if (pending >= 0) {
        process_step(pending);
        pending = -1;
      }

      // x += P(V y).  (gmres_solve_host: an early copy of x from the previous cycle must land before
      // x changes again)
      auto wait_host_copy = [&]() {
        if (ho && ho->copied) {
          RTE_CHECK_CUDA(cudaStreamWaitEvent(st, W.ev_cp, 0));
          ho->copied = false;
        }
      };
      prof_begin(st, "backsolve");
      if (reorth == 3) {
        dcgs_backsolve_kernel<<<(B + 63) / 64, 64, 0, st>>>(B, m, W.Hraw, W.h2, hld, W.alpha, m + 1, W.kcols,
                                                            W.brkd, W.coef, m + 1);
      } else {
        backsolve_kernel<<<(B + 63) / 64, 64, 0, st>>>(B, m, W.Hr, W.g, W.alpha, m + 1, W.kcols, W.coef, m + 1);
      }
      after_launch("backsolve", st);
      if (first_cycle) {  // the first cycle's unrotated Hessenberg matrix (DCGS2: after its last column's
                          // delayed correction in the back-solve)
        for (int b = 0; b < B; ++b)
          if (rep[b].hessenberg)
            RTE_CHECK_CUDA(cudaMemcpyAsync(rep[b].hessenberg, W.Hraw + (size_t)b * (m + 1) * m,
                                           sizeof(double) * (m + 1) * m, cudaMemcpyDeviceToHost, st));
      }
      first_cycle = false;
      if (f64) {
        prof_begin(st, "combine");
        combine_kernel<double, double><<<dim3(W.nblk, B), kThreads, 0, st>>>(W.V64, n, W.coef, m + 1, W.kcols, W.z64,
                                                                              W.ns, W.nblk);
        after_launch("combine", st, 2.0 * m * (double)n, 8.0 * (double)n * (m + 1), 0);
        const double* corr = W.z64;
        if (opts->precond == 1) {
          vcycle_run_f64(net, W.z64, W.r64, true, st);
          corr = W.r64;
        } else if (opts->precond == 2) {
          bj_apply<double>(p, W.z64, W.r64, nullptr, 0, st);
          corr = W.r64;
        }
        wait_host_copy();
        prof_begin(st, "axpy64");
        axpy64_kernel<double><<<dim3(W.nblk, B), kThreads, 0, st>>>(x_dev, corr, nullptr, W.kcols, W.ns, W.nblk);
        after_launch("axpy64", st, (double)n, 28.0 * (double)n, 0);
      } else {
        prof_begin(st, "combine");
        combine_kernel<float, float><<<dim3(W.nblk, B), kThreads, 0, st>>>(W.V, n, W.coef, m + 1, W.kcols, W.w, W.ns,
                                                                            W.nblk);
        after_launch("combine", st, 2.0 * m * (double)n, 4.0 * (double)n * (m + 1), 0);
        const float* corr = W.w;
        if (opts->precond == 1) {
          vcycle_run(net, W.w, W.z, true, nullptr, 0, st);
          corr = W.z;
        } else if (opts->precond == 2) {
          bj_apply<float>(p, W.w, W.z, nullptr, 0, st);
          corr = W.z;
        }
        wait_host_copy();
        prof_begin(st, "axpy64");
        axpy64_kernel<float><<<dim3(W.nblk, B), kThreads, 0, st>>>(x_dev, corr, nullptr, W.kcols, W.ns, W.nblk);
        after_launch("axpy64", st, (double)n, 20.0 * (double)n, 0);
      }
      // samples that broke down stop (oracle: breakdown ends the solve)
      bool any_brk = false;
      for (int b = 0; b < B; ++b)
        if (brk[b] && !done[b]) { done[b] = 1; any_brk = true; }
      if (any_brk) RTE_CHECK_CUDA(cudaMemcpyAsync(W.done, done.data(), sizeof(int) * B, cudaMemcpyHostToDevice, st));
      if (ho) {
        // gmres_solve_host: x is final unless another cycle runs, i.e. unless the budget is left and
        // some sample's estimate has not converged.  Start its device->host copy now on the copy
        // stream, overlapping the closing fp64 true residual; a wrong guess costs a second copy.
        bool fin = total_all >= opts->maxit;
        if (!fin) {
          fin = true;
          for (int b = 0; b < B; ++b)
            if (!brk[b] && !(est_last[b] <= opts->rtol)) fin = false;
        }
        if (fin) {
          RTE_CHECK_CUDA(cudaEventRecord(W.ev_x, st));
          RTE_CHECK_CUDA(cudaStreamWaitEvent(W.cp, W.ev_x, 0));
          RTE_CHECK_CUDA(cudaMemcpyAsync(ho->x_host, x_dev, sizeof(double) * n, cudaMemcpyDeviceToHost, W.cp));
          RTE_CHECK_CUDA(cudaEventRecord(W.ev_cp, W.cp));
          ho->copied = true;
        }
      }
    }
    for (int b = 0; b < B; ++b) {
      rep[b].iterations = total[b];
      rep[b].restarts = restarts[b];
      rep[b].converged = conv[b];
      rep[b].breakdown = brk[b];
      rep[b].relres_true = relres[b];
      rep[b].relres_est = est_last[b];
    }
    if (ho && !ho->copied)
      RTE_CHECK_CUDA(cudaMemcpyAsync(ho->x_host, x_dev, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    RTE_CHECK_CUDA(cudaStreamSynchronize(st));
    if (ho && ho->copied) RTE_CHECK_CUDA(cudaEventSynchronize(W.ev_cp));
    for (int b = 0; b < B; ++b)
      if (brk[b] == 2) {
        set_error("gmres_solve: non-finite value (NaN/Inf) in the Arnoldi process of sample " + std::to_string(b) +
                  " at iteration " + std::to_string(total[b]) + "; the reports are filled (breakdown = 2)");
        return RTE_ENUMERIC;
      }
    return RTE_OK;
  } catch (const Fail& f) {
    return f.st;
  } catch (const std::exception& e) {
    set_error(std::string("internal: ") + e.what());
    return RTE_EINTERNAL;
  }
}

extern "C" rte_status gmres_solve(const rte_problem* p, const mgnet_net* net, const float* b_dev, double* x_dev,
                                  const gmres_opts* opts, gmres_report* rep, void* stream) {
  return solve_impl(p, net, b_dev, x_dev, opts, rep, as_stream(stream), nullptr, nullptr);
}

extern "C" rte_status gmres_solve_host(const rte_problem* p, const mgnet_net* net, const float* b_host,
                                       double* x_host, const gmres_opts* opts, gmres_report* rep, void* stream) {
  try {
    RTE_REQUIRE(p && b_host && x_host && opts && rep, "gmres_solve_host: NULL argument");
    RTE_REQUIRE(opts->restart >= 1 && opts->restart <= kMaxRestartApi, "gmres_solve: restart must be in [1, 32]");
    GmresWork& W = get_work(p, opts->restart);
    const int64_t n = p->n;
    if (!W.bh) {
      W.bh = dalloc<float>(n);
      W.xh = dalloc<double>(n);
      RTE_CHECK_CUDA(cudaStreamCreateWithFlags(&W.cp, cudaStreamNonBlocking));
      RTE_CHECK_CUDA(cudaEventCreateWithFlags(&W.ev_x, cudaEventDisableTiming));
      RTE_CHECK_CUDA(cudaEventCreateWithFlags(&W.ev_cp, cudaEventDisableTiming));
    }
    cudaStream_t st = as_stream(stream);
    RTE_CHECK_CUDA(cudaMemcpyAsync(W.bh, b_host, sizeof(float) * n, cudaMemcpyHostToDevice, st));
    if (!opts->x0_zero) RTE_CHECK_CUDA(cudaMemcpyAsync(W.xh, x_host, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    HostOut ho{x_host};
    const rte_status rc = solve_impl(p, net, W.bh, W.xh, opts, rep, st, &W, &ho);
    // (on an error return too: no copy into the caller's x_host may still be in flight)
    if (rc != RTE_OK && W.cp) cudaStreamSynchronize(W.cp);
    return rc;
  } catch (const Fail& f) {
    return f.st;
  } catch (const std::exception& e) {
    set_error(std::string("internal: ") + e.what());
    return RTE_EINTERNAL;
  }
}
