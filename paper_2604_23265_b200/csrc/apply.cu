// Discrete-ordinates operator kernels: rhs, fp32 apply (SIMT reference path for any M),
// fp64 apply (restart residual).  The tensor-core 3xTF32 apply lives in apply_tc.cu.
//
// Operator (PAPER.md:91-93 eq:DORTE_2d with the upwind stencil of DESIGN.md R9):
//   (A psi)_{jim} = (|c_m|/h + |s_m|/h + sigma_t) psi_{jim} - (|c_m|/h) psi_{j,i-sgn c_m,m}
//                   - (|s_m|/h) psi_{j-sgn s_m,i,m} - sigma_s sum_n S_mn psi_{jin}
// Layout psi[b][j][i][m]; the scattering term is the GEMM  Psi[cells x M] . S^T[M x M], computed
// in the conservation-preserving form S psi = c + S (psi - c), c = psi_{cell, m=0} (apply_tc.cu).
#include <type_traits>

#include "common.h"

namespace rte {
namespace {

// b = eps q + ghost terms.  One thread per unknown.
__global__ void rhs_kernel(int B, int N, int M, const float* __restrict__ f, const float* __restrict__ inflow,
                           const float* __restrict__ ax, const float* __restrict__ ay,
                           const int8_t* __restrict__ sgx, const int8_t* __restrict__ sgy,
                           float* __restrict__ b) {
  int64_t n = (int64_t)B * N * N * M;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    int m = (int)(e % M);
    int64_t cell = e / M;
    int i = (int)(cell % N);
    int j = (int)((cell / N) % N);
    int bb = (int)(cell / ((int64_t)N * N));
    double v = f[cell];
    if (inflow) {
      const float* fin = inflow + (int64_t)bb * 4 * N * M;
      if (sgx[m] > 0 && i == 0) v += (double)ax[m] * fin[(0 * N + j) * M + m];
      if (sgx[m] < 0 && i == N - 1) v += (double)ax[m] * fin[(1 * N + j) * M + m];
      if (sgy[m] > 0 && j == 0) v += (double)ay[m] * fin[(2 * N + i) * M + m];
      if (sgy[m] < 0 && j == N - 1) v += (double)ay[m] * fin[(3 * N + i) * M + m];
    }
    b[e] = (float)v;
  }
}

// SIMT fused stencil + scattering GEMM.  Tile = TP cells x TMO ordinates (TP*TMO = 4096),
// 256 threads, each 4 cells x 4 ordinates, K chunks of 16 ordinates through shared memory.
template <typename T, int TMO>
__global__ void __launch_bounds__(256) apply_simt_kernel(
    int N, int M, const T* __restrict__ x, T* __restrict__ y, const T* __restrict__ St,
    const T* __restrict__ sig_d, const T* __restrict__ sig_s, const T* __restrict__ axv,
    const T* __restrict__ ayv, const int8_t* __restrict__ sgx, const int8_t* __restrict__ sgy,
    const float* __restrict__ bvec, const double* __restrict__ alpha, int alpha_stride) {
  constexpr int TP = 4096 / TMO;
  constexpr int KC = 16;
  constexpr int TX = TMO / 4;          // threads along ordinates
  __shared__ __align__(16) T As[KC][TP + 4];
  __shared__ __align__(16) T Bs[KC][TMO + 4];
  const int tid = threadIdx.x;
  const int tx = tid % TX, ty = tid / TX;
  const int bsample = blockIdx.z;
  const int64_t cells = (int64_t)N * N;
  const int64_t c0 = (int64_t)blockIdx.x * TP;        // first cell (within sample) of the tile
  const int m0 = blockIdx.y * TMO;
  const T* xs = x + (int64_t)bsample * cells * M;
  const T* Sts = St + (int64_t)bsample * M * M;
  T acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[a][c] = T(0);

  for (int k0 = 0; k0 < M; k0 += KC) {
    // A chunk: TP cells x KC ordinates (x[cell][k0..k0+15] - c_cell) -> As[k][cell]; the
    // contraction is S psi = c + S (psi - c) with c = psi at ordinate 0 (S row-stochastic, R5)
    for (int e = tid; e < TP * KC; e += 256) {
      int cl = e / KC, kk = e % KC;
      int64_t cell = c0 + cl;
      T v = T(0);
      if (cell < cells && k0 + kk < M) v = xs[cell * M + k0 + kk] - xs[cell * M];
      As[kk][cl] = v;
    }
    // B chunk: St[k0+kk][m0 + o]
    for (int e = tid; e < KC * TMO; e += 256) {
      int kk = e / TMO, o = e % TMO;
      T v = T(0);
      if (k0 + kk < M && m0 + o < M) v = Sts[(int64_t)(k0 + kk) * M + m0 + o];
      Bs[kk][o] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      T av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[kk][ty * 4 + a];
#pragma unroll
      for (int c = 0; c < 4; ++c) bv[c] = Bs[kk][tx * 4 + c];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c] = fma(av[a], bv[c], acc[a][c]);
    }
    __syncthreads();
  }
  // epilogue: stencil + diagonal - sigma_s * (S psi)
  const T al = alpha ? (T)alpha[(int64_t)bsample * alpha_stride] : T(1);
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    int64_t cell = c0 + ty * 4 + a;
    if (cell >= cells) continue;
    int i = (int)(cell % N), j = (int)(cell / N);
    int64_t gcell = (int64_t)bsample * cells + cell;
    const T sd = sig_d[gcell], ss = sig_s[gcell];
    const T cc = xs[cell * M];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      int m = m0 + tx * 4 + c;
      if (m >= M) continue;
      const T psi = xs[cell * M + m];
      const int ii = i - sgx[m], jj = j - sgy[m];
      const T nx = (ii >= 0 && ii < N) ? xs[(cell - sgx[m]) * M + m] : T(0);
      const T ny = (jj >= 0 && jj < N) ? xs[(cell - (int64_t)sgy[m] * N) * M + m] : T(0);
      T v = al * stencil_diag(axv[m], ayv[m], sd, ss, psi, nx, ny, cc, acc[a][c]);
      int64_t o = gcell * M + m;
      if (bvec) v = (T)bvec[o] - v;
      y[o] = v;
    }
  }
}

// Wide-tile SIMT apply (M % 128 == 0; the fp64 restart residual): tile = 128 cells x 128
// ordinates, 256 threads, each 8 cells x 8 ordinates (cells ty*4+a and 64+ty*4+a, ordinates tx*4+c
// and 64+tx*4+c: conflict-free LDS.128 and 64 FMAs per 8 shared loads), K in chunks of 8 staged
// through double-buffered shared memory with a register prefetch of the next chunk.  Same
// arithmetic as apply_simt_kernel: centred contraction, then the stencil epilogue.
template <typename T>
__global__ void __launch_bounds__(256) apply_simt_wide_kernel(
    int N, int M, const T* __restrict__ x, T* __restrict__ y, const T* __restrict__ St,
    const T* __restrict__ sig_d, const T* __restrict__ sig_s, const T* __restrict__ axv,
    const T* __restrict__ ayv, const int8_t* __restrict__ sgx, const int8_t* __restrict__ sgy,
    const float* __restrict__ bvec, const double* __restrict__ alpha, int alpha_stride) {
  constexpr int TP = 128, TMO = 128, KC = 8;
  __shared__ __align__(16) T As[2][KC][TP];
  __shared__ __align__(16) T Bs[2][KC][TMO];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int bsample = blockIdx.z;
  const int64_t cells = (int64_t)N * N;
  const int64_t c0 = (int64_t)blockIdx.x * TP;
  const int m0 = blockIdx.y * TMO;
  const T* xs = x + (int64_t)bsample * cells * M;
  const T* Sts = St + (int64_t)bsample * M * M;
  // global -> register staging: A chunk = 128 cells x 8 k (4 per thread: cell tid/8 + 32r,
  // k tid%8), B chunk = 8 k x 128 ordinates (4 per thread: k tid/128*... row-contiguous)
  const int a_cl = tid / KC, a_k = tid % KC;
  T ctr[4];  // centres psi_{cell, 0} of this thread's 4 staged cells
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t cell = c0 + a_cl + 32 * r;
    ctr[r] = cell < cells ? xs[cell * M] : T(0);
  }
  T ra[4], rb[4];
  auto load_chunk = [&](int k0) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int64_t cell = c0 + a_cl + 32 * r;
      ra[r] = cell < cells ? xs[cell * M + k0 + a_k] - ctr[r] : T(0);
      const int e = tid + 256 * r, kk = e / TMO, o = e % TMO;
      rb[r] = Sts[(int64_t)(k0 + kk) * M + m0 + o];
    }
  };
  auto store_chunk = [&](int buf) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      As[buf][a_k][a_cl + 32 * r] = ra[r];
      const int e = tid + 256 * r;
      Bs[buf][e / TMO][e % TMO] = rb[r];
    }
  };
  T acc[8][8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[a][c] = T(0);
  load_chunk(0);
  store_chunk(0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < M; k0 += KC) {
    const bool more = k0 + KC < M;
    if (more) load_chunk(k0 + KC);
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      T av[8], bv[8];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          av[4 * h + q] = As[buf][kk][64 * h + ty * 4 + q];
          bv[4 * h + q] = Bs[buf][kk][64 * h + tx * 4 + q];
        }
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[a][c] = fma(av[a], bv[c], acc[a][c]);
    }
    if (more) {
      store_chunk(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
  const T al = alpha ? (T)alpha[(int64_t)bsample * alpha_stride] : T(1);
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int64_t cell = c0 + 64 * (a / 4) + ty * 4 + (a % 4);
    if (cell >= cells) continue;
    const int i = (int)(cell % N), j = (int)(cell / N);
    const int64_t gcell = (int64_t)bsample * cells + cell;
    const T sd = sig_d[gcell], ss = sig_s[gcell];
    const T cc = xs[cell * M];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int m = m0 + 64 * (c / 4) + tx * 4 + (c % 4);
      const T psi = xs[cell * M + m];
      const int ii = i - sgx[m], jj = j - sgy[m];
      const T nx = (ii >= 0 && ii < N) ? xs[(cell - sgx[m]) * M + m] : T(0);
      const T ny = (jj >= 0 && jj < N) ? xs[(cell - (int64_t)sgy[m] * N) * M + m] : T(0);
      T v = al * stencil_diag(axv[m], ayv[m], sd, ss, psi, nx, ny, cc, acc[a][c]);
      const int64_t o = gcell * M + m;
      if (bvec) v = (T)bvec[o] - v;
      y[o] = v;
    }
  }
}

// fp64 apply on the DMMA pipe (mma.sync m8n8k4 f64: measured 37 TF/s on the B200 vs 36 for SIMT
// DFMA, scripts/fp64_bench.cu), M % 64 == 0.  Block = 128 cells x 64 ordinates, 8 warps, warp tile
// 32 x 32 = 4 x 4 MMA tiles (32 fp64 accumulators per thread, so several blocks per SM); K in
// chunks of 8 through double-buffered shared memory: A[k][cell] = psi - c (centred, as the other
// paths), B[k][m] = S^T.  Fragments (PTX m8n8k4 .f64): A row = lane/4, k = lane%4; B k = lane%4,
// col = lane/4; C row = lane/4, cols 2(lane%4) + {0, 1}.  Same epilogue as apply_simt_kernel.
__global__ void __launch_bounds__(256) apply_dmma_kernel(
    int N, int M, const double* __restrict__ x, double* __restrict__ y, const double* __restrict__ St,
    const double* __restrict__ sig_d, const double* __restrict__ sig_s, const double* __restrict__ axv,
    const double* __restrict__ ayv, const int8_t* __restrict__ sgx, const int8_t* __restrict__ sgy,
    const float* __restrict__ bvec) {
  constexpr int TP = 128, TM = 64, KC = 8, PA = TP + 4, PB = TM + 4;
  __shared__ __align__(16) double As[2][KC][PA];
  __shared__ __align__(16) double Bs[2][KC][PB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2;  // warp tile: cells wm*32.., ordinates wn*32..
  const int bsample = blockIdx.z;
  const int64_t cells = (int64_t)N * N;
  const int64_t c0 = (int64_t)blockIdx.x * TP;
  const int m0 = blockIdx.y * TM;
  const double* xs = x + (int64_t)bsample * cells * M;
  const double* Sts = St + (int64_t)bsample * M * M;
  // staging: A chunk 128 cells x 8 k (4 per thread: cell tid/8 + 32 r, k tid%8),
  // B chunk 8 k x 64 ordinates (2 per thread)
  const int a_cl = tid >> 3, a_k = tid & 7;
  double ctr[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t cell = c0 + a_cl + 32 * r;
    ctr[r] = cell < cells ? xs[cell * M] : 0.0;
  }
  double ra[4], rb[2];
  auto load_chunk = [&](int k0) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int64_t cell = c0 + a_cl + 32 * r;
      ra[r] = cell < cells ? xs[cell * M + k0 + a_k] - ctr[r] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int e = tid + 256 * r, kk = e / TM, o = e % TM;
      rb[r] = Sts[(int64_t)(k0 + kk) * M + m0 + o];
    }
  };
  auto store_chunk = [&](int buf) {
#pragma unroll
    for (int r = 0; r < 4; ++r) As[buf][a_k][a_cl + 32 * r] = ra[r];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int e = tid + 256 * r;
      Bs[buf][e / TM][e % TM] = rb[r];
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  load_chunk(0);
  store_chunk(0);
  __syncthreads();
  int buf = 0;
  const int fr = lane >> 2, fk = lane & 3;
  for (int k0 = 0; k0 < M; k0 += KC) {
    const bool more = k0 + KC < M;
    if (more) load_chunk(k0 + KC);
#pragma unroll
    for (int ks = 0; ks < KC; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[buf][ks + fk][wm * 32 + 8 * i + fr];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs[buf][ks + fk][wn * 32 + 8 * j + fr];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(acc[i][j][0]), "+d"(acc[i][j][1])
                       : "d"(af[i]), "d"(bf[j]));
    }
    if (more) {
      store_chunk(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
  // epilogue: stencil + diagonal - sigma_s * (c + S (psi - c))
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t cell = c0 + wm * 32 + 8 * i + fr;
    if (cell >= cells) continue;
    const int ci = (int)(cell % N), cj = (int)(cell / N);
    const int64_t gcell = (int64_t)bsample * cells + cell;
    const double sd = sig_d[gcell], ss = sig_s[gcell];
    const double cc = xs[cell * M];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = m0 + wn * 32 + 8 * j + 2 * fk + h;
        const int ii = ci - sgx[m], jj = cj - sgy[m];
        const double nx = (ii >= 0 && ii < N) ? xs[(cell - sgx[m]) * M + m] : 0.0;
        const double ny = (jj >= 0 && jj < N) ? xs[(cell - (int64_t)sgy[m] * N) * M + m] : 0.0;
        double v = stencil_diag(axv[m], ayv[m], sd, ss, xs[cell * M + m], nx, ny, cc, acc[i][j][h]);
        const int64_t o = gcell * M + m;
        if (bvec) v = (double)bvec[o] - v;
        y[o] = v;
      }
  }
}

template <typename T>
void launch_simt(const rte_problem* p, const T* x, T* y, const T* St, const T* st, const T* ss,
                 const T* ax, const T* ay, const float* b, const double* alpha, int alpha_stride,
                 cudaStream_t stream) {
  int64_t cells = (int64_t)p->N * p->N;
  auto go = [&](auto tmo_tag) {
    constexpr int TMO = decltype(tmo_tag)::value;
    constexpr int TP = 4096 / TMO;
    dim3 grid((unsigned)((cells + TP - 1) / TP), (unsigned)((p->M + TMO - 1) / TMO), (unsigned)p->B);
    apply_simt_kernel<T, TMO><<<grid, 256, 0, stream>>>(p->N, p->M, x, y, St, st, ss, ax, ay, p->sgx, p->sgy,
                                                         b, alpha, alpha_stride);
  };
  if constexpr (std::is_same<T, double>::value) {
    if (p->M % 64 == 0 && alpha == nullptr && getenv("RTE_NO_DMMA") == nullptr) {
      dim3 grid((unsigned)((cells + 127) / 128), (unsigned)(p->M / 64), (unsigned)p->B);
      apply_dmma_kernel<<<grid, 256, 0, stream>>>(p->N, p->M, x, y, St, st, ss, ax, ay, p->sgx, p->sgy, b);
      return;
    }
  }
  if (p->M % 128 == 0) {
    dim3 grid((unsigned)((cells + 127) / 128), (unsigned)(p->M / 128), (unsigned)p->B);
    apply_simt_wide_kernel<T><<<grid, 256, 0, stream>>>(p->N, p->M, x, y, St, st, ss, ax, ay, p->sgx, p->sgy, b,
                                                        alpha, alpha_stride);
    return;
  }
  if (p->M <= 16) go(std::integral_constant<int, 16>{});
  else if (p->M <= 32) go(std::integral_constant<int, 32>{});
  else go(std::integral_constant<int, 64>{});
}

}  // namespace

// Algorithmic work of one apply: 2 B N^2 M^2 flops for the scattering GEMM plus
// 8 per unknown for the stencil; bytes = read x once + write y once (+ read b) + 2 coefficients
// per cell + the B M x M scattering matrices (+ the 2 M stencil weights, negligible).
double apply_flops(const rte_problem* p) { return 2.0 * (double)p->ncell * p->M * p->M + 8.0 * (double)p->n; }
double apply_bytes(const rte_problem* p, int elt, int b_elt) {
  return (double)p->n * (2 * elt + b_elt) + 2.0 * elt * (double)p->ncell + (double)elt * p->B * p->M * p->M;
}

void launch_rhs(const rte_problem* p, float* b, cudaStream_t st) {
  if (p->kind == 1) {
    launch_tfps_rhs(p, b, st);
    return;
  }
  if (p->kind == 2) {
    launch_atfps<float>(p, 1, nullptr, b, nullptr, 0, nullptr, st);
    return;
  }
  int64_t n = p->n;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
  prof_begin(st, "rhs");
  rhs_kernel<<<blocks, 256, 0, st>>>(p->B, p->N, p->M, p->f, p->inflow, p->ax, p->ay, p->sgx, p->sgy, b);
  after_launch("rhs", st, 0.0, 4.0 * (double)n + 4.0 * p->ncell, 0);
}

void launch_apply_f32(const rte_problem* p, const float* x, float* y, const double* alpha, int alpha_stride,
                      cudaStream_t st) {
  if (p->kind == 1) {
    launch_tfps_apply<float>(p, x, y, alpha, alpha_stride, nullptr, st);
    return;
  }
  if (p->kind == 2) {
    launch_atfps<float>(p, 0, x, y, alpha, alpha_stride, nullptr, st);
    return;
  }
  if (p->tc_apply) {
    launch_apply_tc(p, x, y, alpha, alpha_stride, st);
    return;
  }
  prof_begin(st, "apply_f32_simt");
  launch_simt<float>(p, x, y, p->St32, p->sig_d, p->sig_s, p->ax, p->ay, nullptr, alpha, alpha_stride, st);
  after_launch("apply_f32_simt", st, apply_flops(p), apply_bytes(p, 4, 0), 2);
}

void launch_apply_f64(const rte_problem* p, const double* x, double* y, const float* b, cudaStream_t st) {
  if (p->kind == 1) {
    launch_tfps_apply<double>(p, x, y, nullptr, 0, b, st);
    return;
  }
  if (p->kind == 2) {
    launch_atfps<double>(p, 0, x, y, nullptr, 0, b, st);
    return;
  }
  prof_begin(st, "apply_f64_simt");
  launch_simt<double>(p, x, y, p->St64, p->sig_d64, p->sig_s64, p->ax64, p->ay64, b, nullptr, 0, st);
  after_launch("apply_f64_simt", st, apply_flops(p), apply_bytes(p, 8, b ? 4 : 0), 3);
}

}  // namespace rte
