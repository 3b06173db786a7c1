// rte_apply on the tcgen05 tensor cores: the scattering contraction Psi[cells x M] . S^T[M x M]
// (eq:DORTE_2d with the row-normalised HG matrix, R4-R5) as a 3xTF32
// GEMM (tc_gemm.cuh, mode 0 / 1x1 "conv" with Ci = Co = M), fused with the upwind stencil and
// the sigma_t diagonal in the epilogue (R9):
//   y_{jim} = alpha [ (|c_m|/h + |s_m|/h + sigma_t) psi_{jim} - sigma_s (Psi S^T)_{jim}
//                     - (|c_m|/h) psi_{j,i-sgn c_m,m} - (|s_m|/h) psi_{j-sgn s_m,i,m} ]
// evaluated as stencil_diag (common.h): a_x (psi - nx) + a_y (psi - ny) + (sigma_t - sigma_s) psi
// + sigma_s ((psi - c) - [S (psi - c)]), the same operator with no sigma_t psi product to cancel.
// The epilogue runs warp-per-cell with lane = ordinate (coalesced 128-byte rows); psi at the cell
// and at its two upwind neighbours is re-read from L2 (the A tiles just streamed through it).
// Conservation-preserving contraction: because S is row-stochastic (R5),
// S psi = c + S (psi - c) for any per-cell scalar c.  The GEMM runs on psi - c with c = psi at the
// cell's first ordinate, so its rounding error scales with the anisotropic part of psi -- O(eps)
// in the diffusive regime, where sigma_t psi - sigma_s S psi cancels by ~1e3-1e4 -- instead of
// with psi itself (the tensor core's biased fp32 accumulation would otherwise not average out).
// Per-sample S (config 4) is selected by the B-operand row offset b*M.
#include <algorithm>

#include "common.h"
#include "tc_gemm.cuh"
#include "tc_host.h"

namespace rte {
namespace tc {

struct EpiApply {
  // The GEMM runs on psi - c (c = the cell's first ordinate, see the file header), so the
  // contraction is S psi = c + S (psi - c): exact because S is row-stochastic (R5).
  static constexpr bool kCenter = true;
  const float* x;
  float* y;
  const float* sig_d;  // sigma_t - sigma_s (= eps sigma_a)
  const float* sig_s;
  const float* ax;
  const float* ay;
  const int8_t* sgx;
  const int8_t* sgy;
  const double* alpha;
  int alpha_stride, N, M;

#ifndef RTE_APPLY_BATCH
#define RTE_APPLY_BATCH 2
#endif
  static constexpr int kBatch = RTE_APPLY_BATCH;  // rows whose global inputs are in flight together (measured best)
  struct Col {
    int m, sx, sy;
    float4 a_x, a_y;
  };
  struct Row {
    long long cell;
    int i, j;
    float sd, ss, al, c;
  };
  struct Pre {
    float4 p, nx, ny;  // psi at the cell and at its two upwind neighbours (0 at inflow faces)
  };
  // columns m .. m+3 share a quadrant (M % 16 == 0), hence both upwind signs
  __device__ __forceinline__ Col col(int m) const {
    return Col{m, sgx[m], sgy[m], *reinterpret_cast<const float4*>(ax + m), *reinterpret_cast<const float4*>(ay + m)};
  }
  struct Tile {
    long long cell0;  // cell of the tile origin
    float al;
  };
  __device__ __forceinline__ Tile tile(int b, int, int j0, int i0) const {
    return Tile{((long long)b * N + j0) * N + i0, alpha ? (float)alpha[(long long)b * alpha_stride] : 1.f};
  }
  __device__ __forceinline__ int rel(int ly, int lx) const { return ly * N + lx; }
  // tile pixel (oy, ox) of the class grid = cell (j, i)
  __device__ __forceinline__ Row row(const Tile& t, int rel, int j, int i, float c) const {
    const long long cell = t.cell0 + rel;
    return Row{cell, i, j, sig_d[cell], sig_s[cell], t.al, c};
  }
  __device__ __forceinline__ Pre load(const Row& rw, const Col& cv) const {
    const long long cell = rw.cell;
    const int m = cv.m, sx = cv.sx, sy = cv.sy;
    Pre q;
    q.p = *reinterpret_cast<const float4*>(x + cell * M + m);
    q.nx = make_float4(0.f, 0.f, 0.f, 0.f);
    q.ny = q.nx;
    if ((unsigned)(rw.i - sx) < (unsigned)N) q.nx = *reinterpret_cast<const float4*>(x + (cell - sx) * M + m);
    if ((unsigned)(rw.j - sy) < (unsigned)N) q.ny = *reinterpret_cast<const float4*>(x + (cell - (long long)sy * N) * M + m);
    return q;
  }
  __device__ __forceinline__ void store4(const Row& rw, const Col& cv, float4 v, const Pre& q) const {
    const float4 a_x = cv.a_x, a_y = cv.a_y, p = q.p, nx = q.nx, ny = q.ny;
    const float sd = rw.sd, ss = rw.ss, al = rw.al, c = rw.c;
    float4 r;
    r.x = al * stencil_diag(a_x.x, a_y.x, sd, ss, p.x, nx.x, ny.x, c, v.x);
    r.y = al * stencil_diag(a_x.y, a_y.y, sd, ss, p.y, nx.y, ny.y, c, v.y);
    r.z = al * stencil_diag(a_x.z, a_y.z, sd, ss, p.z, nx.z, ny.z, c, v.z);
    r.w = al * stencil_diag(a_x.w, a_y.w, sd, ss, p.w, nx.w, ny.w, c, v.w);
    __stcs(reinterpret_cast<float4*>(y + rw.cell * M + cv.m), r);  // evict-first: keeps the prefetched inputs in L2
  }
  __device__ __forceinline__ void store_partial4(int, const Row&, int, float4) const {}
};

// The same operator with the TMA epilogue (tc_gemm.cuh, APPLY = 2): the epilogue reads psi at the
// cell and its upwind neighbours from a TMA-loaded (TW + 2) x (TH + 2) halo chunk in shared memory
// (tmH, box 32 ordinates x (TW + 2) x (TH + 2), zero fill = inflow faces) and writes y through a
// swizzled staging tile and one bulk tensor store per chunk (tmY, box 32 x TW x TH).
struct EpiApplyT : EpiApply {
  static constexpr int kTmaEpi = 1;
  CUtensorMap tmH;
  CUtensorMap tmY;
};

template <int BN, class E>
void launch_apply_bn(const Geom& g, int mtiles, const CUtensorMap& ta, const CUtensorMap& tbh,
                     const CUtensorMap& tbl, const CUtensorMap& te, const E& epi, cudaStream_t st) {
  auto kern = gemm3xtf32_kernel<BN, 0, false, E>;
  constexpr int smem = gemm_smem_bytes<BN, 0, false, 1, tma_epi_of<E>::value ? 2 : 1>();
  ensure_smem((const void*)kern, smem);
  const int grid = std::min(mtiles * g.ntiles, num_sms());
  launch_gemm(kern, grid, smem, st, ta, tbh, tbl, te, g, epi);
}

}  // namespace tc

// this translation unit's copy of the role counters (tc_gemm.cuh g_tc_prof; experiments only)
void apply_tc_debug_counters(unsigned long long* out, int n, bool reset) {
  unsigned long long h[24];
  RTE_CHECK_CUDA(cudaMemcpyFromSymbol(h, tc::g_tc_prof, sizeof(h)));
  for (int i = 0; i < n && i < 24; ++i) out[i] += h[i];
  if (reset) {
    unsigned long long z[24] = {0};
    RTE_CHECK_CUDA(cudaMemcpyToSymbol(tc::g_tc_prof, z, sizeof(z)));
  }
}

bool apply_tc_supported(int M) { return M >= 32 && M <= 1024 && M % 32 == 0; }

void free_tc_state(rte_problem*) {}

void launch_apply_tc(const rte_problem* p, const float* x, float* y, const double* alpha, int alpha_stride,
                     cudaStream_t st) {
  const int N = p->N, M = p->M, B = p->B;
  int BN = 32;
  while (BN < 128 && BN * 2 <= M && M % (BN * 2) == 0) BN *= 2;
  tc::Geom g{};
  g.mode = 0;
  g.ks = 1;
  g.cchunks = M / 32;
  g.taps = 1;
  g.classes = 1;
  g.Hc = g.Wc = N;
  // 16 x 8-cell tiles: most upwind y-neighbours are rows of the same tile, which the epilogue's other
  // lanes have just loaded (a 128 x 1 strip takes every one from L2): apply 0.328 -> 0.291 ms at
  // config 5, also best at configs 3-4 (RTE_APPLY_TW overrides the width)
  static const int tw_env = getenv("RTE_APPLY_TW") ? atoi(getenv("RTE_APPLY_TW")) : 16;
  g.TW = std::min(N, std::max(1, std::min(128, tw_env)));
  g.TH = std::min(N, std::max(1, 128 / g.TW));
  g.pitch = g.TW;
  g.tiles_x = (N + g.TW - 1) / g.TW;
  g.tiles_y = (N + g.TH - 1) / g.TH;
  g.kb_total = g.cchunks;
  g.kb_per_split = g.kb_total;
  g.nsplit = 1;
  g.b_rows_class = 0;
  g.b_rows_batch = M;
  g.ntiles = M / BN;
  const int mtiles = B * g.tiles_y * g.tiles_x;
  g.mtiles = mtiles;
  g.bn = BN;
  g.dbg = tc::tc_debug_flags();
  g.epf = 2;  // prefetch x over the tile and its one-cell halo (cells and upwind neighbours)
  g.epf_planes = 1;
  CUtensorMap te = tc::make_map_prefetch(x, M, N, N, B, BN, g.TW + 2, g.TH + 2);  // (halo box, epi_prefetch)
  CUtensorMap ta = tc::make_map_act(x, M, N, N, B, g.TW, g.TH, 1);
  CUtensorMap tbh = tc::make_map_kmajor(p->S_hi, M, B * M, BN);
  CUtensorMap tbl = tc::make_map_kmajor(p->S_lo, M, B * M, BN);
  tc::EpiApply epi{x, y, p->sig_d, p->sig_s, p->ax, p->ay, p->sgx, p->sgy, alpha, alpha_stride, N, M};
  // TMA epilogue for N tiles of 64 / 128 whose halo box fits a slot (RTE_APPLY_OLDEPI: the per-lane
  // L2 epilogue, kept as the measured alternative)
  static const bool old_epi = getenv("RTE_APPLY_OLDEPI") != nullptr;
  const bool tma_epi = !old_epi && BN >= 64 && (g.TW + 2) * (g.TH + 2) <= tc::kHaloEpiRows;
  prof_begin(st, "apply_f32_tc");
  if (tma_epi) {
    tc::EpiApplyT et;
    static_cast<tc::EpiApply&>(et) = epi;
    et.tmH = tc::make_map_act(x, M, N, N, B, g.TW + 2, g.TH + 2, 1);
    et.tmY = tc::make_map_act(y, M, N, N, B, g.TW, g.TH, 1);
    if (BN == 64)
      tc::launch_apply_bn<64>(g, mtiles, ta, tbh, tbl, te, et, st);
    else
      tc::launch_apply_bn<128>(g, mtiles, ta, tbh, tbl, te, et, st);
  } else {
    switch (BN) {
      case 32: tc::launch_apply_bn<32>(g, mtiles, ta, tbh, tbl, te, epi, st); break;
      case 64: tc::launch_apply_bn<64>(g, mtiles, ta, tbh, tbl, te, epi, st); break;
      default: tc::launch_apply_bn<128>(g, mtiles, ta, tbh, tbl, te, epi, st); break;
    }
  }
  after_launch("apply_f32_tc", st, apply_flops(p), apply_bytes(p, 4, 0), p->M >= 256 ? 1 : 0);
}

}  // namespace rte
