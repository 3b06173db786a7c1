// Warp-specialised 3xTF32 implicit GEMM on tcgen05 (sm_100a), shared by the MgNet convolutions
// (conv_tc.cu) and the scattering contraction of rte_apply (apply_tc.cu).  NOT part of the ABI.
//
// One CTA computes a 128-pixel x BN-channel output tile over a range of K blocks (split-K):
//   D[128 x BN] (TMEM, fp32) = sum_kb  A_kb[128 x 32] . B_kb[BN x 32]^T
// where a K block kb = (tap, 32-channel chunk).  A_kb is a shifted (and for the stride-2
// restriction, strided) window of the NHWC activation, fetched by a 4-D TMA tiled load whose
// out-of-bounds zero fill implements the convolution's zero padding; B_kb is a 32-wide K slice of
// the weights stored [rows][K] K-major.  3xTF32 (R26): the converter warps read each A
// row once from shared memory, split it into hi + lo and store both into TMEM (tcgen05.st); the
// MMAs take A from TMEM and only the pre-split weights (B hi, B lo) from shared memory, which keeps
// the shared-memory traffic per K block at raw-A TMA write + one read + B (the SS form saturated
// the 128 B/clk shared-memory port).  Each k-step issues lo.hi + hi.lo (cross-term accumulator)
// and hi.hi (main accumulator).
//
// Warp roles (448 threads): warp 0 = TMA producer, warp 1 = TMEM allocator + MMA issuer (both walk
// the pipeline warp-wide, one elected lane issues), warps 2..5 = A hi/lo converters (smem -> TMEM),
// warps 6..13 = accumulator promotion and the epilogue (TMEM -> registers -> global; two warps per
// lane quarter, each owning half of the columns); warp w accesses TMEM lanes 32*(w%4) .. +31.  Pipelines:
// full[s] (TMA bytes landed) -> conv[s] (hi/lo written) -> empty[s] (MMAs done, tcgen05.commit);
// mfull[t] / mempty[t] hand the two main-accumulator TMEM buffers between MMA and promoters.
#pragma once

#include <cuda.h>
#include <stdint.h>

#include "tc_common.cuh"

namespace rte {
namespace tc {

constexpr int kGemmThreads = 448;   // 14 warps (see kernel)
constexpr int kPromoteKB = 4;       // K blocks per TMEM accumulation group
constexpr int kTileM = 128;
constexpr int kABytes = kTileM * 128;   // 128 rows x 32 fp32

// Geometry of the A/B K-block walk (see header comment).
struct Geom {
  int mode;         // 0: KSxKS stride 1 (pad KS/2); 1: 3x3 stride 2 pad 1; 2: 4x4 stride-2 transposed, per class
  int ks;           // mode 0/1 kernel size
  int cchunks;      // Ci / 32
  int taps;         // taps per output pixel (ks*ks, or 4 for mode 2)
  int TW, TH;       // output tile (TW*TH <= 128 pixels of the output (class) grid)
  int tiles_x, tiles_y;
  int classes;      // 1, or 4 parity classes (mode 2)
  int Hc, Wc;       // output (class) grid size
  int kb_total;     // taps * cchunks
  int kb_per_split;
  int nsplit;
  int b_rows_class; // B-operand row offset per class (mode 2)
  int b_rows_batch; // B-operand row offset per batch sample (per-sample operators)
  int ntiles;       // N tiles
  int mtiles;       // M tiles (B * classes * tiles_y * tiles_x)
  int bn;           // N tile (the kernel's BN)
  int dbg;          // perf-experiment switches (RTE_TC_DBG; 0 in production): bit0 skip the hi/lo
                    // conversion, bit1 skip the B-lo load and MMA, bit2 skip the cross-term MMAs,
                    // bit3 no MMAs at all, bit4 no TMA loads, bit5 no epilogue global traffic
};


template <int BN>
struct Smem {
  static constexpr int kBBytes = BN * 128;
  static constexpr int kStage = kABytes + 2 * kBBytes;   // raw A tile + B hi + B lo
};

template <int BN>
constexpr int gemm_stages() {
#ifdef RTE_TC_STAGES
  if (Smem<BN>::kStage * RTE_TC_STAGES <= 192 * 1024) return RTE_TC_STAGES;
#endif
  return Smem<BN>::kStage * 6 <= 192 * 1024 ? 6 : (192 * 1024) / Smem<BN>::kStage;
}

// TMEM layout.  Fused form (BN <= 64): two group buffers t = 0, 1 of 2BN columns [main_t | X_t];
// one MMA hi.[B_hi; B_lo] (N = 2BN) writes both halves and lo.B_hi (N = BN) adds into X_t, so a
// k-step costs 2 MMAs; both halves are promoted per group.  Split form (BN = 128): main buffers
// M0, M1 [0, 2BN) and a unit-long cross-term accumulator X [2BN, 3BN), 3 MMAs per k-step.  Then
// the A buffers, 64 columns each (hi: 32 K columns, lo: 32 K columns).
template <int BN>
constexpr bool tmem_fused() {
  return BN <= 64;
}
template <int BN>
constexpr int tmem_acc_cols() {
  return tmem_fused<BN>() ? 4 * BN : 3 * BN;
}
template <int BN>
constexpr int tmem_abufs() {
  return (512 - tmem_acc_cols<BN>()) / 64 < 6 ? (512 - tmem_acc_cols<BN>()) / 64 : 6;
}

template <int BN>
constexpr int gemm_smem_bytes() {
  return gemm_stages<BN>() * Smem<BN>::kStage + 1024 /*align*/ + 512 /*barriers*/ + 1024 /*row centres*/;
}

struct TileCoord {
  int b, cls, ty, tx;
};

__device__ __forceinline__ TileCoord decode_tile(const Geom& g, int t) {
  TileCoord c;
  c.tx = t % g.tiles_x;
  t /= g.tiles_x;
  c.ty = t % g.tiles_y;
  t /= g.tiles_y;
  c.cls = t % g.classes;
  c.b = t / g.classes;
  return c;
}

// Persistent schedule: CTA c processes work units u = c, c + gridDim.x, ...; a unit is
// (split, m tile, n tile) with the N tile fastest (consecutive units share their A tile in L2) and
// the split slowest (concurrent units share their K range of the weights).
struct Unit {
  TileCoord tc;
  int n0, split, kb0, kb1;
};

__device__ __forceinline__ Unit decode_unit(const Geom& g, int u) {
  Unit w;
  const int nt = u % g.ntiles;
  u /= g.ntiles;
  const int mt = u % g.mtiles;
  w.split = u / g.mtiles;
  w.tc = decode_tile(g, mt);
  w.n0 = nt * g.bn;
  w.kb0 = w.split * g.kb_per_split;
  w.kb1 = min(g.kb_total, w.kb0 + g.kb_per_split);
  return w;
}

// A-window origin (x, y) in the input tensor for K block kb of tile c.
__device__ __forceinline__ void a_origin(const Geom& g, const TileCoord& c, int tap, int& xA, int& yA) {
  if (g.mode == 0) {
    const int ky = tap / g.ks, kx = tap % g.ks, p = g.ks / 2;
    xA = c.tx * g.TW + kx - p;
    yA = c.ty * g.TH + ky - p;
  } else if (g.mode == 1) {
    const int ky = tap / 3, kx = tap % 3;
    xA = 2 * (c.tx * g.TW) + kx - 1;
    yA = 2 * (c.ty * g.TH) + ky - 1;
  } else {
    const int py = c.cls >> 1, px = c.cls & 1, ty_ = tap >> 1, tx_ = tap & 1;
    yA = c.ty * g.TH + (py ? 1 - ty_ : -ty_);
    xA = c.tx * g.TW + (px ? 1 - tx_ : -tx_);
  }
}

// Epilogue interface: row = epi.row(b, cls, oy, ox, c_row) prepares the per-output-pixel state of a
// valid pixel (oy, ox) of the class grid (c_row = the row centre when Epi::kCenter: the GEMM then
// computed (a - c_row 1) . B^T); epi.store4(row, col, v4) finishes columns col .. col+3;
// epi.store_partial4(split, row, col, v4) stores raw partial sums when split-K is active.
//
// Accumulation precision.  The tensor core's fp32 accumulation does not round to nearest (a
// biased, truncating add), so a long K loop into one TMEM accumulator drifts by ~K/8 * 2^-24
// relative.  Two measures keep the GEMM at fp32 accuracy:
//   - the small 3xTF32 cross terms (lo.hi + hi.lo, ~2^-11 of the result) go to their own TMEM
//     accumulator X, so the main accumulator sees one add per k-step;
//   - the main product hi.hi accumulates for at most kPromoteKB K blocks in one of two TMEM
//     buffers; four promoter warps then add the buffer into fp32 registers (round-to-nearest)
//     while the MMA warp fills the other buffer (the "promotion" used by FP8 GEMMs).
// dbg bit6: block 0 reports per-role cycles spent waiting (printf at exit; experiments only)
__device__ __forceinline__ void tw_wait(uint64_t* bar, uint32_t par, bool on, long long& acc) {
  if (!on) {
    mbar_wait(bar, par);
    return;
  }
  const long long t0 = clock64();
  mbar_wait(bar, par);
  acc += clock64() - t0;
}

template <int BN, class Epi>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm3xtf32_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBhi,
                      const __grid_constant__ CUtensorMap tmBlo, const Geom g, const Epi epi) {
  static_assert(BN == 32 || BN == 64 || BN == 128, "N tile must be 32, 64 or 128");
  constexpr int STAGES = gemm_stages<BN>();
  constexpr int NA = tmem_abufs<BN>();
  constexpr int BBYTES = Smem<BN>::kBBytes;
  constexpr int STAGE = Smem<BN>::kStage;
  constexpr uint32_t TMEM_COLS = 512;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* full = bars;                       // [STAGES] TMA bytes landed
  uint64_t* conv = bars + STAGES;              // [STAGES] A hi/lo in TMEM (4 converter warps)
  uint64_t* empty = bars + 2 * STAGES;         // [STAGES] MMAs done with the stage's B tiles
  uint64_t* afree = bars + 3 * STAGES;         // [NA] MMAs done with a TMEM A buffer
  uint64_t* mfull = afree + NA;                // [2] main buffer ready for promotion
  uint64_t* mempty = mfull + 2;                // [2] main buffer drained (4 promoter warps)
  uint64_t* xempty = mempty + 2;               // [1] cross buffer drained by the epilogue
  uint64_t* cfull = xempty + 1;                // [2] row centres written (128 converter threads)
  uint64_t* cempty = cfull + 2;                // [2] row centres read (128 epilogue threads)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cempty + 2);
  float* cvec = reinterpret_cast<float*>(smem + STAGES * STAGE + 512);  // [2][128] row centres

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int units = g.mtiles * g.ntiles * g.nsplit;
  const int rows = g.TW * g.TH;
  const uint32_t a_bytes = (uint32_t)rows * 128u;
  const bool prof = (g.dbg & 64) && blockIdx.x == 0 && lane == 0;
  long long w_a = 0, w_b = 0, w_c = 0;
  const long long t_start = clock64();
  int n_kb = 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 4);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < NA; ++a) mbar_init(&afree[a], 1);
    for (int t = 0; t < 2; ++t) {
      mbar_init(&mfull[t], 1);
      mbar_init(&mempty[t], 8);
      mbar_init(&cfull[t], 128);
      mbar_init(&cempty[t], 256);
    }
    mbar_init(xempty, 8);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmBhi);
    tma_prefetch(&tmBlo);
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr bool FUSED = tmem_fused<BN>();
  const uint32_t tmem_x = tmem + 2 * BN;  // split form only
  const uint32_t tmem_a = tmem + tmem_acc_cols<BN>();

  if (warp == 0) {
    // ===== TMA producer: the whole warp walks the pipeline, one elected lane issues =====
    int s = 0;
    uint32_t ph = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const Unit w = decode_unit(g, u);
      const int brow = w.n0 + w.tc.cls * g.b_rows_class + w.tc.b * g.b_rows_batch;
      for (int kb = w.kb0; kb < w.kb1; ++kb, ++n_kb) {
        tw_wait(&empty[s], ph ^ 1, prof, w_a);
        uint8_t* sa = smem + s * STAGE;
        const int tap = kb / g.cchunks, ci0 = (kb % g.cchunks) * 32;
        int xA, yA;
        a_origin(g, w.tc, tap, xA, yA);
        if (elect_one()) {
          if (g.dbg & 16) {
            mbar_arrive(&full[s]);
          } else {
            mbar_arrive_expect_tx(&full[s], a_bytes + 2u * BBYTES);
            tma_load_4d(sa, &tmA, &full[s], ci0, xA, yA, w.tc.b);
            tma_load_2d(sa + kABytes, &tmBhi, &full[s], kb * 32, brow);
            tma_load_2d(sa + kABytes + BBYTES, &tmBlo, &full[s], kb * 32, brow);
          }
        }
        __syncwarp();
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer: the whole warp walks the pipeline, one elected lane issues =====
    constexpr uint32_t idesc = idesc_tf32(kTileM, BN);
    const bool no_mma = (g.dbg & 8) != 0;
    int s = 0, ab = 0;
    uint32_t ph = 0;
    int gcount = 0;  // main-buffer groups issued so far (all units)
    int li = 0;      // local unit index
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++li) {
      const Unit w = decode_unit(g, u);
      tw_wait(xempty, ((uint32_t)li & 1u) ^ 1u, prof, w_c);
      tc_fence_after();
      uint32_t acc_x = 0;
      for (int kbg = w.kb0; kbg < w.kb1; kbg += kPromoteKB, ++gcount) {
        const int t = gcount & 1;
        tw_wait(&mempty[t], ((uint32_t)(gcount >> 1) & 1u) ^ 1u, prof, w_b);
        tc_fence_after();
        const uint32_t tm = tmem + (uint32_t)(t * BN);
        uint32_t acc_m = 0;
        const int kbe = min(w.kb1, kbg + kPromoteKB);
        for (int kb = kbg; kb < kbe; ++kb, ++n_kb) {
          tw_wait(&conv[s], ph, prof, w_a);
          tc_fence_after();
          const uint32_t sb = smem_u32(smem + s * STAGE) + kABytes;
          const uint64_t d_bh = sdesc_sw128(sb), d_bl = sdesc_sw128(sb + BBYTES);
          const uint32_t a_hi = tmem_a + (uint32_t)(64 * ab), a_lo = a_hi + 32;
          if (!no_mma) {
            if constexpr (FUSED) {
              // hi.[B_hi; B_lo] -> [main_t | X_t] (N = 2BN), lo.B_hi -> X_t
              constexpr uint32_t idesc2 = idesc_tf32(kTileM, 2 * BN);
              const uint32_t tbuf = tmem + (uint32_t)(t * 2 * BN);
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                mma_tf32_ts_elect(tbuf, a_hi + 8u * k, d_bh + 2u * k, idesc2, acc_m);
                acc_m = 1;
                mma_tf32_ts_elect(tbuf + BN, a_lo + 8u * k, d_bh + 2u * k, idesc, 1);
              }
            } else {
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                // K step of 8 tf32: +8 TMEM columns for A, +32 B (= +2) in the B descriptors
                mma_tf32_ts_elect(tmem_x, a_lo + 8u * k, d_bh + 2u * k, idesc, acc_x);
                acc_x = 1;
                mma_tf32_ts_elect(tmem_x, a_hi + 8u * k, d_bl + 2u * k, idesc, 1);
                mma_tf32_ts_elect(tm, a_hi + 8u * k, d_bh + 2u * k, idesc, acc_m);
                acc_m = 1;
              }
            }
          }
          mma_commit_elect(&empty[s]);
          mma_commit_elect(&afree[ab]);
          if (++s == STAGES) { s = 0; ph ^= 1; }
          if (++ab == NA) ab = 0;
        }
        mma_commit_elect(&mfull[t]);
      }
    }
  } else if (warp < 6) {
    // ===== converters (warps 2..5; warp w owns A rows / TMEM lanes 32*(w%4) .. +31) =====
    const int r = 32 * (warp & 3) + lane;  // A tile row of this thread
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    int s = 0, ab = 0, auses = 0;
    uint32_t ph = 0;
    int li = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++li) {
      const Unit w = decode_unit(g, u);
      float c = 0.f;
      for (int kb = w.kb0; kb < w.kb1; ++kb, ++n_kb) {
        tw_wait(&full[s], ph, prof, w_a);
        tw_wait(&afree[ab], ((uint32_t)(auses / NA) & 1u) ^ 1u, prof, w_b);
        tc_fence_after();
        // row r of the raw A tile: 16-byte chunk q sits at chunk position q ^ (r & 7) (SW128)
        const uint32_t row_s = smem_u32(smem + s * STAGE) + (uint32_t)r * 128u;
        float hi[32], lo[32];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 v = lds128(row_s + (uint32_t)((q ^ (r & 7)) << 4));
          hi[4 * q] = v.x;
          hi[4 * q + 1] = v.y;
          hi[4 * q + 2] = v.z;
          hi[4 * q + 3] = v.w;
        }
        if constexpr (Epi::kCenter) {
          // row centre c_r = the row's first element in the unit's first K block; the GEMM then
          // runs on a - c_r (see EpiApply); published to the epilogue through cvec
          if (kb == w.kb0) {
            c = hi[0];
            mbar_wait(&cempty[li & 1], ((uint32_t)(li >> 1) & 1u) ^ 1u);
            cvec[(li & 1) * 128 + r] = c;
            mbar_arrive(&cfull[li & 1]);
          }
        }
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float x = Epi::kCenter ? hi[e] - c : hi[e];
          split_tf32_fast(x, hi[e], lo[e]);
        }
        const uint32_t ta = tmem_a + (uint32_t)(64 * ab) + lane_base;
        tmem_st32(ta, hi);
        tmem_st32(ta + 32, lo);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[s]);
        if (++s == STAGES) { s = 0; ph ^= 1; }
        if (++ab == NA) ab = 0;
        ++auses;
      }
    }
  } else {
    // ===== promoters + epilogue (warps 6..13): warp w owns TMEM lanes 32*(w%4) .. +31 and the
    // column half h = (w - 6) / 4 of the tile (two warps per lane quarter double the epilogue's
    // memory-level parallelism) =====
    constexpr int HB = BN / 2;  // columns per promoter warp
    const int quarter = warp & 3;
    const int half = (warp - 6) >> 2;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const int r = quarter * 32 + lane;  // tile row = TMEM lane
    const int cbase = half * HB;
    int gcount = 0;
    int li = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++li) {
      const Unit w = decode_unit(g, u);
      float acc[HB];
#pragma unroll
      for (int i = 0; i < HB; ++i) acc[i] = 0.f;
      for (int kbg = w.kb0; kbg < w.kb1; kbg += kPromoteKB, ++gcount) {
        const int t = gcount & 1;
        tw_wait(&mfull[t], (uint32_t)(gcount >> 1) & 1u, prof, w_a);
        tc_fence_after();
        // fused form: main_t at t*2BN, X_t at t*2BN + BN; split form: main_t at t*BN
        const uint32_t mcol = FUSED ? (uint32_t)(t * 2 * BN) : (uint32_t)(t * BN);
#pragma unroll
        for (int c0 = 0; c0 < HB; c0 += 16) {
          float v[16];
          tmem_ld16(tmem + lane_base + mcol + (uint32_t)(cbase + c0), v);
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[c0 + i] += v[i];
          if constexpr (FUSED) {
            tmem_ld16(tmem + lane_base + mcol + (uint32_t)(BN + cbase + c0), v);
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[c0 + i] += v[i];
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&mempty[t]);
      }
      if constexpr (!FUSED) {
        // the unit's last group commit covers every MMA of the unit, including the X buffer
#pragma unroll
        for (int c0 = 0; c0 < HB; c0 += 16) {
          float v[16];
          tmem_ld16(tmem_x + lane_base + (uint32_t)(cbase + c0), v);
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[c0 + i] += v[i];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(xempty);
      float crow = 0.f;
      if constexpr (Epi::kCenter) {
        mbar_wait(&cfull[li & 1], (uint32_t)(li >> 1) & 1u);
        crow = cvec[(li & 1) * 128 + r];
        mbar_arrive(&cempty[li & 1]);
      }
      // Direct epilogue: thread r writes tile row r, columns cbase .. cbase + HB, as float4s.
      const int ly = r / g.TW, lx = r - ly * g.TW;
      const int oy = w.tc.ty * g.TH + ly, ox = w.tc.tx * g.TW + lx;
      if (r < rows && oy < g.Hc && ox < g.Wc && !(g.dbg & 32)) {
        const typename Epi::Row row = epi.row(w.tc.b, w.tc.cls, oy, ox, crow);
#pragma unroll
        for (int c = 0; c < HB; c += 4) {
          const float4 v = make_float4(acc[c], acc[c + 1], acc[c + 2], acc[c + 3]);
          if (g.nsplit > 1)
            epi.store_partial4(w.split, row, w.n0 + cbase + c, v);
          else
            epi.store4(row, w.n0 + cbase + c, v);
        }
      }
    }
  }
  if (prof && (warp <= 2 || warp == 6))
    printf("tcprof BN=%d units=%d grid=%d warp=%d kb=%d total=%lld waitA=%lld waitB=%lld waitC=%lld\n", BN, units,
           gridDim.x, warp, n_kb, clock64() - t_start, w_a, w_b, w_c);
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

}  // namespace tc
}  // namespace rte
