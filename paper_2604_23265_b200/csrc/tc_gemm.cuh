// Warp-specialised, persistent 3xTF32 implicit GEMM on tcgen05 (sm_100a), shared by the MgNet
// convolutions (conv_tc.cu) and the scattering contraction of rte_apply (apply_tc.cu).  NOT part
// of the ABI.
//
// A work unit computes a 128-pixel x BN-channel output tile over a range of K blocks (split-K):
//   D[128 x BN] (TMEM, fp32) = sum_kb  A_kb[128 x 32] . B_kb[BN x 32]^T
// where a K block kb = (tap, 32-channel chunk).  A is an NHWC activation window fetched by a 4-D
// TMA tiled load whose out-of-bounds zero fill implements the convolution's zero padding; B_kb is
// a 32-wide K slice of the weights stored [rows][K] K-major (pre-split into TF32 hi and lo).
//
//  * HALO (stride-1 3x3 convs): one TMA load brings the (TW+2) x (TH+2) halo of the output tile
//    for a 32-channel chunk; the 9 taps read their shifted 128-pixel windows out of it, so the
//    input crosses L2 -> SM once per chunk instead of 9 times.  Other shapes load one A tile per
//    K block (shifted / strided window).
//  * 3xTF32 (R26): the converter warps read each A row from shared memory, split it
//    into hi + lo and store both into TMEM (tcgen05.st); the MMAs take A from TMEM and only the
//    weights from shared memory (the shared-memory port is the scarce resource).
//  * Accumulation precision: the tensor core's fp32 accumulation is not round-to-nearest, so the
//    main product hi.hi accumulates for at most kPromoteKB K blocks in one of two TMEM buffers
//    before promoter warps add it into fp32 registers; the small cross terms (lo.hi + hi.lo) go to
//    a separate accumulator.  For N tiles <= 64 a k-step is 2 MMAs (hi.[B_hi; B_lo] with N = 2BN
//    writing [main_t | X_t], then lo.B_hi into X_t); for BN = 128 it is 3 MMAs with a unit-long X.
//
// Warp roles (448 threads): warp 0 = TMA producer, warp 1 = TMEM allocator + MMA issuer (both walk
// the pipeline warp-wide, one elected lane issues), warps 2..5 = A converters (smem -> TMEM),
// warps 6..13 = promotion and epilogue (two warps per TMEM lane quarter, half the columns each);
// warp w accesses TMEM lanes 32*(w%4) .. +31.
// Pipelines: afull/aempty (A tiles), bfull/bempty (B tiles), conv/afree (TMEM A buffers),
// mfull/mempty (main accumulator buffers), xempty (unit-long X), cfull/cempty (row centres).
#pragma once

#include <cuda.h>
#include <stdint.h>

#include "tc_common.cuh"

namespace rte {
namespace tc {

constexpr int kGemmThreads = 448;   // 14 warps (see above)

// Launches a GEMM kernel with programmatic dependent launch (PDL: its prologue overlaps the previous
// kernel's tail; the kernel waits at griddepcontrol.wait before reading dependent data).
// RTE_NO_PDL=1 launches plainly.
template <typename K, typename... Args>
void launch_pdl(K kern, int grid, int block, int smem, cudaStream_t st, Args... args) {
  static const bool pdl = getenv("RTE_NO_PDL") == nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid, 1, 1);
  cfg.blockDim = dim3((unsigned)block, 1, 1);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  RTE_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}
template <typename K, typename... Args>
void launch_gemm(K kern, int grid, int smem, cudaStream_t st, Args... args) {
  launch_pdl(kern, grid, kGemmThreads, smem, st, args...);
}

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
  int kb_per_split; // (halo kernels: a multiple of 9)
  int nsplit;
  int b_rows_class; // B-operand row offset per class (mode 2)
  int b_rows_batch; // B-operand row offset per batch sample (per-sample operators)
  int ntiles;       // N tiles
  int mtiles;       // M tiles (B * classes * tiles_y * tiles_x)
  int bn;           // N tile (the kernel's BN)
  int pitch;        // MMA-tile rows per output line (= TW, or the halo pitch P of SS-halo kernels)
  int epf;          // epilogue-input L2 prefetch through tmE at each unit start: 0 none, 1 the
                    // output-shaped tile (conv addend; epf_planes planes), 2 the tile with its
                    // one-cell halo (apply: the cells and their upwind neighbours)
  int epf_planes;
  int fix;          // split-K fixup in the kernel (conv TMA epilogue, one unit per CTA, every CTA resident):
                    // after a grid barrier every CTA reduces a slice of the output (no reduction launch)
  int cl;           // cluster split-K: 0 off; else = nsplit, the K splits of one output tile run
                    // as one thread-block cluster (one unit per CTA) and are reduced through
                    // distributed shared memory (no global partials, no reduction launch)
  int dbg;          // perf-experiment switches (RTE_TC_DBG; 0 in production): bit0 converters skip
                    // the row load/split/TMEM store, bit3 no MMAs, bit4 no TMA loads, bit5 no
                    // epilogue global traffic, bit6 role timers
};

// Shared-memory plan: A ring (HALO: halo tiles of up to kHaloRows rows; else 128-row tiles), B
// ring, and the epilogue staging tiles (one 128 x 32 fp32 tile per column half).
constexpr int kHaloRows = 208;                  // (TW+2)(TH+2) <= 208, e.g. 34 x 6 for a 32 x 4 tile
constexpr int kSSRows = 200;                    // SS-halo tile: (TH+2) P + 2 rows <= 200 (P = 16, 32)
constexpr int kStageBytes = kTileM * 128;       // one staging tile: 128 rows x 32 fp32
// epilogue staging: per column half, one tile per 32-column chunk (BN = 128: 2 chunks)
template <int BN>
constexpr int stage_chunks() {
  return BN / 2 > 32 ? BN / 64 : 1;
}
// A modes: 0 = per-K-block window tiles (TS), 1 = halo tiles, 9 taps per tile (TS), 2 = SS halo:
// the halo tile is split once in shared memory and each tap's A operand is a row-shifted SW128
// descriptor into it (see the kernel comment).
#ifndef RTE_NA128
#define RTE_NA128 4  // A ring depth of the N = 128 apply (measured: 3 -> 4 is 4% on the apply, 5 no better)
#endif
#ifndef RTE_NA128C
#define RTE_NA128C 3  // ... and of the N = 128 window convs (strided / transposed / 1x1): the slot they
                      // free becomes a B slot for their long weight streams (e.g. the 32 x 1024
                      // transposed conv 0.039 -> 0.032 ms/it; the apply streams A and keeps 4)
#endif
// CPS = CTAs per SM (1, or 2 for BN = 32: two independent pipelines per SM hide each other's
// hand-off latency; each gets half of TMEM and ~113 KB of shared memory)
// TMA epilogue of the apply (APPLY = 2, Epi::kTmaEpi): per column half, RTE_EPI_HS halo slots of
// one 32-ordinate chunk of the tile's (TW + 2) x (TH + 2) cell box (<= 184 rows of 128 B, SW128) and
// one 128 x 32 output staging tile that a bulk tensor store drains
constexpr int kHaloEpiRows = 184;
constexpr int kHaloEpiBytes = kHaloEpiRows * 128;   // 23 KB: a multiple of the 1024-byte SW128 atom
#ifndef RTE_EPI_HS
#define RTE_EPI_HS 1
#endif
// TMA epilogue of a convolution (APPLY = 3, Epi::kTmaEpi == 2): one 128 x 32 tile per 32-column chunk
// of the unit, loaded with the addend by TMA, finished in place and drained by a bulk tensor store
template <int BN, int APPLY>
constexpr int epi_smem_bytes() {
  return APPLY == 2   ? 2 * (RTE_EPI_HS * kHaloEpiBytes + kStageBytes)
         : APPLY == 3 ? (BN / 32) * kStageBytes
                      : 2 * stage_chunks<BN>() * kStageBytes;
}
// Epi::kTmaEpi if the epilogue type declares it (1 = apply halo epilogue, 2 = conv tile epilogue), else 0
template <class E, class = void>
struct tma_epi_of {
  static constexpr int value = 0;
};
template <class E>
struct tma_epi_of<E, decltype(void(E::kTmaEpi))> {
  static constexpr int value = E::kTmaEpi;
};

// APPLY: 0 = convolution, 1 = apply (row-centred), 2 = apply with the TMA epilogue, 3 = convolution
// with the TMA epilogue
template <int BN, int AM, bool ASPLIT = false, int CPS = 1, int APPLY = 0>
struct Plan {
  static constexpr int kBBytes = BN * 128;                          // one of B hi / B lo
  static constexpr int kATile = AM == 2 ? kSSRows * 128 : AM == 1 ? kHaloRows * 128 : kABytes;
  static constexpr int kASlot = (ASPLIT || AM == 2 ? 2 : 1) * kATile;  // hi + lo tiles when split
  static constexpr int kBSlot = 2 * kBBytes;
  static constexpr int kBudget = (CPS == 1 ? 222 : 110) * 1024 - epi_smem_bytes<BN, APPLY>() -
                                 (APPLY == 2 ? 10 * 1024 : 0);  // rings (APPLY 2: minus the column table)
  // A ring depth: halo tiles are reused for 9 K blocks; window tiles are one K block each, so
  // they need a deeper ring to cover the HBM latency (BN = 32 leaves room for 8)
  // (CPS = 2, N = 64: a single halo slot -- the other CTA on the SM covers its load latency)
#ifndef RTE_HALO_NA32
#define RTE_HALO_NA32 2  // halo A slots of the two-per-SM N = 32 convs (experiments: the TMA epilogue frees 16 KB)
#endif
  static constexpr int kNA = (AM != 0 || ASPLIT) ? (CPS == 2 && BN == 64 ? 1 : CPS == 2 && BN == 32 && APPLY == 3 ? RTE_HALO_NA32 : 2)
                             : CPS == 2 ? (BN == 64 ? 2 : 3) : BN == 32 ? 8 : BN == 64 ? 4
                             : (APPLY == 1 || APPLY == 2) ? RTE_NA128 : RTE_NA128C;
  static constexpr int kNBraw = (kBudget - kNA * kASlot) / kBSlot;
  static constexpr int kNB = kNBraw > 8 ? 8 : kNBraw;               // B ring depth
  static_assert(kNB >= 1, "shared-memory plan leaves no B slot");
  static constexpr int kRingBytes = kNA * kASlot + kNB * kBSlot;
};

// TMA epilogue column table: per group of 4 ordinates {a_x[4], a_y[4]} and the two upwind halo-row
// offsets (M <= 1024: 256 groups)
constexpr int kColGroups = 256;
constexpr int kColTabBytes = kColGroups * (32 + 8);
template <int BN, int AM, bool ASPLIT = false, int CPS = 1, int APPLY = 0>
constexpr int gemm_smem_bytes() {
  return Plan<BN, AM, ASPLIT, CPS, APPLY>::kRingBytes + epi_smem_bytes<BN, APPLY>() + 1024 /*align*/ + 1024 /*barriers*/ +
         1024 /*row centres*/ + (APPLY == 2 ? kColTabBytes : 0);
}

// TMEM layout.  Fused form (BN <= 64): two group buffers t = 0, 1 of 2BN columns [main_t | X_t].
// Split form (BN = 128): main buffers M0, M1 [0, 2BN) and a unit-long X [2BN, 3BN).  Then the
// TMEM A buffers, 64 columns each (hi: 32 K columns, lo: 32 K columns).
template <int BN>
constexpr bool tmem_fused() {
  return BN <= 64;
}
// Fused form: NG group buffers of 2BN columns (the MMA can run NG - 1 groups ahead of the
// promoters, so a tile's epilogue overlaps the next tile's K loop) and 2 A buffers.
// Split form: 2 main buffers + X + the rest as A buffers.
// per-role cycle counters (dbg bit 6) are compiled in only with -DRTE_TC_PROF=1 (experiment builds:
// scripts/perf_roles.py); the production build keeps their registers free
#ifndef RTE_TC_PROF
#define RTE_TC_PROF 0
#endif
#ifndef RTE_CONV_EARLY_LOAD
#define RTE_CONV_EARLY_LOAD 1  // converters load + split before waiting for the TMEM A buffer
#endif
#ifndef RTE_TC_HALFK
#define RTE_TC_HALFK 1  // split form (BN = 128): the converter -> MMA hand-off runs in half K blocks (16 K
                        // columns): each TMEM A buffer has a barrier pair per half, so the MMAs of the
                        // first half issue while the converters still write the second, and a half is
                        // refilled as soon as its two k-steps retire
#endif
#ifndef RTE_TC_DEFER
#define RTE_TC_DEFER 0  // (experiment, off) fused-form halo convs (BN <= 64, the 32/64-channel levels): a K
                        // block's tcgen05.wait::st + arrive is deferred until the next K block's first
                        // pass is loaded and split.  Measured slower (level 0 0.371 -> 0.385 ms per
                        // V-cycle, level 1 0.266 -> 0.276): the converter -> MMA -> converter loop is
                        // latency-bound, and the deferral lengthens it
#endif
#ifndef RTE_EPI_BATCH_MAX
#define RTE_EPI_BATCH_MAX 8
#endif
#ifndef RTE_TC_NG_MAX
#define RTE_TC_NG_MAX 6
#endif
#ifndef RTE_TC_NA_MIN
#define RTE_TC_NA_MIN 2
#endif
// (TC = TMEM columns of one CTA: 512 / CPS)
#ifndef RTE_TC_NA_MIN32
#define RTE_TC_NA_MIN32 RTE_TC_NA_MIN  // (experiments: TMEM A buffers kept for the N = 32 kernels)
#endif
template <int BN, int TC = 512>
constexpr int tmem_groups() {
  constexpr int room = (TC - 64 * (BN == 32 ? RTE_TC_NA_MIN32 : RTE_TC_NA_MIN)) / (2 * BN);
  return tmem_fused<BN>() ? (room < RTE_TC_NG_MAX ? room : RTE_TC_NG_MAX) : 2;
}
template <int BN, int TC = 512>
constexpr int tmem_acc_cols() {
  return tmem_fused<BN>() ? tmem_groups<BN, TC>() * 2 * BN : 3 * BN;
}
template <int BN, int TC = 512>
constexpr int tmem_abufs() {
  return (TC - tmem_acc_cols<BN, TC>()) / 64 < 6 ? (TC - tmem_acc_cols<BN, TC>()) / 64 : 6;
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
  int split = 0;
  if (g.cl) {  // cluster split-K: the splits of a tile are consecutive CTAs (the cluster)
    split = u % g.cl;
    u /= g.cl;
  }
  const int nt = u % g.ntiles;
  u /= g.ntiles;
  const int mt = u % g.mtiles;
  w.split = g.cl ? split : u / g.mtiles;
  w.tc = decode_tile(g, mt);
  w.n0 = nt * g.bn;
  w.kb0 = w.split * g.kb_per_split;
  w.kb1 = min(g.kb_total, w.kb0 + g.kb_per_split);
  return w;
}

// K block kb -> (tap, channel chunk).  HALO kernels walk chunk-major (9 taps per halo tile).
template <bool HALO>
__device__ __forceinline__ void kb_split(const Geom& g, int kb, int& tap, int& cc) {
  if (HALO) {
    cc = kb / 9;
    tap = kb - 9 * cc;
  } else {
    tap = kb / g.cchunks;
    cc = kb - tap * g.cchunks;
  }
}

// A-window origin (x, y) in the input tensor for tap `tap` of tile c (non-halo kernels).
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

// dbg bit6: per-role cycle counters accumulated over all CTAs into g_tc_prof (experiments only;
// read with rte_debug_counters).  Slots: 0 producer total, 1 producer wait; 2 MMA total, 3 MMA
// wait conv+bfull, 4 MMA wait mempty/xempty, 5 MMA issue; 6 converter total, 7 converter wait,
// 8 converter work; 9 promoter total, 10 promoter wait mfull, 11 promoter TMEM loads,
// 12 epilogue; 13 K blocks (per CTA, producer); 14 converter K-block loop, 15 MMA K-block loop;
// 16 epilogue staging + first barrier, 17 epilogue row loop, 18 epilogue final barrier; 19 producer
// wait A slot, 20 producer A TMA issue, 21 producer B TMA issue; 22 MMA wait bfull; 23 converter
// wait afull.
__device__ unsigned long long g_tc_prof[24];

// Grid barrier of the in-kernel split-K fixup (Geom::fix): arrival count and generation.  Safe because
// the fixup is planned only when every CTA of the grid is resident (one unit per CTA, grid <= SMs) --
// a later kernel launched early by PDL cannot take an SM before all of this grid's CTAs have started --
// and a later kernel reaches its own barrier only after its griddepcontrol.wait (this grid complete).
__device__ unsigned int g_fix_cnt;
__device__ unsigned int g_fix_gen;

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void grid_barrier_fix() {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g0 = ld_acquire_u32(&g_fix_gen);
    asm volatile("fence.proxy.async.global;" ::: "memory");  // the bulk (async-proxy) partial stores
    __threadfence();
    if (atomicAdd(&g_fix_cnt, 1u) == gridDim.x - 1) {
      atomicExch(&g_fix_cnt, 0u);
      __threadfence();
      atomicAdd(&g_fix_gen, 1u);
    } else {
      while (ld_acquire_u32(&g_fix_gen) == g0) __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}

// (the warp stays converged: the timer is predicated, the wait is executed once by all lanes)
// Epilogue-input L2 prefetch for unit w (Geom::epf): the output-shaped tile (per plane), or the
// tile's rows oy0 - 1 .. oy0 + TH.
__device__ __forceinline__ void epi_prefetch(const Geom& g, const CUtensorMap* tmE, const Unit& w) {
  const int x0 = w.tc.tx * g.TW, y0 = w.tc.ty * g.TH;
  if (g.epf == 1) {
    for (int pl = 0; pl < g.epf_planes; ++pl) tma_prefetch_l2_4d(tmE, w.n0, x0, y0, w.tc.b * g.epf_planes + pl);
  } else {
    // the tile's cells and their upwind neighbours: one (TW + 2) x (TH + 2) box at (x0 - 1, y0 - 1)
    // (out-of-range coordinates at the domain edge are skipped by the TMA unit)
    tma_prefetch_l2_4d(tmE, w.n0, x0 - 1, y0 - 1, w.tc.b);
  }
}

__device__ __forceinline__ void tw_wait(uint64_t* bar, uint32_t par, bool on, long long& acc) {
  const long long t0 = on ? clock64() : 0;
  mbar_wait(bar, par);
  if (on) acc += clock64() - t0;
}

// Epilogue interface: cv = epi.col(col) holds per-column constants of columns col .. col+3;
// t = epi.tile(b, cls, oy0, ox0) the per-unit constants of the tile with origin (oy0, ox0);
// epi.rel(ly, lx) the output offset of tile pixel (ly, lx) relative to the origin's;
// row = epi.row(t, rel, oy, ox, c_row) the per-output-pixel state of a valid pixel (oy, ox) of the
// class grid (c_row = the row centre when Epi::kCenter: the GEMM then computed (a - c_row 1) . B^T);
// pre = epi.load(row, cv) issues the pixel's global inputs; epi.store4(row, cv, v4, pre) finishes
// the four columns; epi.store_partial4(split, row, col, v4) stores raw partial sums when split-K is
// active.  Epi::kBatch = rows whose loads are in flight together.
// ASPLIT: the A activation is stored pre-split as two planes (hi = rna_tf32(a), lo = a - hi; see
// EpiConv) and the tensor map has a plane dimension; the converters then only copy rows into
// TMEM.  Otherwise A is plain fp32 and the converters split it.
//
// SS halo (AM = 2, stride-1 3x3 convolutions): the output tile is TH lines of P = g.pitch MMA rows
// (P = 16 or 32) of which TW = P - 2 are output pixels (the last two rows of each line are computed
// and discarded).  The TMA loads the (TH + 2) x P halo of input lines at pitch P, so for tap
// (dy, dx) the A operand of output row r = ly P + lx is halo row r + dy P + dx: ONE contiguous
// 128-row slice, i.e. an SW128 descriptor starting dy P + dx rows in (the swizzle follows the
// absolute shared-memory address, so any row offset is valid; scripts/ss_offset_test.cu).  The
// converter warps split the halo once per tile in place (hi over the fp32 tile, lo into its twin)
// and the tensor core reads both straight from shared memory: no per-tap conversion, no TMEM A.
template <int BN, int AM, bool ASPLIT, class Epi, int CPS = 1>
__global__ void __launch_bounds__(kGemmThreads, CPS)
    gemm3xtf32_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBhi,
                      const __grid_constant__ CUtensorMap tmBlo, const __grid_constant__ CUtensorMap tmE,
                      const Geom g, const __grid_constant__ Epi epi) {
  constexpr bool HALO = AM != 0;
  constexpr bool SSH = AM == 2;
  static_assert(BN == 32 || BN == 64 || BN == 128, "N tile must be 32, 64 or 128");
  static_assert(!(HALO && Epi::kCenter), "row centring is for the 1x1 (apply) kernels");
  static_assert(!(ASPLIT && Epi::kCenter), "row centring needs the plain fp32 A operand");
  static_assert(!(SSH && ASPLIT), "SS-halo kernels split the activations themselves");
  static_assert(CPS == 1 || (CPS == 2 && BN <= 64 && !ASPLIT && AM != 2), "two CTAs per SM: BN <= 64 only");
  constexpr bool TMAEPI = tma_epi_of<Epi>::value == 1;  // apply: halo chunks + stencil
  constexpr bool CTEPI = tma_epi_of<Epi>::value == 2;   // conv: addend / output tiles
  static_assert(!TMAEPI || (Epi::kCenter && AM == 0 && !ASPLIT && CPS == 1 && BN >= 64), "TMA epilogue: apply kernels");
  static_assert(!CTEPI || (!Epi::kCenter && AM != 2 && !ASPLIT), "conv TMA epilogue: TS kernels");
  constexpr int HS = RTE_EPI_HS;
  static_assert(HS >= 1 && HS <= 2, "RTE_EPI_HS: 1 or 2 halo slots per half");
  using PL = Plan<BN, AM, ASPLIT, CPS, Epi::kCenter ? (TMAEPI ? 2 : 1) : (CTEPI ? 3 : 0)>;
  constexpr int TCOLS = 512 / CPS;
  constexpr int NAR = PL::kNA, NBR = PL::kNB;
  constexpr int NA = tmem_abufs<BN, TCOLS>();
  constexpr bool HK = RTE_TC_HALFK && !tmem_fused<BN>() && !SSH;  // half-K-block hand-off (see RTE_TC_HALFK)
  constexpr int NAH = HK ? 2 * NA : NA;     // conv / afree barriers of the TMEM A buffers
  constexpr int NCV = NAH > NAR ? NAH : NAR;  // conv barriers (SSH: one per A ring slot)
  constexpr int BBYTES = PL::kBBytes;
  constexpr uint32_t TMEM_COLS = TCOLS;
  constexpr bool FUSED = tmem_fused<BN>();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* aring = smem;
  uint8_t* bring = smem + NAR * PL::kASlot;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + PL::kRingBytes);
  uint64_t* afull = bars;              // [NAR] A tile landed
  uint64_t* aempty = afull + NAR;      // [NAR] converters done reading the A tile (4 warps)
  uint64_t* bfull = aempty + NAR;      // [NBR] B tiles landed
  uint64_t* bempty = bfull + NBR;      // [NBR] MMAs done with the B tiles
  uint64_t* conv = bempty + NBR;       // [NA] TMEM A buffer written (4 converter warps); SSH: A slot split
  uint64_t* afree = conv + NCV;        // [NA] MMAs done with the TMEM A buffer
  constexpr int NG = tmem_groups<BN, TCOLS>();
  uint64_t* mfull = afree + NAH;       // [NG] group buffer ready for promotion
  uint64_t* mempty = mfull + NG;       // [NG] group buffer drained (8 promoter warps)
  uint64_t* xempty = mempty + NG;      // [1] unit-long X drained (8 promoter warps)
  uint64_t* cfull = xempty + 1;        // [2] row centres written (128 converter threads)
  uint64_t* cempty = cfull + 2;        // [2] row centres read (256 epilogue threads)
  uint64_t* hfull = cempty + 2;        // [2 halves][HS] TMA epilogue: halo chunk landed; conv: [BN / 32] tile ready
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hfull + 4);
  float* cvec = reinterpret_cast<float*>(smem + PL::kRingBytes + 1024);  // [2][128] row centres
  const uint32_t stage_s = smem_u32(smem + PL::kRingBytes + 2048);        // [2 halves][chunks][128][32] staging
  // TMA epilogue column table (after the epilogue region): coltab[2g], coltab[2g + 1] = a_x, a_y of
  // ordinates 4g .. 4g+3 (one quadrant); coloff[g] = halo-row offsets of their x / y upwind neighbours
  // (pointers derived from smem_raw by an offset keep the shared state space: LDS / STS, not generic
  // LD / ST as through the uintptr_t-aligned `smem`)
  uint8_t* smem_sh = smem_raw + (smem_u32(smem) - smem_u32(smem_raw));
  float4* coltab = reinterpret_cast<float4*>(smem_sh + PL::kRingBytes + 2048 + epi_smem_bytes<BN, 2>());
  int2* coloff = reinterpret_cast<int2*>(coltab + 2 * kColGroups);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int units = g.mtiles * g.ntiles * g.nsplit;
  const int rows = g.pitch * g.TH;  // MMA-tile rows in use
  const uint32_t a_bytes = SSH    ? (uint32_t)((g.TH + 2) * g.pitch) * 128u
                           : HALO ? (uint32_t)((g.TW + 2) * (g.TH + 2)) * 128u
                                  : (uint32_t)rows * 128u;
  // bit6 enables the counters; bits 8..15 (if set) restrict them to kernels with that BN, bit16 to
  // halo kernels
  // (bit 17: only non-halo kernels, bit 18: only row-centred (apply) kernels, bit 19: only convs)
  const bool prof = RTE_TC_PROF && (g.dbg & 64) && lane == 0 && (((g.dbg >> 8) & 0xff) == 0 || ((g.dbg >> 8) & 0xff) == BN) &&
                    (!((g.dbg >> 16) & 1) || HALO) && (!((g.dbg >> 17) & 1) || !HALO) &&
                    (!((g.dbg >> 18) & 1) || Epi::kCenter) && (!((g.dbg >> 19) & 1) || !Epi::kCenter) &&
                    (((g.dbg >> 24) & 0x7f) == 0 || ((g.dbg >> 24) & 0x7f) == (g.kb_total & 0x7f));  // bits 24..30: K blocks (mod 128)
  long long w_d = 0, w_e = 0;
  long long w_a = 0, w_b = 0, w_c = 0;
  long long w_s1 = 0, w_s2 = 0, w_s3 = 0;
  const long long t_start = clock64();
  int n_kb = 0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NAR; ++i) {
      mbar_init(&afull[i], 1);
      mbar_init(&aempty[i], SSH ? 1 : 4);  // SSH: freed by the MMA commit after the 9th tap
    }
    for (int i = 0; i < NBR; ++i) {
      mbar_init(&bfull[i], 1);
      mbar_init(&bempty[i], 1);
    }
    for (int i = 0; i < NCV; ++i) mbar_init(&conv[i], 4);
    for (int i = 0; i < NAH; ++i) mbar_init(&afree[i], 1);
    for (int t = 0; t < NG; ++t) {
      mbar_init(&mfull[t], 1);
      mbar_init(&mempty[t], 8);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&cfull[t], 128);
      mbar_init(&cempty[t], 256);
    }
    mbar_init(xempty, 8);
    for (int i = 0; i < 4; ++i) mbar_init(&hfull[i], 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmBhi);
    tma_prefetch(&tmBlo);
    if (g.epf) tma_prefetch(&tmE);
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  if constexpr (TMAEPI) {  // (problem constants: no PDL wait needed)
    const int hw = g.TW + 2;
    for (int gi = threadIdx.x; gi < epi.M / 4; gi += blockDim.x) {
      const int m = 4 * gi;
      coltab[2 * gi] = *reinterpret_cast<const float4*>(epi.ax + m);
      coltab[2 * gi + 1] = *reinterpret_cast<const float4*>(epi.ay + m);
      coloff[gi] = make_int2(-(int)epi.sgx[m], -(int)epi.sgy[m] * hw);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // PDL: the next kernel in the stream may start its prologue as SMs free up; it waits for this
  // grid's completion (and memory) at its own griddepcontrol.wait before reading our outputs
  if (threadIdx.x == 0) griddep_launch_dependents();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tmem_x = tmem + 2 * BN;  // split form only
  const uint32_t tmem_a = tmem + tmem_acc_cols<BN, TCOLS>();

  if (warp == 0) {
    // ===== TMA producer: the whole warp walks the pipeline, one elected lane issues =====
    // every read of the previous kernel's outputs is causally after this wait (the A/B tiles here;
    // the epilogue's addend and maps through the pipeline barriers); a no-op without PDL
    // The B operand (weights, or S for the apply) is a constant of the problem, never a previous
    // kernel's output: the first unit's first NBR B tiles are requested *before* the PDL wait, so
    // their HBM latency overlaps the previous kernel's tail (dbg bit 22 switches this off; measured
    // neutral to +0.8% on the V-cycle.  Also pulling the rest of the unit's weight range towards L2
    // with bulk prefetches there was 7% slower: the prefetches compete with the previous kernel's tail)
    int b_pre = 0;
    if ((int)blockIdx.x < units && !(g.dbg & (1 << 22)) && !(g.dbg & 16)) {
      const Unit w = decode_unit(g, blockIdx.x);
      const int brow = w.n0 + w.tc.cls * g.b_rows_class + w.tc.b * g.b_rows_batch;
      b_pre = min(NBR, w.kb1 - w.kb0);
      if (elect_one()) {
        for (int i = 0; i < b_pre; ++i) {
          int tap, cc;
          kb_split<HALO>(g, w.kb0 + i, tap, cc);
          const int kcol = HALO ? tap * g.cchunks * 32 + cc * 32 : (w.kb0 + i) * 32;
          uint8_t* sb = bring + i * PL::kBSlot;
          mbar_arrive_expect_tx(&bfull[i], 2u * BBYTES);
          tma_load_2d(sb, &tmBhi, &bfull[i], kcol, brow);
          tma_load_2d(sb + BBYTES, &tmBlo, &bfull[i], kcol, brow);
        }
      }
      __syncwarp();
    }
    griddep_wait();
    int as = 0, bs = 0, b_cnt = 0;
    uint32_t aph = 0, bph = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const Unit w = decode_unit(g, u);
      const int brow = w.n0 + w.tc.cls * g.b_rows_class + w.tc.b * g.b_rows_batch;
      // epf = 2 (apply: long K loops): the producer's unit start is lead time enough
      if (g.epf == 2 && elect_one()) epi_prefetch(g, &tmE, w);
      __syncwarp();
      for (int kb = w.kb0; kb < w.kb1; ++kb, ++n_kb) {
        int tap, cc;
        kb_split<HALO>(g, kb, tap, cc);
        if (!HALO || tap == 0 || kb == w.kb0) {
          // new A tile: the halo of chunk cc (HALO) or the window of this K block
          tw_wait(&aempty[as], aph ^ 1, prof, w_a);
          int xA, yA;
          if (HALO) {
            xA = w.tc.tx * g.TW - 1;
            yA = w.tc.ty * g.TH - 1;
          } else {
            a_origin(g, w.tc, tap, xA, yA);
          }
          const long long tp0 = prof ? clock64() : 0;
          if (elect_one()) {
            if (g.dbg & 16) {
              mbar_arrive(&afull[as]);
            } else {
              uint8_t* sa = aring + as * PL::kASlot;
              if (ASPLIT) {  // 5-D map (C, W, H, plane, B): hi tile then lo tile
                mbar_arrive_expect_tx(&afull[as], 2u * a_bytes);
                tma_load_5d(sa, &tmA, &afull[as], cc * 32, xA, yA, 0, w.tc.b);
                tma_load_5d(sa + PL::kATile, &tmA, &afull[as], cc * 32, xA, yA, 1, w.tc.b);
              } else {
                mbar_arrive_expect_tx(&afull[as], a_bytes);
                tma_load_4d(sa, &tmA, &afull[as], cc * 32, xA, yA, w.tc.b);
              }
            }
          }
          __syncwarp();
          if (prof) w_s2 += clock64() - tp0;
          if (++as == NAR) { as = 0; aph ^= 1; }
        }
        if (b_cnt < b_pre) {  // requested before the PDL wait (slot b_cnt = bs, first use)
          ++b_cnt;
          if (++bs == NBR) { bs = 0; bph ^= 1; }
          continue;
        }
        tw_wait(&bempty[bs], bph ^ 1, prof, w_b);
        const long long tp1 = prof ? clock64() : 0;
        if (elect_one()) {
          uint8_t* sb = bring + bs * PL::kBSlot;
          const int kcol = HALO ? tap * g.cchunks * 32 + cc * 32 : kb * 32;
          if (g.dbg & 16) {
            mbar_arrive(&bfull[bs]);
          } else {
            mbar_arrive_expect_tx(&bfull[bs], 2u * BBYTES);
            tma_load_2d(sb, &tmBhi, &bfull[bs], kcol, brow);
            tma_load_2d(sb + BBYTES, &tmBlo, &bfull[bs], kcol, brow);
          }
        }
        __syncwarp();
        if (prof) w_s3 += clock64() - tp1;
        if (++bs == NBR) { bs = 0; bph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer: the whole warp walks the pipeline, one elected lane issues =====
    constexpr uint32_t idesc = idesc_tf32(kTileM, BN);
    const bool no_mma = (g.dbg & 8) != 0;
    int bs = 0, ab = 0, as = 0;
    uint32_t bph = 0, abph = 0, aph = 0;
    int gcount = 0;  // main-buffer groups issued so far (all units)
    int li = 0;      // local unit index
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++li) {
      const Unit w = decode_unit(g, u);
      if constexpr (!FUSED) {
        tw_wait(xempty, ((uint32_t)li & 1u) ^ 1u, prof, w_c);
        tc_fence_after();
      }
      uint32_t acc_x = 0;
      for (int kbg = w.kb0; kbg < w.kb1; kbg += kPromoteKB, ++gcount) {
        const int t = gcount % NG;
        tw_wait(&mempty[t], ((uint32_t)(gcount / NG) & 1u) ^ 1u, prof, w_b);
        tc_fence_after();
        uint32_t acc_m = 0;
        const int kbe = min(w.kb1, kbg + kPromoteKB);
        for (int kb = kbg; kb < kbe; ++kb, ++n_kb) {
          const long long tk0 = prof ? clock64() : 0;
          int tap = 0, cc = 0;
          if (SSH) kb_split<true>(g, kb, tap, cc);
          if (!SSH) tw_wait(&conv[HK ? 2 * ab : ab], abph, prof, w_a);
          else if (tap == 0 || kb == w.kb0) tw_wait(&conv[as], aph, prof, w_a);  // halo tile split
          tw_wait(&bfull[bs], bph, prof, w_s1);
          tc_fence_after();
          const uint32_t sb = smem_u32(bring + bs * PL::kBSlot);
          const uint64_t d_bh = sdesc_sw128(sb), d_bl = sdesc_sw128(sb + BBYTES);
          const uint32_t a_hi = tmem_a + (uint32_t)(64 * ab), a_lo = a_hi + 32;
          const long long ti0 = prof ? clock64() : 0;
          if (SSH && !no_mma) {
            // tap (dy, dx) = row shift dy P + dx into the split halo (hi tile, lo tile)
            const uint32_t sa = smem_u32(aring + as * PL::kASlot) + (uint32_t)((tap / 3) * g.pitch + tap % 3) * 128u;
            const uint64_t d_ah = sdesc_sw128(sa), d_al = sdesc_sw128(sa + PL::kATile);
            if constexpr (FUSED) {
              constexpr uint32_t idesc2 = idesc_tf32(kTileM, 2 * BN);
              const uint32_t tbuf = tmem + (uint32_t)(t * 2 * BN);
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                mma_tf32_elect(tbuf, d_ah + 2u * k, d_bh + 2u * k, idesc2, acc_m);
                acc_m = 1;
                mma_tf32_elect(tbuf + BN, d_al + 2u * k, d_bh + 2u * k, idesc, 1);
              }
            } else {
              const uint32_t tm = tmem + (uint32_t)(t * BN);
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                mma_tf32_elect(tmem_x, d_al + 2u * k, d_bh + 2u * k, idesc, acc_x);
                acc_x = 1;
                mma_tf32_elect(tmem_x, d_ah + 2u * k, d_bl + 2u * k, idesc, 1);
                mma_tf32_elect(tm, d_ah + 2u * k, d_bh + 2u * k, idesc, acc_m);
                acc_m = 1;
              }
            }
          } else if (!no_mma) {
            if constexpr (FUSED) {
              // hi.[B_hi; B_lo] -> [main_t | X_t] (N = 2BN), lo.B_hi -> X_t: one elected issue
              constexpr uint32_t idesc2 = idesc_tf32(kTileM, 2 * BN);
              const uint32_t tbuf = tmem + (uint32_t)(t * 2 * BN);
              mma_kblock_fused_ts(tbuf, tbuf + BN, a_hi, a_lo, d_bh, idesc2, idesc, acc_m);
              acc_m = 1;
            } else {
              const uint32_t tm = tmem + (uint32_t)(t * BN);
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                if constexpr (HK) {
                  if (k == 2) {  // first half retired -> refillable; second half written?
                    mma_commit_elect(&afree[2 * ab]);
                    tw_wait(&conv[2 * ab + 1], abph, prof, w_a);
                    tc_fence_after();
                  }
                }
                // K step of 8 tf32: +8 TMEM columns for A, +32 B (= +2) in the B descriptors
                mma_tf32_ts_elect(tmem_x, a_lo + 8u * k, d_bh + 2u * k, idesc, acc_x);
                acc_x = 1;
                mma_tf32_ts_elect(tmem_x, a_hi + 8u * k, d_bl + 2u * k, idesc, 1);
                mma_tf32_ts_elect(tm, a_hi + 8u * k, d_bh + 2u * k, idesc, acc_m);
                acc_m = 1;
              }
            }
          }
          if constexpr (HK) {
            if (no_mma) {  // (debug skeleton: keep the half hand-off protocol alive)
              mma_commit_elect(&afree[2 * ab]);
              tw_wait(&conv[2 * ab + 1], abph, prof, w_a);
            }
          }
          if (SSH) {
            mma_commit_elect(&bempty[bs]);
            if (tap == 8 || kb + 1 == w.kb1) {  // last tap of this halo tile: release the A slot
              mma_commit_elect(&aempty[as]);
              if (++as == NAR) { as = 0; aph ^= 1; }
            }
          } else {
            mma_commit2_elect(&bempty[bs], &afree[HK ? 2 * ab + 1 : ab]);
            if (++ab == NA) { ab = 0; abph ^= 1; }
          }
          if (prof) w_d += clock64() - ti0;
          if (++bs == NBR) { bs = 0; bph ^= 1; }
          if (prof) w_e += clock64() - tk0;
        }
        mma_commit_elect(&mfull[t]);
      }
    }
  } else if (SSH && warp < 6) {
    // ===== SS-halo converters (warps 2..5): split each halo tile once, in place =====
    const int tid = threadIdx.x - 64;
    int as = 0;
    uint32_t aph = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const Unit w = decode_unit(g, u);
      for (int kb = w.kb0; kb < w.kb1; ++kb, ++n_kb) {
        int tap, cc;
        kb_split<true>(g, kb, tap, cc);
        if (!(tap == 0 || kb == w.kb0)) continue;
        const long long tk0 = prof ? clock64() : 0;
        tw_wait(&afull[as], aph, prof, w_a);
        const long long tc0 = prof ? clock64() : 0;
        // elementwise, so the SW128 placement is irrelevant: hi = tf32 head in place, lo = rest
        const uint32_t base = smem_u32(aring + as * PL::kASlot);
        const int n16 = (int)(a_bytes >> 4);
#pragma unroll 4
        for (int i = tid; i < n16; i += 128) {
          const float4 v = lds128(base + (uint32_t)i * 16u);
          float4 h, l;
          split_tf32_fast(v.x, h.x, l.x);
          split_tf32_fast(v.y, h.y, l.y);
          split_tf32_fast(v.z, h.z, l.z);
          split_tf32_fast(v.w, h.w, l.w);
          sts128(base + (uint32_t)i * 16u, h);
          sts128(base + (uint32_t)PL::kATile + (uint32_t)i * 16u, l);
        }
        fence_proxy_async_smem();  // generic-proxy writes -> tensor-core (async proxy) reads
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[as]);
        if (++as == NAR) { as = 0; aph ^= 1; }
        if (prof) {
          w_d += clock64() - tc0;
          w_e += clock64() - tk0;
        }
      }
    }
  } else if (warp < 6) {
    // ===== converters (warps 2..5; warp w owns A rows / TMEM lanes 32*(w%4) .. +31) =====
    const int r = 32 * (warp & 3) + lane;  // output-tile row of this thread
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    const int rr = r < rows ? r : 0;       // rows beyond the tile read row 0 (results unused)
    const int ly = rr / g.TW, lx = rr - ly * g.TW;
    int as = 0, ab = 0;
    uint32_t aph = 0, abph = 0;
    int li = 0;
    // deferred publication (RTE_TC_DEFER): the TMEM A buffer whose stores are issued but not yet waited
    // for / announced; flushed before the next buffer's stores, before waiting for a new A tile (so the
    // MMAs never wait on a TMA load through it) and after the last unit
    constexpr bool DEFER = RTE_TC_DEFER && RTE_CONV_EARLY_LOAD && HALO && !HK && !ASPLIT && !Epi::kCenter;
    int pend = -1;
    auto flush_pend = [&]() {
      if (pend >= 0) {
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[pend]);
        pend = -1;
      }
    };
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++li) {
      const Unit w = decode_unit(g, u);
      float c = 0.f;
      for (int kb = w.kb0; kb < w.kb1; ++kb, ++n_kb) {
        const long long tk0 = prof ? clock64() : 0;
        int tap, cc;
        kb_split<HALO>(g, kb, tap, cc);
        const bool new_tile = !HALO || tap == 0 || kb == w.kb0;
        if (new_tile) {
          if constexpr (DEFER) flush_pend();
          tw_wait(&afull[as], aph, prof, w_a);
        }
#if !RTE_CONV_EARLY_LOAD
        tw_wait(&afree[HK ? 2 * ab : ab], abph ^ 1, prof, w_b);
        if (HK) tw_wait(&afree[2 * ab + 1], abph ^ 1, prof, w_b);
        tc_fence_after();
#endif
        // source row in the A tile: the tap-shifted halo row (HALO) or the row itself; 16-byte
        // chunk q of a row sits at chunk position q ^ (row & 7) (SW128)
        int arow = rr;
        if (HALO) arow = (ly + tap / 3) * (g.TW + 2) + lx + tap % 3;
        const uint32_t row_s = smem_u32(aring + as * PL::kASlot) + (uint32_t)arow * 128u;
        const bool skip = (g.dbg & 1) != 0;
        const long long tc0 = prof ? clock64() : 0;
        // the K block's 32 columns in passes of CWC (CPS = 2: 16, to fit the register budget)
        constexpr int CWC = (CPS == 1 && !HK) ? 32 : 16;
        const bool last_of_tile = !HALO || tap == 8 || kb + 1 == w.kb1;
        const uint32_t ta = tmem_a + (uint32_t)(64 * ab) + lane_base;
#pragma unroll
        for (int c0 = 0; c0 < 32; c0 += CWC) {
          float hi[CWC], lo[CWC];
#pragma unroll
          for (int q = 0; q < CWC / 4; ++q) {
            if (skip) break;
            const uint32_t qo = (uint32_t)(((c0 / 4 + q) ^ (arow & 7)) << 4);
            const float4 v = lds128(row_s + qo);
            hi[4 * q] = v.x;
            hi[4 * q + 1] = v.y;
            hi[4 * q + 2] = v.z;
            hi[4 * q + 3] = v.w;
            if (ASPLIT) {
              const float4 l = lds128(row_s + PL::kATile + qo);
              lo[4 * q] = l.x;
              lo[4 * q + 1] = l.y;
              lo[4 * q + 2] = l.z;
              lo[4 * q + 3] = l.w;
            }
          }
          // done with this A tile after its last K block's last pass
          if (last_of_tile && c0 + CWC == 32) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&aempty[as]);
            if (++as == NAR) { as = 0; aph ^= 1; }
          }
          if constexpr (Epi::kCenter) {
            // row centre c_r = the row's first element in the unit's first K block; the GEMM then
            // runs on a - c_r (see EpiApply); published to the epilogue through cvec
            if (kb == w.kb0 && c0 == 0) {
              c = hi[0];
              mbar_wait(&cempty[li & 1], ((uint32_t)(li >> 1) & 1u) ^ 1u);
              cvec[(li & 1) * 128 + r] = c;
              mbar_arrive(&cfull[li & 1]);
            }
          }
          if (!ASPLIT) {
#pragma unroll
            for (int e = 0; e < CWC; ++e) {
              const float x = Epi::kCenter ? hi[e] - c : hi[e];
              split_tf32_fast(x, hi[e], lo[e]);
            }
          }
#if RTE_CONV_EARLY_LOAD
          // the TMEM A buffer is needed only from here: the first pass's shared-memory loads and
          // split overlap the wait for the MMAs to release it
          if (HK || c0 == 0) {
            if constexpr (DEFER) flush_pend();
            tw_wait(&afree[HK ? 2 * ab + c0 / 16 : ab], abph ^ 1, prof, w_b);
            tc_fence_after();
          }
#endif
          if (!skip) {
            if constexpr (CWC == 32) {
              tmem_st32(ta, hi);
              tmem_st32(ta + 32, lo);
            } else {
              tmem_st16(ta + (uint32_t)c0, hi);
              tmem_st16(ta + 32 + (uint32_t)c0, lo);
            }
          }
          if constexpr (HK) {  // publish this half
            if (!skip) tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&conv[2 * ab + c0 / 16]);
          }
        }
        if constexpr (DEFER) {
          pend = ab;
        } else if constexpr (!HK) {
          if (!skip) tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&conv[ab]);
        }
        if (prof) w_d += clock64() - tc0;
        if (++ab == NA) { ab = 0; abph ^= 1; }
        if (prof) w_e += clock64() - tk0;
      }
    }
    if constexpr (DEFER) flush_pend();
  } else {
    // ===== promoters + epilogue (warps 6..13): warp w owns TMEM lanes 32*(w%4) .. +31 and the
    // column half h = (w - 6) / 4 of the tile =====
    constexpr int HB = BN / 2;  // columns per promoter warp
    const int quarter = warp & 3;
    const int half = (warp - 6) >> 2;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const int r = quarter * 32 + lane;  // tile row = TMEM lane
    const int cbase = half * HB;
    // epilogue row walk (unit-invariant): chunks of CW columns, LPR lanes per row, RPI rows per warp
    // instruction; lane's first row e_rr0 = (e_ly0, e_lx0) in the tile, then steps of RPI rows
    constexpr int CW = HB < 32 ? HB : 32;
    constexpr int LPR = CW / 4;
    constexpr int RPI = 32 / LPR;
    const int e_rr0 = quarter * 32 + lane / LPR;
    const int e_ly0 = e_rr0 / g.pitch, e_lx0 = e_rr0 - e_ly0 * g.pitch;
    const int e_dly = RPI / g.pitch, e_dlx = RPI - e_dly * g.pitch;
    int gcount = 0;
    // TMA epilogue (apply): this half's halo chunks s = li * ECH + j run through HS slots; the half's
    // leader (first warp of the half, lane 0) issues the loads ahead and drains the output staging
    constexpr int ECH = HB / 32 > 0 ? HB / 32 : 1;
    const bool hlead = TMAEPI && ((warp - 6) & 3) == 0 && lane == 0;
    const uint32_t epi_s = stage_s + (uint32_t)(half * (HS * kHaloEpiBytes + kStageBytes));
    const uint32_t ostage = epi_s + (uint32_t)(HS * kHaloEpiBytes);
    const uint32_t hbytes = (uint32_t)((g.TW + 2) * (g.TH + 2)) * 128u;
    auto issue_halo = [&](int s) {
      if constexpr (TMAEPI) {
        const int lj = s / ECH, j = s - lj * ECH;
        const int uu = (int)blockIdx.x + lj * (int)gridDim.x;
        if (uu >= units) return;
        const Unit w2 = decode_unit(g, uu);
        const int slot = s % HS;
        uint64_t* hb = &hfull[half * HS + slot];
        mbar_arrive_expect_tx(hb, hbytes);
        tma_load_4d(smem + (epi_s - smem_u32(smem)) + (uint32_t)(slot * kHaloEpiBytes), &epi.tmH, hb,
                    w2.n0 + 32 * (half * ECH + j), w2.tc.tx * g.TW - 1, w2.tc.ty * g.TH - 1, w2.tc.b);
      }
    };
    if (hlead) {
      griddep_wait();  // the halos read the previous kernel's output (PDL)
      for (int s = 0; s < HS; ++s) issue_halo(s);
    }
    // TMA epilogue (conv): chunk c of the unit lives in tile slot c (stage_s + c * 16 KB); a half owns
    // CPH chunks from cfirst (BN = 32: the one chunk is shared by both halves, half 0's leader drives it)
    constexpr int CCH = BN / 32;
    constexpr int CPH = CCH >= 2 ? CCH / 2 : 1;
    const bool clead = CTEPI && ((warp - 6) & 3) == 0 && lane == 0 && (CCH >= 2 || half == 0);
    const int cfirst = CCH >= 2 ? half * CPH : 0;
    const uint32_t tbytes = (uint32_t)(g.TW * g.TH) * 128u;
    if (clead) griddep_wait();  // the addend tiles may be the previous kernel's output (PDL)
    int li = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++li) {
      const Unit w = decode_unit(g, u);
      if constexpr (CTEPI) {
        if (clead) {
          // the previous unit's stores have read the slots; refill them with this unit's addend
          bulk_wait_read0();
          for (int c = cfirst; c < cfirst + CPH; ++c) {
            if (epi.addend && g.nsplit == 1) {
              // (transposed convs: class cls = (py, px) is the stride-2 box at (2 x0 + px, 2 y0 + py))
              const int ax = g.mode == 2 ? 2 * w.tc.tx * g.TW + (w.tc.cls & 1) : w.tc.tx * g.TW;
              const int ay = g.mode == 2 ? 2 * w.tc.ty * g.TH + (w.tc.cls >> 1) : w.tc.ty * g.TH;
              mbar_arrive_expect_tx(&hfull[c], tbytes);
              tma_load_4d(smem + (stage_s - smem_u32(smem)) + (uint32_t)(c * kStageBytes), &epi.tmAdd, &hfull[c],
                          w.n0 + 32 * c, ax, ay, w.tc.b);
            } else {
              mbar_arrive(&hfull[c]);
            }
          }
        }
      }
      if (g.epf == 1 && warp == 6 && lane == 0) {
        // pull the epilogue's global inputs into L2 one unit ahead (this unit's at the first):
        // far enough ahead to cover a short K loop, near enough that the output stream does not
        // evict them first (measured)
        if (li == 0) {
          // (after the PDL wait: an L2 prefetch of lines the previous kernel is still writing through
          // TMA stores was the suspected source of the stride-2 TMA-epilogue nondeterminism, §5)
          griddep_wait();
          epi_prefetch(g, &tmE, w);
        }
        if (u + (int)gridDim.x < units) epi_prefetch(g, &tmE, decode_unit(g, u + gridDim.x));
      }
      // TMA epilogue: this thread's cell constants, loaded while the K loop runs
      float t_sd = 0.f, t_ss = 0.f;
      if constexpr (TMAEPI) {
        const int ly = r / g.TW, lx = r - ly * g.TW;
        const int oy = w.tc.ty * g.TH + ly, ox = w.tc.tx * g.TW + lx;
        if (r < rows && oy < g.Hc && ox < g.Wc) {
          const long long cell = ((long long)w.tc.b * g.Hc + oy) * g.Wc + ox;
          t_sd = epi.sig_d[cell];
          t_ss = epi.sig_s[cell];
        }
      }
      float acc[HB];
#pragma unroll
      for (int i = 0; i < HB; ++i) acc[i] = 0.f;
      for (int kbg = w.kb0; kbg < w.kb1; kbg += kPromoteKB, ++gcount) {
        const int t = gcount % NG;
        {
          // one leader polls the mbarrier; the other promoter warps block on a hardware named
          // barrier (no issue slots spent polling), then order their TMEM loads after it
          const long long tw0 = prof ? clock64() : 0;
          if (warp == 6) mbar_wait(&mfull[t], (uint32_t)(gcount / NG) & 1u);
          named_bar_sync(4, 256);
          if (prof) w_a += clock64() - tw0;
        }
        tc_fence_after();
        const long long tl0 = prof ? clock64() : 0;
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
        if (prof) w_b += clock64() - tl0;
      }
      const long long te0 = prof ? clock64() : 0;
      if constexpr (!FUSED) {
        // the unit's last group commit covers every MMA of the unit, including the X buffer
#pragma unroll
        for (int c0 = 0; c0 < HB; c0 += 16) {
          float v[16];
          tmem_ld16(tmem_x + lane_base + (uint32_t)(cbase + c0), v);
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[c0 + i] += v[i];
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(xempty);
      }
      if constexpr (Epi::kCenter) mbar_wait(&cfull[li & 1], (uint32_t)(li >> 1) & 1u);
      if constexpr (CTEPI) {
        // ---- conv epilogue through TMA: thread = output pixel r (its TMEM lane); the addend tile of
        // each 32-column chunk is already in its slot; out = s_in v + s_add addend is written in place
        // and one bulk tensor store per chunk writes the tile (out-of-domain rows are clipped)
        const int e_oy0 = w.tc.ty * g.TH, e_ox0 = w.tc.tx * g.TW;
        const typename Epi::Tile et = epi.tile(w.tc.b, w.tc.cls, e_oy0, e_ox0);
#pragma unroll
        for (int cc = 0; cc < CPH; ++cc) {
          const int c = cfirst + cc;
          mbar_wait(&hfull[c], (uint32_t)li & 1u);
          float4* sp = reinterpret_cast<float4*>(smem_sh + (stage_s - smem_u32(smem)) + c * kStageBytes);
          constexpr int NQ = HB >= 32 ? 8 : HB / 4;  // float4 groups of this thread in the chunk
#pragma unroll
          for (int qq = 0; qq < NQ; ++qq) {
            const int q = HB >= 32 ? qq : half * NQ + qq;
            const float* v = &acc[HB >= 32 ? 32 * cc + 4 * qq : 4 * qq];
            float4& slot = sp[r * 8 + (q ^ (r & 7))];
            if (g.nsplit > 1) {  // split-K: the raw partial sums (EpiConv::store_partial4)
              slot = make_float4(v[0], v[1], v[2], v[3]);
              continue;
            }
            float4 o = make_float4(et.si * (1.f * v[0]), et.si * (1.f * v[1]), et.si * (1.f * v[2]), et.si * (1.f * v[3]));
            if (epi.addend) {
              const float4 a = slot;
              o.x = fmaf(et.sa, a.x, o.x);
              o.y = fmaf(et.sa, a.y, o.y);
              o.z = fmaf(et.sa, a.z, o.z);
              o.w = fmaf(et.sa, a.w, o.w);
            }
            slot = o;
          }
        }
        fence_proxy_async_smem();  // slot writes -> the bulk store (async proxy)
        if (CCH >= 2)
          named_bar_sync(2 + half, 128);
        else
          named_bar_sync(5, 256);
        if (clead) {
          const int sx = g.mode == 2 ? 2 * e_ox0 + (w.tc.cls & 1) : e_ox0;
          const int sy = g.mode == 2 ? 2 * e_oy0 + (w.tc.cls >> 1) : e_oy0;
          for (int c = cfirst; c < cfirst + CPH; ++c) {
            if (g.nsplit > 1)  // partial plane `split` of the [nsplit B][Ho][Wo][Co] workspace
              tma_store_4d(stage_s + (uint32_t)(c * kStageBytes), &epi.tmPart, w.n0 + 32 * c, sx, sy,
                           w.split * epi.nb + w.tc.b);
            else
              tma_store_4d(stage_s + (uint32_t)(c * kStageBytes), &epi.tmOut, w.n0 + 32 * c, sx, sy, w.tc.b);
          }
          bulk_commit();
        }
      } else if constexpr (TMAEPI) {
        // ---- apply epilogue through TMA: thread = cell r (its TMEM lane), 32
        // ordinates per chunk.  psi at the cell and at both upwind neighbours comes from the halo
        // chunk in shared memory (out-of-domain neighbours = the TMA's zero fill = the inflow
        // face), the outputs go to a swizzled staging tile that one bulk tensor store writes out.
        const int e_oy0 = w.tc.ty * g.TH, e_ox0 = w.tc.tx * g.TW;
        const typename Epi::Tile et = epi.tile(w.tc.b, w.tc.cls, e_oy0, e_ox0);
        const int hw = g.TW + 2;
        const int ly = r / g.TW, lx = r - ly * g.TW;
        (void)hw;
        // rows beyond the tile compute on a valid halo row; their staging rows are not stored
        const int hrow = r < rows ? (ly + 1) * hw + lx + 1 : hw + 1;
        const float cr = cvec[(li & 1) * 128 + r];
#pragma unroll
        for (int j = 0; j < ECH; ++j) {  // unrolled: acc stays in registers
          const int s = li * ECH + j;
          const long long tq0 = prof ? clock64() : 0;
          if (hlead) bulk_wait_read0();  // the previous chunk's store has read the staging tile
          named_bar_sync(2 + half, 128);
          const long long tq1 = prof ? clock64() : 0;
          mbar_wait(&hfull[half * HS + s % HS], (uint32_t)(s / HS) & 1u);
          const long long tq2 = prof ? clock64() : 0;
          // plain C++ shared-memory accesses (not volatile asm): the compiler may interleave the eight
          // column groups' loads; the barrier / mbarrier asm above and below carry memory clobbers
          const float4* hsp = reinterpret_cast<const float4*>(smem_sh + (epi_s - smem_u32(smem)) + (s % HS) * kHaloEpiBytes);
          float4* osp = reinterpret_cast<float4*>(smem_sh + (ostage - smem_u32(smem)));
          const int m0 = w.n0 + 32 * (half * ECH + j);
          const int g0 = m0 >> 2;  // columns 4g .. 4g+3 share a quadrant (M % 16 == 0)
          const float al = et.al;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 a_x = coltab[2 * (g0 + q)], a_y = coltab[2 * (g0 + q) + 1];
            const int2 off = coloff[g0 + q];
            const int rx = hrow + off.x, ry = hrow + off.y;
            const float4 p = hsp[hrow * 8 + (q ^ (hrow & 7))];
            const float4 nx = hsp[rx * 8 + (q ^ (rx & 7))];
            const float4 ny = hsp[ry * 8 + (q ^ (ry & 7))];
            const float* v = &acc[32 * j + 4 * q];
            float4 o;
            o.x = al * stencil_diag(a_x.x, a_y.x, t_sd, t_ss, p.x, nx.x, ny.x, cr, v[0]);
            o.y = al * stencil_diag(a_x.y, a_y.y, t_sd, t_ss, p.y, nx.y, ny.y, cr, v[1]);
            o.z = al * stencil_diag(a_x.z, a_y.z, t_sd, t_ss, p.z, nx.z, ny.z, cr, v[2]);
            o.w = al * stencil_diag(a_x.w, a_y.w, t_sd, t_ss, p.w, nx.w, ny.w, cr, v[3]);
            osp[r * 8 + (q ^ (r & 7))] = o;
          }
          const long long tq3 = prof ? clock64() : 0;
          fence_proxy_async_smem();  // staging writes -> the bulk store (async proxy)
          named_bar_sync(2 + half, 128);
          if (hlead) {
            tma_store_4d(ostage, &epi.tmY, m0, e_ox0, e_oy0, w.tc.b);
            bulk_commit();
            issue_halo(s + HS);  // every thread of the half has read this slot
          }
          if (prof) {  // slots 16 / 17 / 18: staging-free barrier, halo wait, compute (+ store barrier)
            w_s1 += tq1 - tq0;
            w_s2 += tq2 - tq1;
            w_s3 += clock64() - tq2;
          }
          (void)tq3;
        }
      } else {
      // Coalesced epilogue.  Each column chunk (<= 32 columns) of this half is staged through a
      // shared tile (row r at r*128 B, 16-byte chunk q at position q ^ (r & 7): conflict-free both
      // ways), then the half's four warps walk their rows with float4 lanes, so every global
      // load/store instruction covers whole rows (128 B each) instead of 32 scattered lines.
      constexpr int NCH = stage_chunks<BN>();
      const uint32_t sh = stage_s + (uint32_t)(half * NCH * kStageBytes);
      // per-unit epilogue state: tile origin in the class grid and the epilogue's tile constants
      const int e_oy0 = w.tc.ty * g.TH, e_ox0 = w.tc.tx * g.TW;
      const typename Epi::Tile et = epi.tile(w.tc.b, w.tc.cls, e_oy0, e_ox0);
      const long long ts0 = prof ? clock64() : 0;
      // stage every column chunk of this half first (the accumulators die here, leaving registers
      // for a batch of rows in flight below)
#pragma unroll
      for (int c0 = 0; c0 < HB; c0 += CW)
#pragma unroll
        for (int k = 0; k < CW / 4; ++k)
          sts128(sh + (uint32_t)((c0 / CW) * kStageBytes + r * 128 + ((k ^ (r & 7)) << 4)),
                 make_float4(acc[c0 + 4 * k], acc[c0 + 4 * k + 1], acc[c0 + 4 * k + 2], acc[c0 + 4 * k + 3]));
      named_bar_sync(2 + half, 128);
      const long long ts1 = prof ? clock64() : 0;
      if (prof) w_s1 += ts1 - ts0;
      if (!Epi::kCenter && g.cl) {
        // ---- cluster split-K: every CTA of the cluster staged its fp32 partial of the same
        // tile; CTA `rank` finishes rows [rank R, rank R + R) by summing the partials in rank
        // order (deterministic) straight out of the peers' shared memory, then the epilogue
        cluster_sync_all();  // phase 1: all partials staged
        const int ns = g.cl;
        const int R = (kTileM + ns - 1) / ns;
        const int rank = (int)cluster_ctarank();
        const int ptid = threadIdx.x - 192;  // 0..255 over the promoter warps
        constexpr int C4 = BN / 4;
        uint32_t peer[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) peer[q] = q < ns ? mapa_shared(stage_s, (uint32_t)q) : 0u;
        for (int item = ptid; item < R * C4; item += 256) {
          const int rr = rank * R + item / C4, c = 4 * (item % C4);
          if (rr >= rows || rr >= kTileM) continue;
          const int ly = rr / g.pitch, lx = rr - ly * g.pitch;
          const int oy = e_oy0 + ly, ox = e_ox0 + lx;
          if (lx >= g.TW || oy >= g.Hc || ox >= g.Wc) continue;
          const int h = c / HB, ch = c - h * HB, kq = (ch & 31) >> 2;
          const uint32_t off = (uint32_t)((h * NCH + (ch >> 5)) * kStageBytes + rr * 128 + ((kq ^ (rr & 7)) << 4));
          float4 v = ld_dsmem128(peer[0] + off);
          for (int q = 1; q < ns; ++q) {  // rank order: deterministic
            const float4 t = ld_dsmem128(peer[q] + off);
            v.x += t.x;
            v.y += t.y;
            v.z += t.z;
            v.w += t.w;
          }
          const typename Epi::Col cv = epi.col(w.n0 + c);
          const typename Epi::Row rw = epi.row(et, epi.rel(ly, lx), oy, ox, 0.f);
          epi.store4(rw, cv, v, epi.load(rw, cv));
        }
      } else if (!(g.dbg & 32)) {
        // rows are finished in batches: every global input of a batch (epi.row + epi.load) is
        // requested before any output of it is stored, so the batch costs one memory round trip
        // (out may alias the epilogue inputs elementwise only, which this order preserves)
        constexpr int NIT = 32 / RPI;
        constexpr int BMAX = Epi::kBatch < RTE_EPI_BATCH_MAX ? Epi::kBatch : RTE_EPI_BATCH_MAX;
        constexpr int BATCH = NIT < BMAX ? NIT : BMAX;
        const int k = lane % LPR;
#pragma unroll 1
        for (int c = 0; c < NCH; ++c) {
          const int col = w.n0 + cbase + c * CW + 4 * k;
          const typename Epi::Col cv = epi.col(col);
          const uint32_t shc = sh + (uint32_t)(c * kStageBytes);
          int ly = e_ly0, lx = e_lx0;  // tile-local pixel of this lane's row rr = e_rr0 + it * RPI
#pragma unroll 1
          for (int it0 = 0; it0 < NIT; it0 += BATCH) {
            typename Epi::Row rw[BATCH];
            typename Epi::Pre pre[BATCH];
            bool ok[BATCH];
#pragma unroll
            for (int q = 0; q < BATCH; ++q) {
              const int rr = e_rr0 + (it0 + q) * RPI;
              const int oy = e_oy0 + ly, ox = e_ox0 + lx;
              ok[q] = rr < rows && lx < g.TW && oy < g.Hc && ox < g.Wc;
              if (ok[q]) {
                const float crr = Epi::kCenter ? cvec[(li & 1) * 128 + rr] : 0.f;
                rw[q] = epi.row(et, epi.rel(ly, lx), oy, ox, crr);
                if (g.nsplit == 1 && !(g.dbg & (1 << 20))) pre[q] = epi.load(rw[q], cv);
              }
              lx += e_dlx;
              ly += e_dly;
              if (lx >= g.pitch) {
                lx -= g.pitch;
                ++ly;
              }
            }
#pragma unroll
            for (int q = 0; q < BATCH; ++q) {
              if (!ok[q] || (g.dbg & (1 << 21))) continue;
              const int rr = e_rr0 + (it0 + q) * RPI;
              const float4 v = lds128(shc + (uint32_t)(rr * 128 + ((k ^ (rr & 7)) << 4)));
              if (g.nsplit > 1)
                epi.store_partial4(w.split, rw[q], col, v);
              else
                epi.store4(rw[q], cv, v, pre[q]);
            }
          }
        }
      }
      const long long ts2 = prof ? clock64() : 0;
      named_bar_sync(2 + half, 128);
      if (prof) {
        const long long ts3 = clock64();
        w_s2 += ts2 - ts1;
        w_s3 += ts3 - ts2;
      }
      }
      if constexpr (Epi::kCenter) mbar_arrive(&cempty[li & 1]);
      if (prof) w_e += clock64() - te0;
    }
    if (hlead || clead) {
      bulk_wait0();  // every output store of this half is complete before the CTA exits
#ifdef RTE_EXP_GFENCE
      asm volatile("fence.proxy.async.global;" ::: "memory");
#endif
    }
  }
  if (g.cl) {
    if (warp < 6) cluster_sync_all();  // phase 1 (the promoters passed it inside the epilogue)
    cluster_sync_all();                // phase 2: no CTA leaves while peers read its partial
  }
  if (prof && (warp <= 2 || warp == 6)) {
    const unsigned long long tot = (unsigned long long)(clock64() - t_start);
    if (warp == 0) {
      atomicAdd(&g_tc_prof[0], tot);
      atomicAdd(&g_tc_prof[1], (unsigned long long)(w_a + w_b));
      atomicAdd(&g_tc_prof[13], (unsigned long long)n_kb);
      atomicAdd(&g_tc_prof[19], (unsigned long long)w_a);   // producer: wait A slot
      atomicAdd(&g_tc_prof[20], (unsigned long long)w_s2);  // producer: issue A TMA
      atomicAdd(&g_tc_prof[21], (unsigned long long)w_s3);  // producer: issue B TMAs
    } else if (warp == 1) {
      atomicAdd(&g_tc_prof[2], tot);
      atomicAdd(&g_tc_prof[3], (unsigned long long)w_a);
      atomicAdd(&g_tc_prof[4], (unsigned long long)(w_b + w_c));
      atomicAdd(&g_tc_prof[5], (unsigned long long)w_d);
      atomicAdd(&g_tc_prof[15], (unsigned long long)w_e);
      atomicAdd(&g_tc_prof[22], (unsigned long long)w_s1);  // MMA: wait bfull (in mma_wait_in: no)
    } else if (warp == 2) {
      atomicAdd(&g_tc_prof[6], tot);
      atomicAdd(&g_tc_prof[7], (unsigned long long)(w_a + w_b));
      atomicAdd(&g_tc_prof[8], (unsigned long long)w_d);
      atomicAdd(&g_tc_prof[14], (unsigned long long)w_e);
      atomicAdd(&g_tc_prof[23], (unsigned long long)w_a);  // converter: wait afull (new A tile)
    } else {
      atomicAdd(&g_tc_prof[9], tot);
      atomicAdd(&g_tc_prof[10], (unsigned long long)w_a);
      atomicAdd(&g_tc_prof[11], (unsigned long long)w_b);
      atomicAdd(&g_tc_prof[12], (unsigned long long)w_e);
      atomicAdd(&g_tc_prof[16], (unsigned long long)w_s1);
      atomicAdd(&g_tc_prof[17], (unsigned long long)w_s2);
      atomicAdd(&g_tc_prof[18], (unsigned long long)w_s3);
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CTEPI) {
    if (g.fix) {
      // ---- in-kernel split-K fixup: every partial tile is stored (the leaders waited for their bulk
      // stores); after the grid barrier CTA c reduces float4 slice c of the output, summing the splits
      // in order and applying the epilogue exactly as splitk_reduce_kernel does (bit-identical)
      grid_barrier_fix();
      const long long n4 = epi.part_stride / 4, per4 = n4 / epi.nb;
      const long long e0 = n4 * blockIdx.x / gridDim.x, e1 = n4 * (blockIdx.x + 1) / gridDim.x;
      const float4* part = reinterpret_cast<const float4*>(epi.part);
      float4* out4 = reinterpret_cast<float4*>(epi.out);
      const float4* add4 = reinterpret_cast<const float4*>(epi.addend);
      for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
        float4 sacc = __ldcg(part + e);
        for (int k = 1; k < g.nsplit; ++k) {
          const float4 q = __ldcg(part + k * n4 + e);
          sacc.x += q.x;
          sacc.y += q.y;
          sacc.z += q.z;
          sacc.w += q.w;
        }
        const int b = (int)(e / per4);
        const float al = epi.alpha ? (float)epi.alpha[(long long)b * epi.alpha_stride] : 1.f;
        const float si = epi.sign * (epi.a_in ? al : 1.f), sa = epi.a_add ? al : 1.f;
        float4 r = make_float4(si * sacc.x, si * sacc.y, si * sacc.z, si * sacc.w);
        if (add4) {
          const float4 a = __ldcg(add4 + e);
          r.x = fmaf(sa, a.x, r.x);
          r.y = fmaf(sa, a.y, r.y);
          r.z = fmaf(sa, a.z, r.z);
          r.w = fmaf(sa, a.w, r.w);
        }
        out4[e] = r;
      }
    }
  }
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

}  // namespace tc
}  // namespace rte
