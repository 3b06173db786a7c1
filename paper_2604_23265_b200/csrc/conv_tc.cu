// MgNet convolutions on the tcgen05 tensor cores, 3xTF32 (R26, §5).
//
// Every conv of the V-cycle is an implicit GEMM
//   out[pixels x Co] = sum_{tap, ci-chunk} X_shift(tap)[pixels x 32] . W_tap[Co x 32]^T
// run by the warp-specialised kernel of tc_gemm.cuh:
//   mode 0: 3x3 (or 1x1) stride 1, pad 1 (0)          -- smoother convs, lift, head
//   mode 1: 3x3 stride 2, pad 1 (TMA traversal stride 2) -- restriction R
//   mode 2: 4x4 stride-2 transposed, pad 1: split into its 4 output parity classes, each a
//           2x2 stride-1 conv on the coarse grid (sub-pixel decomposition) -- prolongation P
// The zero padding is the TMA out-of-bounds fill.  The epilogue fuses the smoother's residual /
// update (out = sign * s_in * acc + s_add * addend) and the Krylov scale alpha.  Small grids use
// deterministic split-K (fp32 partials, fixed-order reduction kernel that applies the epilogue).
// Shapes the kernel does not take (Ci % 32 != 0, Co not a multiple of the N tile) return false
// and run on the SIMT implicit GEMM in mgnet.cu.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <set>
#include <string>
#include <type_traits>
#include <vector>

#include "mgnet.h"
#include "tc_gemm.cuh"
#include "tc_host.h"

namespace rte {
namespace tc {

// ---- host helpers (tc_host.h) ------------------------------------------------------------
namespace {
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) {
    set_error("cuTensorMapEncodeTiled is not available from the driver");
    throw Fail{RTE_ECUDA};
  }
  return fn;
}

void encode(CUtensorMap* m, int rank, const void* base, const cuuint64_t* dims, const cuuint64_t* strides,
            const cuuint32_t* box, const cuuint32_t* es, bool swizzle = true) {
  CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)rank, const_cast<void*>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (code " + std::to_string((int)r) + ")");
    throw Fail{RTE_ECUDA};
  }
}
}  // namespace

CUtensorMap make_map_act(const float* base, int C, int W, int H, int B, int box_w, int box_h, int es) {
  CUtensorMap m;
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)C * 4, (cuuint64_t)W * C * 4, (cuuint64_t)H * W * C * 4};
  cuuint32_t box[4] = {32u, (cuuint32_t)(box_w * es), (cuuint32_t)(box_h * es), 1u};
  cuuint32_t est[4] = {1u, (cuuint32_t)es, (cuuint32_t)es, 1u};
  encode(&m, 4, base, dims, strides, box, est);
  return m;
}

CUtensorMap make_map_act_split(const float* base, int C, int W, int H, int B, int box_w, int box_h, int es) {
  CUtensorMap m;
  cuuint64_t dims[5] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, 2u, (cuuint64_t)B};
  const cuuint64_t plane = (cuuint64_t)H * W * C * 4;
  cuuint64_t strides[4] = {(cuuint64_t)C * 4, (cuuint64_t)W * C * 4, plane, 2 * plane};
  cuuint32_t box[5] = {32u, (cuuint32_t)(box_w * es), (cuuint32_t)(box_h * es), 1u, 1u};
  cuuint32_t est[5] = {1u, (cuuint32_t)es, (cuuint32_t)es, 1u, 1u};
  encode(&m, 5, base, dims, strides, box, est);
  return m;
}

// L2-prefetch map (no shared-memory destination, so no swizzle): [B'][H][W][C] fp32, box
// (box_c, box_w, box_h, 1)
CUtensorMap make_map_prefetch(const float* base, int C, int W, int H, int B, int box_c, int box_w, int box_h) {
  CUtensorMap m;
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)C * 4, (cuuint64_t)W * C * 4, (cuuint64_t)H * W * C * 4};
  cuuint32_t box[4] = {(cuuint32_t)box_c, (cuuint32_t)box_w, (cuuint32_t)box_h, 1u};
  cuuint32_t est[4] = {1u, 1u, 1u, 1u};
  encode(&m, 4, base, dims, strides, box, est, false);
  return m;
}

CUtensorMap make_map_kmajor(const float* base, int K, int rows, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 4};
  cuuint32_t box[2] = {32u, (cuuint32_t)box_rows};
  cuuint32_t est[2] = {1u, 1u};
  encode(&m, 2, base, dims, strides, box, est);
  return m;
}

float tf32_rna_host(float v) {
  uint32_t u;
  memcpy(&u, &v, 4);
  if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

void split_host(const std::vector<float>& w, std::vector<float>& hi, std::vector<float>& lo) {
  hi.resize(w.size());
  lo.resize(w.size());
  for (size_t i = 0; i < w.size(); ++i) {
    hi[i] = tf32_rna_host(w[i]);
    lo[i] = tf32_rna_host(w[i] - hi[i]);
  }
}

int tc_debug_flags() {
  static int v = [] {
    const char* e = getenv("RTE_TC_DBG");
    return e ? atoi(e) : 0;
  }();
  return v;
}

void ensure_smem(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::set<const void*> done;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(kernel)) return;
  RTE_CHECK_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.insert(kernel);
}

// ---- conv epilogue -------------------------------------------------------------------------
struct EpiConv {
  static constexpr bool kCenter = false;
  float* out;
  const float* addend;
  const double* alpha;
  float* part;            // split-K partials (nsplit x output elements) or NULL
  long long part_stride;  // elements per split
  float sign;
  int alpha_stride, a_in, a_add;
  int mode, Ho, Wo, Co;
  int out_split;  // output and addend stored as hi/lo planes (ConvDesc::out_split)
  const float* mod;  // CoeffNet modulation of the conv result (plain layout) or NULL

  __device__ __forceinline__ long long plane() const { return (long long)Ho * Wo * Co; }
  // offset of (pixel, col) in the output layout (plane 0 for split outputs)
  __device__ __forceinline__ long long index(int b, int cls, int oy, int ox, int col) const {
    int Y = oy, X = ox;
    if (mode == 2) {
      Y = 2 * oy + (cls >> 1);
      X = 2 * ox + (cls & 1);
    }
    return (((long long)b * (out_split ? 2 : 1) * Ho + Y) * Wo + X) * Co + col;
  }
  // offset of (pixel, col) in the plain partial-sum layout of split-K
  __device__ __forceinline__ long long pindex(int b, int cls, int oy, int ox, int col) const {
    int Y = oy, X = ox;
    if (mode == 2) {
      Y = 2 * oy + (cls >> 1);
      X = 2 * ox + (cls & 1);
    }
    return (((long long)b * Ho + Y) * Wo + X) * Co + col;
  }
#ifndef RTE_CONV_BATCH
#define RTE_CONV_BATCH 1
#endif
  static constexpr int kBatch = RTE_CONV_BATCH;  // rows whose global inputs are in flight together (measured best)
  struct Col {
    int col;
  };
  struct Row {
    long long o;  // output offset of column 0 of this pixel
    long long po; // partial-sum offset of column 0 (split-K)
    float si, sa;
  };
  struct Pre {
    float4 a;  // addend (hi + lo planes summed when split)
    float4 m;  // modulation (1 when none)
  };
  struct Tile {
    long long o0, po0;  // output / partial-sum offsets of the tile origin
    float si, sa;
  };
  __device__ __forceinline__ Col col(int c) const { return Col{c}; }
  __device__ __forceinline__ Tile tile(int b, int cls, int oy0, int ox0) const {
    const float al = alpha ? (float)alpha[(long long)b * alpha_stride] : 1.f;
    return Tile{index(b, cls, oy0, ox0, 0), pindex(b, cls, oy0, ox0, 0), sign * (a_in ? al : 1.f), a_add ? al : 1.f};
  }
  // class-grid step (ly, lx) -> output offset step (transposed conv: the class grid is stride 2)
  __device__ __forceinline__ int rel(int ly, int lx) const {
    return mode == 2 ? 2 * (ly * Wo + lx) * Co : (ly * Wo + lx) * Co;
  }
  __device__ __forceinline__ Row row(const Tile& t, int rel, int, int, float) const {
    return Row{t.o0 + rel, t.po0 + rel, t.si, t.sa};
  }
  __device__ __forceinline__ Pre load(const Row& rw, const Col& cv) const {
    Pre p{make_float4(0.f, 0.f, 0.f, 0.f), make_float4(1.f, 1.f, 1.f, 1.f)};
    if (mod) p.m = *reinterpret_cast<const float4*>(mod + rw.po + cv.col);
    if (addend) {
      const long long o = rw.o + cv.col;
      p.a = *reinterpret_cast<const float4*>(addend + o);
      if (out_split) {
        const float4 l = *reinterpret_cast<const float4*>(addend + o + plane());
        p.a.x += l.x;
        p.a.y += l.y;
        p.a.z += l.z;
        p.a.w += l.w;
      }
    }
    return p;
  }
  __device__ __forceinline__ void store4(const Row& rw, const Col& cv, float4 v, const Pre& p) const {
    const long long o = rw.o + cv.col;
    float4 r = make_float4(rw.si * (p.m.x * v.x), rw.si * (p.m.y * v.y), rw.si * (p.m.z * v.z), rw.si * (p.m.w * v.w));
    if (addend) {
      r.x = fmaf(rw.sa, p.a.x, r.x);
      r.y = fmaf(rw.sa, p.a.y, r.y);
      r.z = fmaf(rw.sa, p.a.z, r.z);
      r.w = fmaf(rw.sa, p.a.w, r.w);
    }
    if (out_split) {
      float4 h, l;
      split_tf32_fast(r.x, h.x, l.x);
      split_tf32_fast(r.y, h.y, l.y);
      split_tf32_fast(r.z, h.z, l.z);
      split_tf32_fast(r.w, h.w, l.w);
      *reinterpret_cast<float4*>(out + o) = h;
      *reinterpret_cast<float4*>(out + o + plane()) = l;
    } else {
      *reinterpret_cast<float4*>(out + o) = r;
    }
  }
  __device__ __forceinline__ void store_partial4(int split, const Row& rw, int col, float4 v) const {
    *reinterpret_cast<float4*>(part + split * part_stride + rw.po + col) = v;
  }
};

// The same epilogue through TMA (tc_gemm.cuh, APPLY = 3): the addend tile of each 32-channel chunk
// is bulk-loaded into shared memory ahead of the unit's K loop (tmAdd, box 32 x TW x TH), the output
// is written over it in place and bulk-stored (tmOut).  Dense single-split tiles without modulation
// or hi/lo output planes only (conv_tc_try); the arithmetic is EpiConv::store4's.
struct EpiConvT : EpiConv {
  static constexpr int kTmaEpi = 2;
  CUtensorMap tmAdd;
  CUtensorMap tmOut;
  CUtensorMap tmPart;  // split-K partials [nsplit * nb][Ho][Wo][Co] (box 32 x TW x TH)
  int nb;              // batch samples
};

// Deterministic split-K reduction + epilogue: out[e] = s_in * sum_s partial[s][e] + s_add * addend[e].
// With out_split the output (and the addend) are hi/lo planes: sample b's planes at 2b, 2b+1.
__global__ void splitk_reduce_kernel(const float4* __restrict__ part, long long stride4, int nsplit, float4* out,
                                     const float4* addend, float sign, const double* __restrict__ alpha,
                                     int alpha_stride, int a_in, int a_add, long long n4, long long per_sample4,
                                     int out_split, const float4* __restrict__ mod) {
  // programmatic dependent launch: let the next GEMM start its prologue, then wait for the GEMM
  // that wrote the partials (its completion and memory flush)
  griddep_launch_dependents();
  griddep_wait();
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n4; e += (long long)gridDim.x * blockDim.x) {
    float4 s = part[e];
    for (int k = 1; k < nsplit; ++k) {
      const float4 p = part[k * stride4 + e];
      s.x += p.x;
      s.y += p.y;
      s.z += p.z;
      s.w += p.w;
    }
    if (mod) {  // CoeffNet modulation of the conv result (plain layout, index e)
      const float4 m = mod[e];
      s.x *= m.x;
      s.y *= m.y;
      s.z *= m.z;
      s.w *= m.w;
    }
    const int b = (int)(e / per_sample4);
    const float al = alpha ? (float)alpha[(long long)b * alpha_stride] : 1.f;
    const float si = sign * (a_in ? al : 1.f), sa = a_add ? al : 1.f;
    float4 r = make_float4(si * s.x, si * s.y, si * s.z, si * s.w);
    // output offset: plain e, split (b, plane 0) = e + b * per_sample4
    const long long o = out_split ? e + (long long)b * per_sample4 : e;
    if (addend) {
      float4 a = addend[o];
      if (out_split) {
        const float4 l = addend[o + per_sample4];
        a.x += l.x;
        a.y += l.y;
        a.z += l.z;
        a.w += l.w;
      }
      r.x = fmaf(sa, a.x, r.x);
      r.y = fmaf(sa, a.y, r.y);
      r.z = fmaf(sa, a.z, r.z);
      r.w = fmaf(sa, a.w, r.w);
    }
    if (out_split) {
      float4 h, l;
      split_tf32_fast(r.x, h.x, l.x);
      split_tf32_fast(r.y, h.y, l.y);
      split_tf32_fast(r.z, h.z, l.z);
      split_tf32_fast(r.w, h.w, l.w);
      out[o] = h;
      out[o + per_sample4] = l;
    } else {
      out[o] = r;
    }
  }
}

}  // namespace tc

// ---- planning --------------------------------------------------------------------------------
namespace {

// Co-resident clusters of `cs` CTAs for the GEMM's footprint (448 threads, the largest shared
// plan: one CTA per SM); cached per cluster size.  GPC boundaries make this smaller than
// SMs / cs for large clusters, which the split-K cost model must see.
int max_active_clusters(int cs) {
  static int cache[9] = {0};
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (cs < 1 || cs > 8) return 0;
  if (cache[cs] == 0) {
    auto kern = tc::gemm3xtf32_kernel<128, 1, false, tc::EpiConv>;
    constexpr int smem = tc::gemm_smem_bytes<128, 1, false>();
    tc::ensure_smem((const void*)kern, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(cs * 64), 1, 1);
    cfg.blockDim = dim3(tc::kGemmThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
      (void)cudaGetLastError();
      n = -1;  // cluster launch unavailable: never plan it
    }
    cache[cs] = n;
  }
  return cache[cs];
}

struct Plan {
  bool ok = false;
  bool halo = false;  // stride-1 3x3: one halo tile per channel chunk feeds all 9 taps
  int am = 0;         // kernel A mode (tc_gemm.cuh Plan): 0 window, 1 TS halo, 2 SS halo
  int BN = 0;
  tc::Geom g{};
  int mtiles = 0, ntiles = 0;
  long long out_elems = 0;
};

Plan make_plan(const ConvDesc& d) {
  Plan P;
  if (d.Ci % 32 != 0 || d.Co % 32 != 0) return P;
  if (d.mode == 0 && !(d.ks == 1 || d.ks == 3)) return P;
  if (d.mode == 2 && (d.Ho % 2 || d.Wo % 2)) return P;
  static const int max_bn = [] {  // (experiments: RTE_TC_MAXBN caps the N tile)
    const char* e = getenv("RTE_TC_MAXBN");
    return e ? atoi(e) : 128;
  }();
  int BN = 32;
  while (BN < max_bn && BN * 2 <= d.Co && d.Co % (BN * 2) == 0) BN *= 2;
  P.BN = BN;
  P.halo = (d.mode == 0 && d.ks == 3);
  tc::Geom& g = P.g;
  g.mode = d.mode;
  g.ks = (d.mode == 2) ? 4 : d.ks;
  g.cchunks = d.Ci / 32;
  g.taps = (d.mode == 2) ? 4 : d.ks * d.ks;
  g.classes = (d.mode == 2) ? 4 : 1;
  g.Hc = (d.mode == 2) ? d.Ho / 2 : d.Ho;
  g.Wc = (d.mode == 2) ? d.Wo / 2 : d.Wo;
  // halo kernels use ~square 32 x 4 tiles (a 34 x 6 halo = 1.6 loaded rows per output row);
  // others 128-wide rows
  g.TW = std::min(g.Wc, P.halo ? 32 : 128);
  g.TH = std::max(1, 128 / g.TW);
  g.TH = std::min(g.TH, g.Hc);
  if (P.halo && (g.TW + 2) * (g.TH + 2) > tc::kHaloRows) {
    P.halo = false;
    g.TW = std::min(g.Wc, 128);
    g.TH = std::min(g.Hc, std::max(1, 128 / g.TW));
  }
  g.pitch = g.TW;
  P.am = P.halo ? 1 : 0;
  // SS halo (see tc_gemm.cuh): lines of P = 16 or 32 MMA rows, TW = P - 2 output pixels.  Opt-in
  // (RTE_TC_SS_MINW = the narrowest grid to use it on): measured shared-memory-bandwidth bound
  // (two 16 KB A reads per K block) and slower than the TS halo kernel on every MgNet level
  // (DESIGN.md §5); BN = 128 would need three A reads, so it is fused-form (BN <= 64) only
  static const int ss_minw = [] {
    const char* e = getenv("RTE_TC_SS_MINW");
    return e ? atoi(e) : 1 << 30;
  }();
  if (P.halo && !d.in_split && BN <= 64 && g.Wc >= ss_minw) {
    int bestP = 0;
    double best_eff = 0.0;
    for (int Pp : {32, 16}) {
      const int tx = (g.Wc + Pp - 3) / (Pp - 2);
      const double eff = (double)g.Wc / ((double)tx * Pp);
      if (eff > best_eff + 1e-9) {
        best_eff = eff;
        bestP = Pp;
      }
    }
    P.am = 2;
    g.pitch = bestP;
    g.TW = bestP - 2;
    g.TH = std::min(128 / bestP, g.Hc);
  }
  g.tiles_x = (g.Wc + g.TW - 1) / g.TW;
  g.tiles_y = (g.Hc + g.TH - 1) / g.TH;
  g.kb_total = g.taps * g.cchunks;
  g.b_rows_class = (d.mode == 2) ? d.Co : 0;
  g.b_rows_batch = 0;
  P.mtiles = d.B * g.classes * g.tiles_y * g.tiles_x;
  P.ntiles = d.Co / BN;
  g.ntiles = P.ntiles;
  g.mtiles = P.mtiles;
  g.bn = BN;
  g.dbg = tc::tc_debug_flags();
  P.out_elems = (long long)d.B * d.Ho * d.Wo * d.Co;
  // split-K from a wave model of the persistent kernel: time = ceil(units / SMs) * (k blocks per
  // unit * t_kb + t_unit) + (split-K reduction: (nsplit + 2) output-sized streams at ~6 TB/s)
  const int sms = num_sms();
  const double t_kb = (P.am == 2 ? (BN == 32 ? 400.0 : BN == 64 ? 500.0 : 800.0)  // SS MMA bound
                                  : std::max(12.0 * BN / 2.0, 700.0)) / 1.9e3;    // us per K block
  const double t_unit = 0.5;
  const double out_us = 4.0 * (double)P.out_elems / 6.0e6;
  // Cluster split-K (opt-in, RTE_TC_CLUSTER=1): the <= 8 splits of a tile run as one thread-block
  // cluster and reduce through distributed shared memory (no global partials, no reduction
  // launch; one unit per CTA, grid = units).  Measured on the MgNet coarse levels: about equal to
  // global partials + the reduction kernel, whose launches it removes but whose full-GPU
  // parallelism it loses (the finishing rows of a tile are 1/nsplit of the cluster's threads)
  static const bool cluster_ok = getenv("RTE_TC_CLUSTER") != nullptr;
  double best = 1e300;
  int best_kps = g.kb_total;
  // K-split granularity in K blocks.  A halo split may start or end inside a channel chunk (its
  // first K block loads the chunk's halo tile), so any K block boundary is allowed; the wave model
  // picks e.g. 9 splits of 32 K blocks for the 16 x 16 x 1024 conv (144 of 148 SMs busy, was 8 x
  // 36 on 128: 0.259 -> 0.234 ms/it at config 5).  RTE_TC_KQ=9 restores whole-chunk splits.
  static const int kq_env = getenv("RTE_TC_KQ") ? atoi(getenv("RTE_TC_KQ")) : 1;
  const int quantum = P.halo ? std::max(1, std::min(9, kq_env)) : 1;
  const int ns_max = cluster_ok ? 8 : 64;
  for (int ns = 1; ns <= std::max(1, std::min(ns_max, g.kb_total / (2 * quantum))); ++ns) {
    const int kps = ((g.kb_total + ns - 1) / ns + quantum - 1) / quantum * quantum;
    const int nsr = (g.kb_total + kps - 1) / kps;
    const long long units = (long long)P.mtiles * P.ntiles * nsr;
    double waves = (double)((units + sms - 1) / sms);
    if (cluster_ok && nsr > 1) {  // clusters of nsr CTAs: co-residency is per GPC, not per SM
      const int mc = max_active_clusters(nsr);
      if (mc <= 0) continue;
      const long long tiles = (long long)P.mtiles * P.ntiles;
      waves = (double)((tiles + mc - 1) / mc);
    }
    static const double red_fixed = getenv("RTE_TC_RED_US") ? atof(getenv("RTE_TC_RED_US")) : 3.0;
    const double red = nsr == 1 ? 0.0 : cluster_ok ? 1.0 : (nsr + 2) * out_us + red_fixed;
    const double t = waves * (kps * t_kb + t_unit) + red;
    if (t < best * 0.97) {
      best = t;
      best_kps = kps;
    }
  }
  g.kb_per_split = best_kps;
  g.nsplit = (g.kb_total + best_kps - 1) / best_kps;
  g.cl = (cluster_ok && g.nsplit > 1) ? g.nsplit : 0;
  static const bool planlog = getenv("RTE_TC_PLANLOG") != nullptr;  // (experiments)
  if (planlog)
    fprintf(stderr, "conv plan %s: BN=%d am=%d tiles=%dx%d kb=%d nsplit=%d cl=%d maxclusters(cl)=%d\n",
            conv_class_name(d, true), BN, P.am, P.mtiles, P.ntiles, g.kb_total, g.nsplit, g.cl,
            g.cl ? max_active_clusters(g.cl) : 0);
  P.ok = true;
  return P;
}

template <int BN, int AM, bool ASPLIT, int CPS = 1, class E = tc::EpiConv>
void launch_bn(const Plan& P, const CUtensorMap& ta, const CUtensorMap& tbh, const CUtensorMap& tbl,
               const CUtensorMap& te, const E& epi, cudaStream_t st) {
  auto kern = tc::gemm3xtf32_kernel<BN, AM, ASPLIT, E, CPS>;
  constexpr int smem = tc::gemm_smem_bytes<BN, AM, ASPLIT, CPS, tc::tma_epi_of<E>::value == 2 ? 3 : 0>();
  tc::ensure_smem((const void*)kern, smem);
  const long long units = (long long)P.mtiles * P.ntiles * P.g.nsplit;
  if (P.g.cl) {
    // one unit per CTA, the nsplit CTAs of a tile form a cluster (consecutive blockIdx.x)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)units, 1, 1);
    cfg.blockDim = dim3(tc::kGemmThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)P.g.cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    RTE_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tbh, tbl, te, P.g, epi));
    return;
  }
  const int grid = (int)std::min<long long>(units, (long long)CPS * num_sms());
  tc::launch_gemm(kern, grid, smem, st, ta, tbh, tbl, te, P.g, epi);
}

}  // namespace

bool conv_tc_try(const ConvDesc& d, const float* in, float* out, const float* addend, float sign,
                 const double* alpha, int alpha_stride, bool alpha_on_input, bool alpha_on_addend, cudaStream_t st) {
  if (!d.w || !d.w->d_hi || !d.ws_owner || !d.ws_owner->tc) return false;
  Plan P = make_plan(d);
  if (!P.ok) return false;
  // epilogue-input prefetch: the addend tile of each unit (dense output tiles only)
  if (addend && P.g.nsplit == 1 && d.mode != 2 && P.g.TW <= 256 && P.g.TH <= 256) {
    P.g.epf = 1;
    P.g.epf_planes = d.out_split ? 2 : 1;
  }
  const tc::Geom& g = P.g;
  const CUtensorMap te = g.epf ? tc::make_map_prefetch(addend, d.Co, d.Wo, d.Ho, d.B * g.epf_planes, P.BN, g.TW, g.TH)
                               : CUtensorMap{};
  const int es = (d.mode == 1) ? 2 : 1;
  // A box: SS halo (TH + 2) lines of P pixels; TS halo (TH + 2) x (TW + 2); else the TW x TH window
  const int bw = P.am == 2 ? g.pitch : P.halo ? g.TW + 2 : g.TW;
  const int bh = P.halo ? g.TH + 2 : g.TH, ees = P.halo ? 1 : es;
  CUtensorMap ta = d.in_split ? tc::make_map_act_split(in, d.Ci, d.Wi, d.Hi, d.B, bw, bh, ees)
                              : tc::make_map_act(in, d.Ci, d.Wi, d.Hi, d.B, bw, bh, ees);
  CUtensorMap tbh = tc::make_map_kmajor(d.w->d_hi, d.w->tc_K, d.w->tc_rows, P.BN);
  CUtensorMap tbl = tc::make_map_kmajor(d.w->d_lo, d.w->tc_K, d.w->tc_rows, P.BN);
  tc::EpiConv epi;
  epi.out = out;
  epi.addend = addend;
  epi.alpha = alpha;
  epi.sign = sign;
  epi.alpha_stride = alpha_stride;
  epi.a_in = alpha_on_input ? 1 : 0;
  epi.a_add = alpha_on_addend ? 1 : 0;
  epi.mode = d.mode;
  epi.Ho = d.Ho;
  epi.Wo = d.Wo;
  epi.Co = d.Co;
  epi.out_split = d.out_split ? 1 : 0;
  epi.mod = static_cast<const float*>(d.mod);
  epi.part = nullptr;
  epi.part_stride = P.out_elems;
  if (g.nsplit > 1 && !g.cl) {
    if ((long long)g.nsplit * P.out_elems > (long long)d.ws_owner->tc_ws_elems) {
      set_error("conv_tc: split-K workspace too small (internal planning mismatch)");
      throw Fail{RTE_EINTERNAL};
    }
    epi.part = d.ws_owner->tc_ws;
  }
  // TMA epilogue (RTE_CONV_OLDEPI: the per-lane global epilogue, kept as the measured alternative)
  static const bool conv_old_epi = getenv("RTE_CONV_OLDEPI") != nullptr;
  static const int tma_mask = getenv("RTE_CONV_TMA_MASK") ? atoi(getenv("RTE_CONV_TMA_MASK")) : 0xffff;
  const int mbit = (P.BN == 32 ? 0 : P.BN == 64 ? 2 : 4) + (P.halo ? 0 : 1) + (addend ? 8 : 0);
  const bool tma_epi = !conv_old_epi && !g.cl && !d.out_split && d.mod == nullptr &&
                       P.am != 2 && !d.in_split && (((tma_mask >> (mbit & 7)) & 1) != 0) && (((tma_mask >> 8) & 1) || !addend);
  tc::EpiConvT et;
  if (tma_epi) {
    static_cast<tc::EpiConv&>(et) = epi;
    // transposed convs (mode 2): a class tile is every other pixel of a 2TW x 2TH output box (stride-2 box)
    const int oes = d.mode == 2 ? 2 : 1;
    if (addend) et.tmAdd = tc::make_map_act(addend, d.Co, d.Wo, d.Ho, d.B, g.TW, g.TH, oes);
    et.tmOut = tc::make_map_act(out, d.Co, d.Wo, d.Ho, d.B, g.TW, g.TH, oes);
    et.nb = d.B;
    if (g.nsplit > 1) et.tmPart = tc::make_map_act(epi.part, d.Co, d.Wo, d.Ho, d.B * g.nsplit, g.TW, g.TH, oes);
    // the addend tiles are loaded ahead anyway -- by a whole K loop.  Units of one or two K blocks (the
    // head conv: K = C0) have no such lead: there the L2 prefetch one unit ahead stays on
    // (RTE_SHORTK_EPF=0 switches it off)
    static const bool shortk_epf = !(getenv("RTE_SHORTK_EPF") && atoi(getenv("RTE_SHORTK_EPF")) == 0);
    P.g.epf = (shortk_epf && g.epf == 1 && g.nsplit == 1 && g.kb_total <= 2) ? 1 : 0;
    // split-K fixup inside the kernel when every unit has its own resident CTA (tc_gemm.cuh Geom::fix):
    // no reduction launch.  Opt-in (RTE_TC_FIX=1): measured slower -- config-5 V-cycle 2.057 -> 2.130 ms;
    // the grid barrier waits for the slowest split and the reduction no longer overlaps the next
    // kernel's prologue
    static const bool nofix = getenv("RTE_TC_FIX") == nullptr;
    const int cps = (P.BN <= 64 && getenv("RTE_TC_CPS1") == nullptr) ? 2 : 1;
    const long long units = (long long)P.mtiles * P.ntiles * g.nsplit;
    P.g.fix = (!nofix && g.nsplit > 1 && units <= (long long)cps * num_sms()) ? 1 : 0;
  }
  prof_begin(st, conv_class_name(d, true));
  // BN = 32 kernels run two CTAs per SM (each half the TMEM, ~113 KB of shared memory): their
  // pipelines are hand-off-latency bound, so two of them per SM hide each other (RTE_TC_CPS1=1: one)
  static const bool two_per_sm = getenv("RTE_TC_CPS1") == nullptr;
  static const bool two_per_sm64 = two_per_sm;  // (N = 64 too: single halo slot per CTA, NG = 1)
  auto dispatch = [&](auto bn_tag) {
    constexpr int BN = decltype(bn_tag)::value;
    if (tma_epi) {
      if constexpr (BN <= 64) {
        if (two_per_sm) {
          if (P.halo) launch_bn<BN, 1, false, 2>(P, ta, tbh, tbl, te, et, st);
          else launch_bn<BN, 0, false, 2>(P, ta, tbh, tbl, te, et, st);
          return;
        }
      }
      if (P.halo) launch_bn<BN, 1, false, 1>(P, ta, tbh, tbl, te, et, st);
      else launch_bn<BN, 0, false, 1>(P, ta, tbh, tbl, te, et, st);
      return;
    }
    if (P.am == 2) {
      if constexpr (BN <= 64) launch_bn<BN, 2, false>(P, ta, tbh, tbl, te, epi, st);
    } else if (P.halo) {
      if (d.in_split) launch_bn<BN, 1, true>(P, ta, tbh, tbl, te, epi, st);
      else if constexpr (BN <= 64) {
        if ((BN == 32 ? two_per_sm : two_per_sm64) && !g.cl) launch_bn<BN, 1, false, 2>(P, ta, tbh, tbl, te, epi, st);
        else launch_bn<BN, 1, false>(P, ta, tbh, tbl, te, epi, st);
      } else launch_bn<BN, 1, false>(P, ta, tbh, tbl, te, epi, st);
    } else {
      if (d.in_split) launch_bn<BN, 0, true>(P, ta, tbh, tbl, te, epi, st);
      else if constexpr (BN <= 64) {
        if ((BN == 32 ? two_per_sm : two_per_sm64) && !g.cl) launch_bn<BN, 0, false, 2>(P, ta, tbh, tbl, te, epi, st);
        else launch_bn<BN, 0, false>(P, ta, tbh, tbl, te, epi, st);
      } else launch_bn<BN, 0, false>(P, ta, tbh, tbl, te, epi, st);
    }
  };
  switch (P.BN) {
    case 32: dispatch(std::integral_constant<int, 32>{}); break;
    case 64: dispatch(std::integral_constant<int, 64>{}); break;
    default: dispatch(std::integral_constant<int, 128>{}); break;
  }
  const bool split = g.nsplit > 1 && !g.cl && !g.fix;  // (cluster split-K and the fixup reduce in the kernel)
  after_launch(conv_class_name(d, true), st, conv_flops(d),
               split ? 0.0 : conv_bytes(d, addend != nullptr) + (g.fix ? 8.0 * g.nsplit * P.out_elems : 0.0), 1);
  if (split) {
    prof_begin(st, "splitk_reduce");
    const long long n4 = P.out_elems / 4;
    const long long per4 = n4 / d.B;
    const int blocks = (int)std::min<long long>((n4 + 255) / 256, (long long)num_sms() * 8);
    tc::launch_pdl(tc::splitk_reduce_kernel, blocks, 256, 0, st, reinterpret_cast<const float4*>(d.ws_owner->tc_ws),
                   n4, g.nsplit, reinterpret_cast<float4*>(out), reinterpret_cast<const float4*>(addend), sign,
                   alpha, alpha_stride, epi.a_in, epi.a_add, n4, per4, d.out_split ? 1 : 0,
                   reinterpret_cast<const float4*>(d.mod));
    // the conv's algorithmic bytes are booked on the reduction (it writes the output)
    after_launch("splitk_reduce", st, 0.0, conv_bytes(d, addend != nullptr) + 4.0 * g.nsplit * P.out_elems, 0);
  }
  return true;
}

// Upload the tensor-core operand layouts of every conv weight and size the split-K workspace.
// Per-role GEMM cycle counters (tc_gemm.cuh, RTE_TC_DBG bit 6): copy out and optionally reset.
void tc_debug_counters(unsigned long long* out, int n, bool reset) {
  unsigned long long h[24];
  RTE_CHECK_CUDA(cudaMemcpyFromSymbol(h, tc::g_tc_prof, sizeof(h)));
  for (int i = 0; i < n && i < 24; ++i) out[i] = h[i];
  if (reset) {
    unsigned long long z[24] = {0};
    RTE_CHECK_CUDA(cudaMemcpyToSymbol(tc::g_tc_prof, z, sizeof(z)));
  }
  apply_tc_debug_counters(out, n, reset);  // the apply kernels' copy (separate translation unit)
}

void conv_tc_prepare(mgnet_net* net) {
  net->tc = (getenv("RTE_DISABLE_TC") == nullptr);
  if (!net->tc) return;
  for (ConvW& w : net->convs) {
    std::vector<float> mat;
    if (w.kind == 0) {
      w.tc_rows = w.Co;
      w.tc_K = w.taps * w.Ci;
      mat = w.host_nk;  // [co][tap][ci]
    } else {
      // transposed 4x4: 4 parity classes (py,px) stacked as rows, K = (tap t, ci) with
      // ky = (py ? 0 : 1) + 2 (t >> 1), kx = (px ? 0 : 1) + 2 (t & 1)
      w.tc_rows = 4 * w.Co;
      w.tc_K = 4 * w.Ci;
      mat.assign((size_t)w.tc_rows * w.tc_K, 0.f);
      for (int cls = 0; cls < 4; ++cls)
        for (int co = 0; co < w.Co; ++co)
          for (int t = 0; t < 4; ++t)
            for (int ci = 0; ci < w.Ci; ++ci) {
              const int ky = ((cls >> 1) ? 0 : 1) + 2 * (t >> 1);
              const int kx = ((cls & 1) ? 0 : 1) + 2 * (t & 1);
              mat[((size_t)cls * w.Co + co) * w.tc_K + (size_t)t * w.Ci + ci] =
                  w.host_nk[((size_t)co * 16 + ky * 4 + kx) * w.Ci + ci];
            }
    }
    std::vector<float> hi, lo;
    tc::split_host(mat, hi, lo);
    w.d_hi = dalloc<float>(hi.size());
    upload(w.d_hi, hi.data(), hi.size());
    w.d_lo = dalloc<float>(lo.size());
    upload(w.d_lo, lo.data(), lo.size());
  }
  // split-K workspace: the largest nsplit * output over every conv shape of the V-cycle
  size_t need = 0;
  auto consider = [&](int mode, int ks, int Hi, int Ci, int Ho, int Co) {
    ConvDesc d;
    d.B = net->B;
    d.mode = mode;
    d.ks = ks;
    d.Hi = d.Wi = Hi;
    d.Ci = Ci;
    d.Ho = d.Wo = Ho;
    d.Co = Co;
    Plan P = make_plan(d);
    if (P.ok && P.g.nsplit > 1 && !P.g.cl) need = std::max(need, (size_t)P.g.nsplit * (size_t)P.out_elems);
  };
  consider(0, 1, net->N, net->M, net->N, net->C0);
  consider(0, 1, net->N, net->C0, net->N, net->M);
  for (int l = 0; l < net->L; ++l) {
    const Level& V = net->lv[l];
    consider(0, 3, V.H, V.C, V.H, V.C);
    if (l < net->L - 1) {
      consider(1, 3, V.H, V.C, V.H / 2, 2 * V.C);
      consider(2, 4, V.H / 2, 2 * V.C, V.H, V.C);
    }
  }
  if (need) {
    net->tc_ws = dalloc<float>(need);
    net->tc_ws_elems = need;
  }
}

}  // namespace rte
