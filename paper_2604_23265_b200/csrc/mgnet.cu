// MgNet V-cycle (§3.3; R12-R20): linear smoother
//   u <- u + B * (f - A * u)   (modulation a = abar = 1, R13),
// stride-2 3x3 conv restriction of the residual, stride-2 4x4 transposed-conv prolongation,
// channel doubling C_l = C0 2^l, 1x1 lift Lambda (M -> C0) and head Theta (C0 -> M) with the
// pass-through P(r) = r + Theta u^0 (R17).  Activations are NHWC float32.
//
// Convolutions run as implicit GEMMs: D[pixels x Co] = sum_taps X_tap[pixels x Ci] . W_tap[Ci x Co].
// This file holds the SIMT (fp32 FMA) implicit-GEMM kernel used for every conv shape; the
// tcgen05 3xTF32 kernel (conv_tc.cu) takes the shapes it supports.
#include <algorithm>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <type_traits>
#include <vector>

#include "common.h"
#include "mgnet.h"
#include "tc_host.h"

namespace rte {
namespace {

// MODE 0: KSxKS conv, stride 1, pad KS/2.  MODE 1: 3x3 conv, stride 2, pad 1.
// MODE 2: 4x4 transposed conv, stride 2, pad 1, one output parity class per blockIdx.z % 4.
// out = (addend ? add_scale*addend : 0) + sign * in_scale * acc
template <typename T, int MODE, int KS, int TCO, bool IN_SPLIT, bool OUT_SPLIT>
__global__ void __launch_bounds__(256) conv_simt_kernel(
    int Hi, int Wi, int Ci, int Ho, int Wo, int Co, const T* __restrict__ in, const T* __restrict__ Wk,
    T* out, const T* addend, float sign, const double* __restrict__ alpha, int alpha_stride,
    int alpha_on_input, int alpha_on_addend, const T* __restrict__ mod) {
  // split formats (float only): value = hi plane + lo plane, planes Hi*Wi*Ci (in) / Ho*Wo*Co (out) apart
  // mod: CoeffNet modulation of the conv result, plain [B][Ho][Wo][Co] (NULL = 1)
  const int64_t in_plane = IN_SPLIT ? (int64_t)Hi * Wi * Ci : 0;
  const int64_t out_plane = OUT_SPLIT ? (int64_t)Ho * Wo * Co : 0;
  constexpr int TP = 4096 / TCO;
  constexpr int KC = 16;
  constexpr int TX = TCO / 4;
  constexpr int NTAPS = (MODE == 2) ? 4 : KS * KS;
  __shared__ __align__(16) T As[KC][TP + 4];
  __shared__ __align__(16) T Bs[KC][TCO + 4];
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  int bz = blockIdx.z;
  int py = 0, px = 0;
  int Hc = Ho, Wc = Wo;  // extent of the pixel set this block iterates
  if (MODE == 2) {
    int cls = bz & 3;
    bz >>= 2;
    py = cls >> 1;
    px = cls & 1;
    Hc = Ho / 2;
    Wc = Wo / 2;
  }
  const int b = bz;
  const int64_t npix = (int64_t)Hc * Wc;
  const int64_t p0 = (int64_t)blockIdx.x * TP;
  const int co0 = blockIdx.y * TCO;
  const T* inb = in + (int64_t)b * Hi * Wi * Ci * (IN_SPLIT ? 2 : 1);
  T acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[a][c] = T(0);

  for (int tap = 0; tap < NTAPS; ++tap) {
    int ky, kx;
    if (MODE == 2) {  // taps with ky = (py+1)%2 + 2*ty_, kx = (px+1)%2 + 2*tx_
      ky = ((py + 1) & 1) + 2 * (tap >> 1);
      kx = ((px + 1) & 1) + 2 * (tap & 1);
    } else {
      ky = tap / KS;
      kx = tap % KS;
    }
    const int wtap = (MODE == 2) ? (ky * 4 + kx) : tap;
    for (int ci0 = 0; ci0 < Ci; ci0 += KC) {
      for (int e = tid; e < TP * KC; e += 256) {
        int pl = e / KC, kk = e % KC;
        int64_t p = p0 + pl;
        T v = T(0);
        if (p < npix && ci0 + kk < Ci) {
          int yo = (int)(p / Wc), xo = (int)(p % Wc);
          int yi, xi;
          bool ok;
          if (MODE == 0) {
            yi = yo + ky - KS / 2; xi = xo + kx - KS / 2;
            ok = true;
          } else if (MODE == 1) {
            yi = 2 * yo + ky - 1; xi = 2 * xo + kx - 1;
            ok = true;
          } else {
            int Y = 2 * yo + py, X = 2 * xo + px;    // output pixel
            int yy = Y + 1 - ky, xx = X + 1 - kx;     // = 2*yi, 2*xi (even by construction)
            yi = yy >> 1; xi = xx >> 1;
            ok = (yy >= 0) && (xx >= 0);
          }
          ok = ok && yi >= 0 && yi < Hi && xi >= 0 && xi < Wi;
          if (ok) {
            const int64_t ii = ((int64_t)yi * Wi + xi) * Ci + ci0 + kk;
            v = inb[ii];
            if (IN_SPLIT) v += inb[ii + in_plane];
          }
        }
        As[kk][pl] = v;
      }
      for (int e = tid; e < KC * TCO; e += 256) {
        int kk = e / TCO, o = e % TCO;
        T v = T(0);
        if (ci0 + kk < Ci && co0 + o < Co) v = Wk[((int64_t)wtap * Ci + ci0 + kk) * Co + co0 + o];
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
  }
  const T al = alpha ? (T)alpha[(int64_t)b * alpha_stride] : T(1);
  const T s_in = (alpha_on_input ? al : T(1)) * (T)sign;
  const T s_add = alpha_on_addend ? al : T(1);
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    int64_t p = p0 + ty * 4 + a;
    if (p >= npix) continue;
    int64_t opix;
    if (MODE == 2) {
      int yo = (int)(p / Wc), xo = (int)(p % Wc);
      opix = (int64_t)(2 * yo + py) * Wo + (2 * xo + px);
    } else {
      opix = p;
    }
    int64_t base = ((int64_t)b * Ho * Wo * (OUT_SPLIT ? 2 : 1) + opix) * Co;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      int co = co0 + tx * 4 + c;
      if (co >= Co) continue;
      T v = s_in * (mod ? mod[((int64_t)b * Ho * Wo + opix) * Co + co] * acc[a][c] : acc[a][c]);
      if (addend) {
        T av = addend[base + co];
        if (OUT_SPLIT) av += addend[base + co + out_plane];
        v += s_add * av;
      }
      if constexpr (OUT_SPLIT) {
        const float hi = __uint_as_float((__float_as_uint((float)v) + 0x1000u) & 0xFFFFE000u);
        out[base + co] = hi;
        out[base + co + out_plane] = (float)v - hi;
      } else {
        out[base + co] = v;
      }
    }
  }
}

}  // namespace

// Algorithmic work of one conv launch: 2 * out_pixels * Co * Ci * taps_per_output
// flops (taps = k*k; the stride-2 transposed 4x4 conv touches 4 taps per output pixel); bytes =
// read the input once, the weights once, the addend once (if any), write the output once.
double conv_flops(const ConvDesc& d) {
  double taps = (d.mode == 2) ? 4.0 : (double)d.ks * d.ks;
  return 2.0 * d.B * (double)d.Ho * d.Wo * d.Co * d.Ci * taps;
}
double conv_bytes(const ConvDesc& d, bool has_addend) {
  double in = (double)d.B * d.Hi * d.Wi * d.Ci, out = (double)d.B * d.Ho * d.Wo * d.Co;
  double wts = (double)d.Co * d.Ci * ((d.mode == 2) ? 16.0 : (double)d.ks * d.ks);
  return 4.0 * (in + out * (has_addend ? 2.0 : 1.0) + wts);
}
const char* conv_class_name(const ConvDesc& d, bool tc) {
  const char* base;
  if (d.mode == 0 && d.ks == 1) base = tc ? "conv1x1_tc" : "conv1x1_simt";
  else if (d.mode == 0) base = tc ? "conv3x3_tc" : "conv3x3_simt";
  else if (d.mode == 1) base = tc ? "conv3x3s2_tc" : "conv3x3s2_simt";
  else base = tc ? "convT4x4s2_tc" : "convT4x4s2_simt";
  // per-resolution class (e.g. conv3x3_tc@512x32->32), interned for the lifetime of the process
  static std::mutex mu;
  static std::set<std::string> names;
  const std::string key = std::string(base) + "@" + std::to_string(d.Ho) + "x" + std::to_string(d.Ci) + "->" +
                          std::to_string(d.Co);
  std::lock_guard<std::mutex> lk(mu);
  return names.insert(key).first->c_str();
}

// 1x1 conv with a short reduction (Ci <= 32, Co = 64, 128 or 256, plain fp32 activations): the MgNet
// head Theta, C0 -> M ordinates, z = r + Theta u (PAPER.md's channel lift back to the unknowns).
// HBM-bound -- it streams the M-wide addend and output -- so it runs on the fp32 FMA pipes, not the
// tensor cores (whose conversion + epilogue dominated at K = 32).
constexpr int kSmallKMaxCi = 32;
// acc[a][c] += sum_k u[pixel a][k] W[k][channel c] for a thread's PPT pixels (rows of ub at pitch Ci)
// and 8 channels {4 tx .. 4 tx + 3} and {TCO/2 + 4 tx .. + 3}: a warp's weight loads are 512
// contiguous bytes (no bank conflicts) and the inputs are read as float4 (4 K steps; the warp's
// lanes share the pixels, so those loads broadcast).  k ascends: the FMA chain of every output is
// the plain sum order.
template <int TCO, int PPT>
__device__ __forceinline__ void smallk_mac(float (&acc)[PPT][8], const float* Ws, const float* ub, int Ci, int tx) {
  for (int k = 0; k < Ci; k += 4) {
    float4 u4[PPT];
#pragma unroll
    for (int a = 0; a < PPT; ++a) u4[a] = *reinterpret_cast<const float4*>(ub + a * Ci + k);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const float* wr = Ws + (k + kk) * TCO;
      const float4 w0 = *reinterpret_cast<const float4*>(wr + tx * 4);
      const float4 w1 = *reinterpret_cast<const float4*>(wr + TCO / 2 + tx * 4);
      const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
      for (int a = 0; a < PPT; ++a) {
        const float uva = kk == 0 ? u4[a].x : kk == 1 ? u4[a].y : kk == 2 ? u4[a].z : u4[a].w;
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[a][c] = fmaf(uva, wv[c], acc[a][c]);
      }
    }
  }
}
// (out and addend may be the same array: every element is read, then written, by one thread in
// one iteration, so __restrict__ only lets the compiler batch the loads of different pixels)
// Every global transfer is a bulk async copy: one thread loads the weights, the tile's inputs and its
// addend rows (contiguous: TPX pixels x Co channels) into shared memory on one mbarrier; the block
// computes in place over the addend tile; after a generic -> async proxy fence one thread stores
// the result with one bulk copy.  NT threads per block (4 pixels x 8 channels each): NT = 256 ->
// 32 KB tiles, 3 blocks per SM (measured at config 5: 0.135 ms against 0.138 for NT = 512 and
// 0.157 for per-thread addend loads and stores; 0.187 before the conflict-free channel mapping).
template <int TCO, int NT>
constexpr int smallk_bulk_smem_bytes() {
  return ((NT * 32 / TCO) * TCO + kSmallKMaxCi * TCO + (NT * 32 / TCO) * kSmallKMaxCi) * 4 + 128;
}
template <int TCO, int NT>
__global__ void __launch_bounds__(NT, NT == 512 ? 2 : NT == 256 ? 3 : 4) conv1x1_smallk_kernel(int npix, int Ci, int Co, const float* __restrict__ in,
                                                                  const float* __restrict__ Wk, float* out,
                                                                  const float* addend, float sign,
                                                                  const double* __restrict__ alpha, int alpha_stride,
                                                                  int alpha_on_input, int alpha_on_addend) {
  constexpr int TPX = NT * 32 / TCO;  // pixels per tile
  constexpr int TXN = TCO / 8;
  constexpr int PPT = TPX * TXN / NT;  // (= 4)
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* As = reinterpret_cast<float*>(smem_raw);  // [TPX][TCO]: addend, then the result
  float* Ws = As + TPX * TCO;                      // [ci][TCO]
  float* Us = Ws + kSmallKMaxCi * TCO;             // [pixel][ci] at pitch Ci
  uint64_t* bar = reinterpret_cast<uint64_t*>(Us + TPX * kSmallKMaxCi);
  const int tid = threadIdx.x, tx = tid % TXN, ty = tid / TXN;
  const int b = blockIdx.z;
  const int64_t p0 = (int64_t)blockIdx.x * TPX;
  const int np = (int)std::min<int64_t>(TPX, npix - p0);
  const int64_t row0 = (int64_t)b * npix + p0;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(bar);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t wbytes = (uint32_t)(Ci * TCO * 4), ubytes = (uint32_t)(np * Ci * 4);
    const uint32_t abytes = addend ? (uint32_t)(np * TCO * 4) : 0u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(wbytes + ubytes + abytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(Ws)),
                 "l"(Wk), "r"(wbytes), "r"(sb)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(Us)),
                 "l"(in + row0 * Ci), "r"(ubytes), "r"(sb)
                 : "memory");
    if (addend)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(As)),
                   "l"(addend + row0 * Co), "r"(abytes), "r"(sb)
                   : "memory");
  }
  __syncthreads();  // (barrier initialised)
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(sb)
      : "memory");
  float acc[PPT][8];
#pragma unroll
  for (int a = 0; a < PPT; ++a)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[a][c] = 0.f;
  smallk_mac<TCO, PPT>(acc, Ws, Us + ty * PPT * Ci, Ci, tx);
  const float al = alpha ? (float)alpha[(int64_t)b * alpha_stride] : 1.f;
  const float s_in = (alpha_on_input ? al : 1.f) * sign;
  const float s_add = alpha_on_addend ? al : 1.f;
#pragma unroll
  for (int a = 0; a < PPT; ++a) {
    const int pl = ty * PPT + a;
    if (pl >= np) continue;
    float* r = As + pl * TCO + tx * 4;  // channels r.., r + TCO/2..
    float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0;
    if (addend) {
      a0 = *reinterpret_cast<const float4*>(r);
      a1 = *reinterpret_cast<const float4*>(r + TCO / 2);
    }
    const float* q = acc[a];
    *reinterpret_cast<float4*>(r) = make_float4(fmaf(s_add, a0.x, s_in * q[0]), fmaf(s_add, a0.y, s_in * q[1]),
                                                fmaf(s_add, a0.z, s_in * q[2]), fmaf(s_add, a0.w, s_in * q[3]));
    *reinterpret_cast<float4*>(r + TCO / 2) = make_float4(fmaf(s_add, a1.x, s_in * q[4]), fmaf(s_add, a1.y, s_in * q[5]),
                                                    fmaf(s_add, a1.z, s_in * q[6]), fmaf(s_add, a1.w, s_in * q[7]));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> the bulk store
  __syncthreads();
  if (tid == 0) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + row0 * Co),
                 "r"((uint32_t)__cvta_generic_to_shared(As)), "r"((uint32_t)(np * TCO * 4))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem stays live until read
  }
}

bool conv1x1_smallk_ok(const ConvDesc& d) {
  // (Co = 64, 128 or 256, one channel tile: the weight block [ci][0 .. Co) is contiguous for the bulk copy)
  // With C0 = 32 the tensor-core GEMM and its TMA epilogue (addend tiles bulk-loaded, output tiles
  // bulk-stored, PDL) now beats this kernel -- config 5: 0.119 against 0.136 ms, config 4: 0.117
  // against 0.135, config 3 equal -- so the small-K kernel serves the C0 = 16 heads (configs 1-2),
  // which the tensor-core path does not take (RTE_SMALLK=1 forces it, RTE_NO_SMALLK=1 disables it)
  static const bool force = getenv("RTE_SMALLK") != nullptr;
  const bool tc_can = d.w && d.w->d_hi && d.ws_owner && d.ws_owner->tc && d.Ci % 32 == 0 && d.Co % 32 == 0;
  return d.mode == 0 && d.ks == 1 && d.Ci <= kSmallKMaxCi && d.Ci % 4 == 0 &&
         (d.Co == 64 || d.Co == 128 || d.Co == 256) && !d.in_split && !d.mod &&
         !d.out_split && getenv("RTE_NO_SMALLK") == nullptr && (force || !tc_can);
}

template <typename T>
void launch_conv_t(const ConvDesc& d, const T* in, const T* Wk, T* out, const T* addend, float sign,
                   const double* alpha, int alpha_stride, bool alpha_on_input, bool alpha_on_addend,
                   cudaStream_t st) {
  if constexpr (std::is_same<T, float>::value) {
    if (conv1x1_smallk_ok(d)) {
      prof_begin(st, conv_class_name(d, false));
      const int npix = d.Ho * d.Wo;
      auto go = [&](auto tco_tag) {
        constexpr int TCO = decltype(tco_tag)::value;
        static const int nt_env = getenv("RTE_SMALLK_NT") ? atoi(getenv("RTE_SMALLK_NT")) : 256;  // (A/B)
        auto bulk = [&](auto nt_tag) {
          constexpr int NT = decltype(nt_tag)::value;
          constexpr int smem = smallk_bulk_smem_bytes<TCO, NT>();
          constexpr int tpx = NT * 32 / TCO;
          tc::ensure_smem((const void*)conv1x1_smallk_kernel<TCO, NT>, smem);
          conv1x1_smallk_kernel<TCO, NT><<<dim3((unsigned)((npix + tpx - 1) / tpx), 1, (unsigned)d.B), NT, smem, st>>>(
              npix, d.Ci, d.Co, in, Wk, out, addend, sign, alpha, alpha_stride, alpha_on_input ? 1 : 0,
              alpha_on_addend ? 1 : 0);
        };
        if (nt_env == 128) bulk(std::integral_constant<int, 128>{});
        else if (nt_env == 512) bulk(std::integral_constant<int, 512>{});
        else bulk(std::integral_constant<int, 256>{});
      };
      if (d.Co == 256) go(std::integral_constant<int, 256>{});
      else if (d.Co == 128) go(std::integral_constant<int, 128>{});
      else go(std::integral_constant<int, 64>{});
      // (bound: HBM -- it streams the M-wide output and addend; its flops are a fraction of the ALU peak)
      after_launch(conv_class_name(d, false), st, conv_flops(d), conv_bytes(d, addend != nullptr), 0);
      return;
    }
    if (conv_tc_try(d, in, out, addend, sign, alpha, alpha_stride, alpha_on_input, alpha_on_addend, st)) return;
  }
  prof_begin(st, conv_class_name(d, false));
  auto go = [&](auto mode_tag, auto ks_tag, auto tco_tag) {
    constexpr int MODE = decltype(mode_tag)::value;
    constexpr int KS = decltype(ks_tag)::value;
    constexpr int TCO = decltype(tco_tag)::value;
    constexpr int TP = 4096 / TCO;
    int64_t npix = (MODE == 2) ? (int64_t)(d.Ho / 2) * (d.Wo / 2) : (int64_t)d.Ho * d.Wo;
    dim3 grid((unsigned)((npix + TP - 1) / TP), (unsigned)((d.Co + TCO - 1) / TCO),
              (unsigned)(d.B * (MODE == 2 ? 4 : 1)));
    auto launch = [&](auto ins, auto outs) {
      constexpr bool IS = decltype(ins)::value, OS = decltype(outs)::value;
      conv_simt_kernel<T, MODE, KS, TCO, IS, OS><<<grid, 256, 0, st>>>(
          d.Hi, d.Wi, d.Ci, d.Ho, d.Wo, d.Co, in, Wk, out, addend, sign, alpha, alpha_stride,
          alpha_on_input ? 1 : 0, alpha_on_addend ? 1 : 0, static_cast<const T*>(d.mod));
    };
    using TT = std::true_type;
    using FF = std::false_type;
    if constexpr (std::is_same<T, float>::value) {
      if (d.in_split && d.out_split) launch(TT{}, TT{});
      else if (d.in_split) launch(TT{}, FF{});
      else if (d.out_split) launch(FF{}, TT{});
      else launch(FF{}, FF{});
    } else {
      launch(FF{}, FF{});
    }
  };
  auto by_tco = [&](auto mode_tag, auto ks_tag) {
    if (d.Co <= 16) go(mode_tag, ks_tag, std::integral_constant<int, 16>{});
    else if (d.Co <= 32) go(mode_tag, ks_tag, std::integral_constant<int, 32>{});
    else go(mode_tag, ks_tag, std::integral_constant<int, 64>{});
  };
  using I0 = std::integral_constant<int, 0>;
  using I1 = std::integral_constant<int, 1>;
  using I2 = std::integral_constant<int, 2>;
  using K1 = std::integral_constant<int, 1>;
  using K3 = std::integral_constant<int, 3>;
  using K4 = std::integral_constant<int, 4>;
  if (d.mode == 0 && d.ks == 1) by_tco(I0{}, K1{});
  else if (d.mode == 0) by_tco(I0{}, K3{});
  else if (d.mode == 1) by_tco(I1{}, K3{});
  else by_tco(I2{}, K4{});
  after_launch(conv_class_name(d, false), st, conv_flops(d), conv_bytes(d, addend != nullptr) * (sizeof(T) / 4),
               sizeof(T) == 8 ? 3 : 2);
}

void launch_conv(const ConvDesc& d, const float* in, const float* Wk, float* out, const float* addend, float sign,
                 const double* alpha, int alpha_stride, bool alpha_on_input, bool alpha_on_addend, cudaStream_t st) {
  launch_conv_t<float>(d, in, Wk, out, addend, sign, alpha, alpha_stride, alpha_on_input, alpha_on_addend, st);
}

}  // namespace rte

using namespace rte;

// ---- weights --------------------------------------------------------------------------
// Reorganise a PyTorch-layout weight into the implicit-GEMM operand layouts:
//   kn : [tap][ci][co]  (SIMT B operand, co contiguous)
//   nk : [co][tap][ci]  (tensor-core B operand, N x K with K contiguous; kept on host until
//                        conv_tc_prepare uploads its tf32 hi/lo split)
// kind 0: OIHW [Co][Ci][k][k] (k = 1 or 3);  kind 1: IOHW [Ci][Co][4][4] (conv_transpose).
namespace rte {

void ConvW::build(const float* w, int kind_, int Co_, int Ci_, int ks_) {
  kind = kind_;
  Co = Co_;
  Ci = Ci_;
  ks = ks_;
  taps = ks * ks;
  std::vector<float> kn((size_t)taps * Ci * Co), nk((size_t)taps * Ci * Co);
  for (int co = 0; co < Co; ++co)
    for (int ci = 0; ci < Ci; ++ci)
      for (int ky = 0; ky < ks; ++ky)
        for (int kx = 0; kx < ks; ++kx) {
          float v = (kind == 1) ? w[(((size_t)ci * Co + co) * ks + ky) * ks + kx]
                                : w[(((size_t)co * Ci + ci) * ks + ky) * ks + kx];
          int tap = ky * ks + kx;
          kn[((size_t)tap * Ci + ci) * Co + co] = v;
          nk[((size_t)co * taps + tap) * Ci + ci] = v;
        }
  d_kn = dalloc<float>(kn.size());
  upload(d_kn, kn.data(), kn.size());
  host_nk = std::move(nk);
}

void ConvW::release() {
  dfree(d_kn);
  dfree(d_kn64);
  d_kn64 = nullptr;
  dfree(d_hi);
  dfree(d_lo);
  d_kn = d_hi = d_lo = nullptr;
}

}  // namespace rte

extern "C" {

void mgnet_destroy(mgnet_net* net) {
  if (!net) return;
  drop_net_graphs(net);
  for (auto& c : net->convs) c.release();
  dfree(net->tc_ws);
  for (auto& lv : net->lv) {
    dfree(lv.f);
    dfree(lv.u);
    dfree(lv.t);
    dfree(lv.f64);
    dfree(lv.u64);
    dfree(lv.t64);
    dfree(lv.a32);
    dfree(lv.ab32);
    dfree(lv.a64);
    dfree(lv.ab64);
  }
  delete net;
}

rte_status mgnet_create(const rte_problem* p, int levels, int c0, int nu, const float* weights, size_t n_floats,
                        mgnet_net** out) {
  mgnet_net* net = nullptr;
  try {
    RTE_REQUIRE(p && weights && out, "mgnet_create: NULL argument");
    *out = nullptr;
    RTE_REQUIRE(levels >= 1 && levels <= 12, "mgnet_create: levels must be in [1,12]");
    RTE_REQUIRE(c0 >= 1 && nu >= 0, "mgnet_create: c0 >= 1 and nu >= 0 required");
    RTE_REQUIRE(p->N % (1 << (levels - 1)) == 0, "mgnet_create: N must be divisible by 2^(levels-1)");
    const int M = p->M;
    size_t need = (size_t)c0 * M * 2;
    for (int l = 0; l < levels; ++l) {
      size_t C = (size_t)c0 << l;
      need += (size_t)(1 + 2 * nu) * C * C * 9;
      if (l < levels - 1) need += 2 * C * C * 9 + 2 * C * C * 16;
    }
    RTE_REQUIRE(n_floats == need, "mgnet_create: weight count mismatch (expected " + std::to_string(need) +
                                      ", got " + std::to_string(n_floats) + ")");
    net = new mgnet_net();
    net->prob = p;
    net->B = p->B;
    net->N = p->N;
    net->M = M;
    net->L = levels;
    net->C0 = c0;
    net->nu = nu;
    const float* w = weights;
    auto take = [&](int kind, int Co, int Ci, int ks) {
      ConvW cw;
      cw.build(w, kind, Co, Ci, ks);
      w += (size_t)Co * Ci * ks * ks;
      net->convs.push_back(std::move(cw));
      return (int)net->convs.size() - 1;
    };
    net->lift = take(0, c0, M, 1);
    net->lv.resize(levels);
    for (int l = 0; l < levels; ++l) {
      int C = c0 << l;
      Level& L = net->lv[l];
      L.C = C;
      L.H = p->N >> l;
      L.A = take(0, C, C, 3);
      for (int i = 0; i < nu; ++i) L.Bpre.push_back(take(0, C, C, 3));
      for (int i = 0; i < nu; ++i) L.Bpost.push_back(take(0, C, C, 3));
      if (l < levels - 1) {
        L.R = take(0, 2 * C, C, 3);
        L.P = take(1, C, 2 * C, 4);  // IOHW: Ci = 2C (coarse), Co = C (fine)
      }
      // levels whose convs run on the tensor cores may keep their activations pre-split (hi/lo planes)
      // (opt-in: measured slower on the B200 -- the doubled plane traffic outweighs the saved splits)
      L.split = getenv("RTE_DISABLE_TC") == nullptr && getenv("RTE_TC_PRESPLIT") != nullptr && C % 32 == 0;
      size_t act = (size_t)p->B * L.H * L.H * C * (L.split ? 2 : 1);
      L.f = dalloc<float>(act);
      L.u = dalloc<float>(act);
      L.t = dalloc<float>(act);
    }
    net->head = take(0, M, c0, 1);
    conv_tc_prepare(net);
    *out = net;
    return RTE_OK;
  } catch (const Fail& f) {
    mgnet_destroy(net);
    return f.st;
  } catch (const std::exception& e) {
    mgnet_destroy(net);
    set_error(std::string("internal: ") + e.what());
    return RTE_EINTERNAL;
  }
}

rte_status mgnet_vcycle(const mgnet_net* net, const float* r_dev, float* z_dev, int add_identity, void* stream) {
  try {
    RTE_REQUIRE(net && r_dev && z_dev, "mgnet_vcycle: NULL argument");
    RTE_REQUIRE((const void*)r_dev != (const void*)z_dev, "mgnet_vcycle: r and z must not alias");
    vcycle_run(net, r_dev, z_dev, add_identity != 0, nullptr, 0, as_stream(stream));
    return RTE_OK;
  } catch (const Fail& f) {
    return f.st;
  }
}

// ---- CoeffNet (NEXT-1, R31-R33) ---------------------------------------
namespace rte {
namespace {
// Setup-time direct convolution in fp64 (once per medium): one thread per output element.
// NHWC in [B][Hi][Wi][Ci], OIHW K [Co][Ci][ks][ks], zero padding ks/2, out = act(K * in + bias),
// act = ReLU if relu; out32 (optional) receives the float copy.
__global__ void coeffnet_conv_kernel(const double* __restrict__ in, int B, int Hi, int Wi, int Ci,
                                     const double* __restrict__ K, const double* __restrict__ bias, int Co, int ks,
                                     int stride, int relu, int Ho, int Wo, double* __restrict__ out,
                                     float* __restrict__ out32) {
  const int64_t n = (int64_t)B * Ho * Wo * Co;
  const int pad = ks / 2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int co = (int)(e % Co);
    const int64_t pix = e / Co;
    const int x = (int)(pix % Wo), y = (int)((pix / Wo) % Ho), b = (int)(pix / ((int64_t)Wo * Ho));
    double acc = bias[co];
    for (int ky = 0; ky < ks; ++ky) {
      const int yi = stride * y + ky - pad;
      if (yi < 0 || yi >= Hi) continue;
      for (int kx = 0; kx < ks; ++kx) {
        const int xi = stride * x + kx - pad;
        if (xi < 0 || xi >= Wi) continue;
        const double* ip = in + (((int64_t)b * Hi + yi) * Wi + xi) * Ci;
        const double* kp = K + ((int64_t)co * Ci * ks + ky) * ks + kx;
        for (int ci = 0; ci < Ci; ++ci) acc += kp[(int64_t)ci * ks * ks] * ip[ci];
      }
    }
    if (relu && acc < 0.0) acc = 0.0;
    out[e] = acc;
    if (out32) out32[e] = (float)acc;
  }
}

void free_modulation(mgnet_net* net) {
  for (auto& lv : net->lv) {
    dfree(lv.a32);
    dfree(lv.ab32);
    dfree(lv.a64);
    dfree(lv.ab64);
    lv.a32 = lv.ab32 = nullptr;
    lv.a64 = lv.ab64 = nullptr;
  }
}
}  // namespace
}  // namespace rte

size_t mgnet_coeffnet_weight_count(int levels, int c0) {
  size_t n = 0;
  for (int l = 0; l < levels; ++l) {
    const size_t C = (size_t)c0 << l, Cin = l == 0 ? 3 : ((size_t)c0 << (l - 1));
    n += C * Cin * 9 + C + 2 * (C * C + C);
  }
  return n;
}

rte_status mgnet_coeffnet(mgnet_net* net, const float* sigma_T, const float* sigma_a, const float* eps,
                          const float* weights, size_t n_floats) {
  try {
    RTE_REQUIRE(net, "mgnet_coeffnet: NULL net");
    ++net->graph_epoch;  // captured V-cycles read the maps (or their absence): recapture
    drop_net_graphs(net);
    free_modulation(net);
    if (!weights) return RTE_OK;  // back to the unmodulated smoother (a = abar = 1)
    RTE_REQUIRE(sigma_T && sigma_a && eps, "mgnet_coeffnet: NULL medium field");
    const size_t need = mgnet_coeffnet_weight_count(net->L, net->C0);
    RTE_REQUIRE(n_floats == need, "mgnet_coeffnet: weight count mismatch (expected " + std::to_string(need) +
                                      ", got " + std::to_string(n_floats) + ")");
    const int B = net->B, N = net->N, L = net->L, C0 = net->C0;
    // input x = [sigma_T, sigma_a, eps] along channels, NHWC fp64
    const size_t ncell = (size_t)B * N * N;
    std::vector<double> xh(ncell * 3), wh(weights, weights + n_floats);
    for (size_t c = 0; c < ncell; ++c) {
      xh[3 * c] = sigma_T[c];
      xh[3 * c + 1] = sigma_a[c];
      xh[3 * c + 2] = eps[c];
    }
    double* dx = dalloc<double>(xh.size());
    double* dw = dalloc<double>(wh.size());
    RTE_CHECK_CUDA(cudaMemcpy(dx, xh.data(), sizeof(double) * xh.size(), cudaMemcpyHostToDevice));
    RTE_CHECK_CUDA(cudaMemcpy(dw, wh.data(), sizeof(double) * wh.size(), cudaMemcpyHostToDevice));
    const double* h_in = dx;
    double* h_prev = nullptr;
    int Hin = N, Cin = 3;
    size_t off = 0;
    auto launch = [&](const double* in, int Hi, int Ci, size_t k_off, size_t b_off, int Co, int ks, int stride,
                      int relu, int Ho, double* out, float* out32) {
      const int64_t n = (int64_t)B * Ho * Ho * Co;
      const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 32);
      prof_begin(nullptr, "coeffnet");
      coeffnet_conv_kernel<<<blocks, 256>>>(in, B, Hi, Hi, Ci, dw + k_off, dw + b_off, Co, ks, stride, relu, Ho, Ho,
                                            out, out32);
      after_launch("coeffnet", nullptr, 2.0 * (double)n * Ci * ks * ks, 8.0 * (double)n, 3);
    };
    for (int l = 0; l < L; ++l) {
      const int C = C0 << l, Ho = l == 0 ? N : Hin / 2;
      Level& V = net->lv[l];
      RTE_REQUIRE(V.H == Ho && V.C == C, "mgnet_coeffnet: internal level-shape mismatch");
      const size_t kK = off, kb = kK + (size_t)C * Cin * 9, kGa = kb + C, kga = kGa + (size_t)C * C,
                   kGb = kga + C, kgb = kGb + (size_t)C * C;
      off = kgb + C;
      const size_t nel = (size_t)B * Ho * Ho * C;
      double* h = dalloc<double>(nel);
      launch(h_in, Hin, Cin, kK, kb, C, 3, l == 0 ? 1 : 2, 1, Ho, h, nullptr);  // trunk
      V.a64 = dalloc<double>(nel);
      V.ab64 = dalloc<double>(nel);
      V.a32 = dalloc<float>(nel);
      V.ab32 = dalloc<float>(nel);
      launch(h, Ho, C, kGa, kga, C, 1, 1, 0, Ho, V.a64, V.a32);   // a^[l]
      launch(h, Ho, C, kGb, kgb, C, 1, 1, 0, Ho, V.ab64, V.ab32); // abar^[l] = a^{-1,[l]}
      dfree(h_prev);
      h_prev = h;
      h_in = h;
      Hin = Ho;
      Cin = C;
    }
    RTE_CHECK_CUDA(cudaDeviceSynchronize());
    dfree(h_prev);
    dfree(dx);
    dfree(dw);
    return RTE_OK;
  } catch (const Fail& f) {
    return f.st;
  } catch (const std::exception& e) {
    set_error(std::string("internal: ") + e.what());
    return RTE_EINTERNAL;
  }
}

rte_status mgnet_modulation(const mgnet_net* net, int level, int which, double* host_out) {
  try {
    RTE_REQUIRE(net && host_out, "mgnet_modulation: NULL argument");
    RTE_REQUIRE(level >= 0 && level < net->L && (which == 0 || which == 1), "mgnet_modulation: bad level/which");
    const Level& V = net->lv[level];
    const double* src = which == 0 ? V.a64 : V.ab64;
    RTE_REQUIRE(src != nullptr, "mgnet_modulation: no CoeffNet maps (call mgnet_coeffnet first)");
    RTE_CHECK_CUDA(cudaMemcpy(host_out, src, sizeof(double) * (size_t)net->B * V.H * V.H * V.C, cudaMemcpyDeviceToHost));
    return RTE_OK;
  } catch (const Fail& f) {
    return f.st;
  }
}

rte_status mgnet_vcycle_f64(const mgnet_net* net, const double* r_dev, double* z_dev, int add_identity,
                            void* stream) {
  try {
    RTE_REQUIRE(net && r_dev && z_dev, "mgnet_vcycle_f64: NULL argument");
    RTE_REQUIRE((const void*)r_dev != (const void*)z_dev, "mgnet_vcycle_f64: r and z must not alias");
    vcycle_run_f64(net, r_dev, z_dev, add_identity != 0, as_stream(stream));
    return RTE_OK;
  } catch (const Fail& f) {
    return f.st;
  }
}

}  // extern "C"

namespace rte {

static ConvDesc desc_for(const mgnet_net* n, int mode, int ks, int H_in, int Ci, int H_out, int Co) {
  ConvDesc d;
  d.B = n->B;
  d.mode = mode;
  d.ks = ks;
  d.Hi = d.Wi = H_in;
  d.Ci = Ci;
  d.Ho = d.Wo = H_out;
  d.Co = Co;
  return d;
}

// One V-cycle.  alpha (device, per sample, stride alpha_stride) scales the input r (the
// Krylov vector is stored unnormalised, see krylov.cu); NULL means 1.
// Activation buffers of level l in the element type T (fp64 buffers are allocated on first use).
template <typename T>
static void level_bufs(const mgnet_net* net, int l, T*& f, T*& u, T*& t);
template <>
void level_bufs<float>(const mgnet_net* net, int l, float*& f, float*& u, float*& t) {
  const Level& V = net->lv[l];
  f = V.f;
  u = V.u;
  t = V.t;
}
template <>
void level_bufs<double>(const mgnet_net* net, int l, double*& f, double*& u, double*& t) {
  Level& V = const_cast<mgnet_net*>(net)->lv[l];
  if (!V.f64) {
    const size_t act = (size_t)net->B * V.H * V.H * V.C;
    V.f64 = dalloc<double>(act);
    V.u64 = dalloc<double>(act);
    V.t64 = dalloc<double>(act);
  }
  f = V.f64;
  u = V.u64;
  t = V.t64;
}
template <typename T>
static const T* conv_weights(const mgnet_net* net, int widx);
template <>
const float* conv_weights<float>(const mgnet_net* net, int widx) {
  return net->convs[widx].d_kn;
}
template <>
const double* conv_weights<double>(const mgnet_net* net, int widx) {
  ConvW& w = const_cast<mgnet_net*>(net)->convs[widx];
  if (!w.d_kn64) {  // [tap][ci][co] in fp64, from the host copy [co][tap][ci]
    std::vector<double> kn((size_t)w.taps * w.Ci * w.Co);
    for (int co = 0; co < w.Co; ++co)
      for (int tap = 0; tap < w.taps; ++tap)
        for (int ci = 0; ci < w.Ci; ++ci)
          kn[((size_t)tap * w.Ci + ci) * w.Co + co] = (double)w.host_nk[((size_t)co * w.taps + tap) * w.Ci + ci];
    w.d_kn64 = dalloc<double>(kn.size());
    upload(w.d_kn64, kn.data(), kn.size());
  }
  return w.d_kn64;
}

// One V-cycle in element type T (float: tensor-core convs where the shape allows, else SIMT;
// double: SIMT fp64).  alpha (device, per sample, stride alpha_stride) scales the input r.
template <typename T>
void vcycle_run_t(const mgnet_net* net, const T* r, T* z, bool add_identity, const double* alpha,
                  int alpha_stride, cudaStream_t st) {
  const int L = net->L, M = net->M, N = net->N;
  constexpr bool F32 = std::is_same<T, float>::value;
  auto sp = [&](int l) { return F32 && net->lv[l].split; };  // level l's activation format
  auto conv = [&](int widx, ConvDesc d, const T* in, T* out, const T* addend, float sign, bool a_in = false,
                  bool a_add = false) {
    d.w = &net->convs[widx];
    d.ws_owner = net;
    launch_conv_t<T>(d, in, conv_weights<T>(net, widx), out, addend, sign, alpha, alpha_stride, a_in, a_add, st);
  };
  struct Bufs {
    T *f, *u, *t;
  };
  std::vector<Bufs> bf(L);
  for (int l = 0; l < L; ++l) level_bufs<T>(net, l, bf[l].f, bf[l].u, bf[l].t);
  // f^0 = Lambda (alpha r)
  {
    const Level& L0 = net->lv[0];
    ConvDesc d = desc_for(net, 0, 1, N, M, N, L0.C);
    d.out_split = sp(0);
    conv(net->lift, d, r, bf[0].f, nullptr, 1.f, true, false);
  }
  // CoeffNet modulation maps (R33; NULL = 1): a multiplies A * u, abar multiplies B * t
  auto amap = [&](int l) -> const void* { return F32 ? (const void*)net->lv[l].a32 : (const void*)net->lv[l].a64; };
  auto bmap = [&](int l) -> const void* { return F32 ? (const void*)net->lv[l].ab32 : (const void*)net->lv[l].ab64; };
  auto smooth = [&](int l, int bidx, bool first) {
    const Level& V = net->lv[l];
    ConvDesc d = desc_for(net, 0, 3, V.H, V.C, V.H, V.C);
    d.in_split = d.out_split = sp(l);
    ConvDesc da = d, db = d;
    da.mod = amap(l);
    db.mod = bmap(l);
    const Bufs& b = bf[l];
    if (first) {  // u = 0: u <- abar (.) B * f  (A * 0 = 0 exactly)
      conv(bidx, db, b.f, b.u, nullptr, 1.f);
    } else {
      conv(V.A, da, b.u, b.t, b.f, -1.f);   // t = f - a (.) A * u
      conv(bidx, db, b.t, b.u, b.u, 1.f);   // u = u + abar (.) B * t
    }
  };
  for (int l = 0; l < L; ++l) {
    const Level& V = net->lv[l];
    std::vector<int> steps(V.Bpre.begin(), V.Bpre.end());
    if (l == L - 1) steps.insert(steps.end(), V.Bpost.begin(), V.Bpost.end());
    if (steps.empty())
      RTE_CHECK_CUDA(cudaMemsetAsync(bf[l].u, 0, sizeof(T) * (size_t)net->B * V.H * V.H * V.C * (sp(l) ? 2 : 1), st));
    for (size_t i = 0; i < steps.size(); ++i) smooth(l, steps[i], i == 0);
    if (l < L - 1) {
      const Level& W = net->lv[l + 1];
      ConvDesc d = desc_for(net, 0, 3, V.H, V.C, V.H, V.C);
      d.in_split = d.out_split = sp(l);
      d.mod = amap(l);
      ConvDesc dr = desc_for(net, 1, 3, V.H, V.C, W.H, W.C);
      dr.in_split = sp(l);
      dr.out_split = sp(l + 1);
      if (steps.empty()) {
        conv(V.R, dr, bf[l].f, bf[l + 1].f, nullptr, 1.f);
      } else {
        conv(V.A, d, bf[l].u, bf[l].t, bf[l].f, -1.f);   // t = f - a (.) A * u
        conv(V.R, dr, bf[l].t, bf[l + 1].f, nullptr, 1.f);  // f^{l+1} = R *_2 t
      }
    }
  }
  for (int l = L - 2; l >= 0; --l) {
    const Level& V = net->lv[l];
    const Level& W = net->lv[l + 1];
    ConvDesc dp = desc_for(net, 2, 4, W.H, W.C, V.H, V.C);
    dp.in_split = sp(l + 1);
    dp.out_split = sp(l);
    conv(V.P, dp, bf[l + 1].u, bf[l].u, bf[l].u, 1.f);  // u += P^T *_2 u^{l+1}
    for (size_t i = 0; i < V.Bpost.size(); ++i) smooth(l, V.Bpost[i], false);
  }
  // z = [alpha r] + Theta u^0
  const Level& L0 = net->lv[0];
  ConvDesc dh = desc_for(net, 0, 1, N, L0.C, N, M);
  dh.in_split = sp(0);
  conv(net->head, dh, bf[0].u, z, add_identity ? r : nullptr, 1.f, false, true);
}

void vcycle_run(const mgnet_net* net, const float* r, float* z, bool add_identity, const double* alpha,
                int alpha_stride, cudaStream_t st) {
  vcycle_run_t<float>(net, r, z, add_identity, alpha, alpha_stride, st);
}
void vcycle_run_f64(const mgnet_net* net, const double* r, double* z, bool add_identity, cudaStream_t st) {
  vcycle_run_t<double>(net, r, z, add_identity, nullptr, 0, st);
}

}  // namespace rte
