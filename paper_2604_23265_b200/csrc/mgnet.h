// Internal MgNet structures (NOT part of the ABI).
#pragma once

#include <vector>

#include "common.h"

namespace rte {

struct ConvW {
  int kind = 0;       // 0: OIHW conv, 1: IOHW conv_transpose
  int Co = 0, Ci = 0, ks = 0, taps = 0;
  float* d_kn = nullptr;   // [tap][ci][co]
  double* d_kn64 = nullptr;  // same, fp64 (fp64 V-cycle; created on first use)
  float* d_hi = nullptr;   // tensor-core operand [tc_rows][tc_K] K-major, tf32 hi (conv_tc.cu)
  float* d_lo = nullptr;   //                       tf32 lo
  int tc_rows = 0, tc_K = 0;
  std::vector<float> host_nk;  // [co][tap][ci]
  void build(const float* w, int kind, int Co, int Ci, int ks);
  void release();
};

struct ConvDesc {
  int B = 1, mode = 0, ks = 3;       // mode 0: stride-1 (ks 1 or 3), 1: stride-2 3x3, 2: transposed 4x4 s2
  // Activation formats (float V-cycle): split = two planes per batch sample, hi = rna_tf32(v) and
  // lo = v - hi ([B][2][H][W][C]); plain = [B][H][W][C].  The addend has the output's format.
  bool in_split = false, out_split = false;
  int Hi = 0, Wi = 0, Ci = 0, Ho = 0, Wo = 0, Co = 0;
  const ConvW* w = nullptr;
  const struct ::mgnet_net* ws_owner = nullptr;  // net owning the split-K workspace (tensor-core path)
  // CoeffNet modulation (R33): the conv result is multiplied elementwise by this map before the
  // addend is added, out = s_add addend + s_in (mod (.) (W * in)); plain [B][Ho][Wo][Co] of the
  // launch's element type (float or double), NULL = 1
  const void* mod = nullptr;
};

struct Level {
  int C = 0, H = 0;
  int A = -1, R = -1, P = -1;
  std::vector<int> Bpre, Bpost;
  float* f = nullptr;   // [B][H][H][C]
  float* u = nullptr;
  float* t = nullptr;
  bool split = false;  // f, u, t stored as hi/lo planes (levels whose convs run on the tensor cores)
  double *f64 = nullptr, *u64 = nullptr, *t64 = nullptr;  // fp64 V-cycle buffers (first use)
  // CoeffNet modulation maps a^[l], abar^[l] (mgnet_coeffnet; NULL = unmodulated): [B][H][H][C]
  float *a32 = nullptr, *ab32 = nullptr;
  double *a64 = nullptr, *ab64 = nullptr;
};

double conv_flops(const ConvDesc& d);
double conv_bytes(const ConvDesc& d, bool has_addend);
const char* conv_class_name(const ConvDesc& d, bool tc);
void launch_conv(const ConvDesc& d, const float* in, const float* Wk, float* out, const float* addend, float sign,
                 const double* alpha, int alpha_stride, bool alpha_on_input, bool alpha_on_addend, cudaStream_t st);
// tensor-core path (conv_tc.cu): returns false when the shape is not supported there.
bool conv_tc_try(const ConvDesc& d, const float* in, float* out, const float* addend, float sign,
                 const double* alpha, int alpha_stride, bool alpha_on_input, bool alpha_on_addend, cudaStream_t st);
void conv_tc_prepare(struct ::mgnet_net* net);
void tc_debug_counters(unsigned long long* out, int n, bool reset);
void apply_tc_debug_counters(unsigned long long* out, int n, bool reset);  // (apply_tc.cu)

void vcycle_run(const struct ::mgnet_net* net, const float* r, float* z, bool add_identity, const double* alpha,
                int alpha_stride, cudaStream_t st);
void vcycle_run_f64(const struct ::mgnet_net* net, const double* r, double* z, bool add_identity, cudaStream_t st);
template <typename T>
void launch_conv_t(const ConvDesc& d, const T* in, const T* Wk, T* out, const T* addend, float sign,
                   const double* alpha, int alpha_stride, bool alpha_on_input, bool alpha_on_addend, cudaStream_t st);

}  // namespace rte

struct mgnet_net {
  const rte_problem* prob = nullptr;
  int B = 1, N = 0, M = 0, L = 0, C0 = 0, nu = 0;
  std::vector<rte::ConvW> convs;
  std::vector<rte::Level> lv;
  int lift = -1, head = -1;
  bool tc = false;                 // tensor-core convs enabled (conv_tc_prepare)
  float* tc_ws = nullptr;          // split-K partials
  size_t tc_ws_elems = 0;
  uint64_t graph_epoch = 0;        // bumped when captured CUDA graphs of this net go stale
};
