// C-ABI entry points for the problem (rte_setup / rte_rhs / rte_apply / rte_apply_f64) and
// the library's error/launch bookkeeping.  Host setup runs in fp64 (PAPER.md:29-33, 79-94,
// 113-117); everything on the per-iteration path runs in the CUDA kernels.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <map>
#include <numeric>
#include <string>
#include <tuple>
#include <vector>

#include "common.h"

#include <cstring>
#include "mgnet.h"

namespace rte {

static thread_local std::string g_err;
static thread_local int64_t g_launches = 0;

void set_error(const std::string& msg) { g_err = msg; }

// ---- per-launch timing (rte_timing_*) -------------------------------------------------
// Each timed launch gets an event pair recorded on its own stream; durations are resolved
// lazily in rte_timing_get (one synchronisation), then aggregated per kernel class.
namespace {
struct ProfRec {
  std::string name;
  cudaEvent_t e0, e1;
  double flops, bytes;
  int kind;
};
struct ProfClass {
  std::string name;
  int kind = 4;
  int64_t launches = 0;
  double ms = 0.0, flops = 0.0, bytes = 0.0;
};
thread_local bool g_prof_on = false;
thread_local cudaEvent_t g_prof_pending = nullptr;
thread_local std::vector<ProfRec> g_prof_recs;
thread_local std::vector<cudaEvent_t> g_prof_pool;
thread_local std::vector<ProfClass> g_prof_classes;

cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) {
    cudaEvent_t e = g_prof_pool.back();
    g_prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  RTE_CHECK_CUDA(cudaEventCreate(&e));
  return e;
}

void prof_resolve() {
  if (g_prof_recs.empty()) return;
  RTE_CHECK_CUDA(cudaEventSynchronize(g_prof_recs.back().e1));
  for (ProfRec& r : g_prof_recs) {
    float ms = 0.f;
    RTE_CHECK_CUDA(cudaEventSynchronize(r.e1));
    RTE_CHECK_CUDA(cudaEventElapsedTime(&ms, r.e0, r.e1));
    ProfClass* c = nullptr;
    for (ProfClass& k : g_prof_classes)
      if (k.name == r.name) c = &k;
    if (!c) {
      g_prof_classes.push_back(ProfClass{r.name, r.kind});
      c = &g_prof_classes.back();
    }
    c->launches += 1;
    c->ms += ms;
    c->flops += r.flops;
    c->bytes += r.bytes;
    g_prof_pool.push_back(r.e0);
    g_prof_pool.push_back(r.e1);
  }
  g_prof_recs.clear();
}
}  // namespace

static std::string g_prof_filter;  // rte_timing_filter: the one class to time ("" = every class)

thread_local bool g_capturing = false;       // a CUDA-graph capture is recording this thread's launches
thread_local bool g_capture_tainted = false;  // ... and a per-launch event would have been recorded
thread_local std::vector<std::string> g_capture_classes;  // timing classes of the captured launches

void prof_begin(cudaStream_t st, const char* cls) {
  if (!g_prof_on) return;
  if (!g_prof_filter.empty() && (!cls || g_prof_filter != cls)) return;
  if (g_capturing) {  // events cannot live in a replayed graph: the caller discards the capture
    g_capture_tainted = true;
    return;
  }
  if (!g_prof_pending) g_prof_pending = prof_event();
  RTE_CHECK_CUDA(cudaEventRecord(g_prof_pending, st));
}

void capture_begin() {
  g_capturing = true;
  g_capture_tainted = false;
  g_capture_classes.clear();
}
std::vector<std::string> capture_classes() { return g_capture_classes; }
// would per-launch timing record any of these classes right now?
bool prof_wants_any(const std::vector<std::string>& classes) {
  if (!g_prof_on) return false;
  if (g_prof_filter.empty()) return true;
  for (const auto& c : classes)
    if (c == g_prof_filter) return true;
  return false;
}
bool capture_end() {  // true if the capture is usable (no per-launch timing was requested in it)
  g_capturing = false;
  return !g_capture_tainted;
}
int64_t launches_now() { return g_launches; }
void launches_add(int64_t d) { g_launches += d; }

void after_launch(const char* what, cudaStream_t st, double flops, double bytes, int kind) {
  ++g_launches;
  if (g_capturing) g_capture_classes.emplace_back(what);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("launch of ") + what + " failed: " + cudaGetErrorString(e));
    throw Fail{RTE_ECUDA};
  }
  if (g_prof_on && g_prof_pending) {
    cudaEvent_t e1 = prof_event();
    RTE_CHECK_CUDA(cudaEventRecord(e1, st));
    g_prof_recs.push_back(ProfRec{what, g_prof_pending, e1, flops, bytes, kind});
    g_prof_pending = nullptr;
  }
}

void dfree(void* p) {
  if (p) cudaFree(p);
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

// ---- angular quadrature (R2, R3) ------------------------------
// Gauss-Legendre nodes/weights on [-1,1] by Newton iteration on P_n (three-term recurrence).
static void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& wt) {
  x.assign(n, 0.0);
  wt.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double z = cos(M_PI * (i + 0.75) / (n + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= n; ++k) {
        double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      if (n == 1) { p1 = z; p0 = 1.0; }
      dp = n * (z * p1 - p0) / (z * z - 1.0);
      double dz = p1 / dp;
      z -= dz;
      if (fabs(dz) < 1e-16) break;
    }
    // recompute derivative at the converged node
    double p0 = 1.0, p1 = z;
    for (int k = 2; k <= n; ++k) {
      double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    dp = n * (z * p1 - p0) / (z * z - 1.0);
    x[i] = -z;  // ascending
    wt[i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
}

static void product_quadrature(int np, int na, std::vector<double>& c, std::vector<double>& s,
                               std::vector<double>& zeta, std::vector<double>& w) {
  std::vector<double> x, a;
  gauss_legendre(np, x, a);
  int nq = na / 4;
  c.clear(); s.clear(); zeta.clear(); w.clear();
  for (int quad = 0; quad < 4; ++quad)
    for (int p = 0; p < np; ++p)
      for (int kk = 0; kk < nq; ++kk) {
        int k = quad * nq + kk;
        double th = (k + 0.5) * 2.0 * M_PI / na;
        double z = 0.5 * (x[p] + 1.0);
        double r = sqrt(1.0 - z * z);
        c.push_back(r * cos(th));
        s.push_back(r * sin(th));
        zeta.push_back(z);
        w.push_back(4.0 * M_PI * (0.5 * a[p]) / na);
      }
}

// Row-normalised HG scattering matrix S = K W (R4, R5).
static void hg_matrix(const std::vector<double>& c, const std::vector<double>& s, const std::vector<double>& z,
                      const std::vector<double>& w, double g, double* S) {
  int M = (int)c.size();
  auto hgf = [g](double mu) { return (1.0 - g * g) / pow(1.0 + g * g - 2.0 * g * mu, 1.5); };
  std::vector<double> kh(M);
  for (int m = 0; m < M; ++m) {
    double rs = 0.0;
    for (int n = 0; n < M; ++n) {
      double pl = c[m] * c[n] + s[m] * s[n];
      double zz = z[m] * z[n];
      kh[n] = 0.5 * (hgf(pl + zz) + hgf(pl - zz));
      rs += kh[n] * w[n];
    }
    for (int n = 0; n < M; ++n) S[(size_t)m * M + n] = kh[n] / rs * w[n];
  }
}

// Round-to-nearest TF32 (10 explicit mantissa bits), as cvt.rna.tf32.f32.
static float tf32_rna(float v) {
  uint32_t u;
  memcpy(&u, &v, 4);
  if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

}  // namespace rte

using namespace rte;

#define RTE_API_BEGIN try {
#define RTE_API_END                                   \
  }                                                   \
  catch (const Fail& f) { return f.st; }              \
  catch (const std::exception& e) {                   \
    set_error(std::string("internal: ") + e.what());  \
    return RTE_EINTERNAL;                             \
  }                                                   \
  return RTE_OK;

extern "C" {

const char* rte_last_error(void) { return g_err.c_str(); }

int64_t rte_launch_count(int reset) {
  int64_t v = g_launches;
  if (reset) g_launches = 0;
  return v;
}

rte_status rte_debug_counters(uint64_t* out, int n, int reset) {
  RTE_API_BEGIN
  RTE_REQUIRE(out && n > 0, "rte_debug_counters: bad argument");
  tc_debug_counters(reinterpret_cast<unsigned long long*>(out), n, reset != 0);
  RTE_API_END
}

rte_status rte_timing_filter(const char* prefix) {
  RTE_API_BEGIN
  g_prof_filter = prefix ? prefix : "";
  RTE_API_END
}

rte_status rte_timing_enable(int on) {
  RTE_API_BEGIN
  g_prof_on = on != 0;
  RTE_API_END
}

rte_status rte_timing_reset(void) {
  RTE_API_BEGIN
  prof_resolve();
  g_prof_classes.clear();
  RTE_API_END
}

rte_status rte_timing_get(int idx, char* name, int name_len, int* kind, int64_t* launches, double* ms,
                          double* flops, double* bytes, int* count) {
  RTE_API_BEGIN
  prof_resolve();
  if (count) *count = (int)g_prof_classes.size();
  if (idx >= 0) {
    RTE_REQUIRE(idx < (int)g_prof_classes.size(), "rte_timing_get: index out of range");
    const ProfClass& c = g_prof_classes[idx];
    if (name && name_len > 0) {
      strncpy(name, c.name.c_str(), name_len - 1);
      name[name_len - 1] = 0;
    }
    if (kind) *kind = c.kind;
    if (launches) *launches = c.launches;
    if (ms) *ms = c.ms;
    if (flops) *flops = c.flops;
    if (bytes) *bytes = c.bytes;
  }
  RTE_API_END
}

static void free_problem(rte_problem* p) {
  if (!p) return;
  void* ptrs[] = {p->sig_t, p->sig_s, p->sig_d, p->sig_d64, p->f, p->sig_t64, p->sig_s64, p->S32, p->St32, p->St64, p->S_hi,
                  p->S_lo, p->ax, p->ay, p->ax64, p->ay64, p->sgx, p->sgy, p->inflow, p->scratch64,
                  p->bj64, p->bj32, p->tf_mat, p->tf_L32, p->tf_L64, p->tf_fac32, p->tf_fac64, p->tf_chis32,
                  p->tf_chis64, p->at_sel, p->at_P32, p->at_P64, p->at_row, p->at_dirs, p->at_tmp32,
                  p->at_tmp64, p->ls_Dp32, p->ls_Dp64, p->ls_ws, p->ls_norm};
  for (void* q : ptrs) dfree(q);
  free_tc_state(p);
  free_gmres_work(p);
  delete p;
}

void rte_destroy(rte_problem* p) { free_problem(p); }

rte_status rte_setup(const rte_grid* grid, const rte_ordinates* ord, const float* sigma_T, const float* sigma_a,
                     const float* q, const float* eps, const float* g, const float* inflow, rte_problem** out) {
  rte_problem* p = nullptr;
  try {
    RTE_REQUIRE(grid && ord && sigma_T && sigma_a && q && eps && g && out, "rte_setup: NULL argument");
    *out = nullptr;
    RTE_REQUIRE(grid->batch >= 1, "rte_setup: batch must be >= 1");
    RTE_REQUIRE(grid->nx >= 1 && grid->nx == grid->ny, "rte_setup: nx must equal ny and be >= 1");
    p = new rte_problem();
    p->B = grid->batch;
    p->N = grid->nx;
    if (ord->c == nullptr) {
      RTE_REQUIRE(ord->n_polar >= 1 && ord->n_azim >= 4 && ord->n_azim % 4 == 0,
                  "rte_setup: built-in quadrature needs n_polar >= 1 and n_azim % 4 == 0");
      RTE_REQUIRE(ord->M == 0 || ord->M == ord->n_polar * ord->n_azim, "rte_setup: M != n_polar*n_azim");
      product_quadrature(ord->n_polar, ord->n_azim, p->c, p->s, p->zeta, p->w);
    } else {
      RTE_REQUIRE(ord->M >= 4 && ord->M % 4 == 0 && ord->s && ord->zeta && ord->w,
                  "rte_setup: user ordinates need M % 4 == 0 and c, s, zeta, w");
      p->c.assign(ord->c, ord->c + ord->M);
      p->s.assign(ord->s, ord->s + ord->M);
      p->zeta.assign(ord->zeta, ord->zeta + ord->M);
      p->w.assign(ord->w, ord->w + ord->M);
      double sw = 0.0;
      for (int m = 0; m < ord->M; ++m) {
        RTE_REQUIRE(p->c[m] != 0.0 && p->s[m] != 0.0, "rte_setup: ordinate with c_m == 0 or s_m == 0");
        RTE_REQUIRE(p->w[m] > 0.0, "rte_setup: non-positive weight");
        sw += p->w[m];
      }
      RTE_REQUIRE(fabs(sw - 4.0 * M_PI) <= 1e-12 * 4.0 * M_PI, "rte_setup: weights must sum to 4 pi");
    }
    p->M = (int)p->c.size();
    const int B = p->B, N = p->N, M = p->M;
    p->ncell = (int64_t)B * N * N;
    p->n = p->ncell * M;
    const double h = 1.0 / N;
    // coefficients (R7)
    std::vector<float> st(p->ncell), ss(p->ncell), ff(p->ncell), sd(p->ncell);
    std::vector<double> st64(p->ncell), ss64(p->ncell), sd64(p->ncell);
    for (int64_t k = 0; k < p->ncell; ++k) {
      double e = eps[k], sT = sigma_T[k], sA = sigma_a[k];
      RTE_REQUIRE(e > 0.0 && e <= 1.0, "rte_setup: eps must lie in (0,1]");
      RTE_REQUIRE(sT >= 0.0 && sA >= 0.0 && q[k] >= 0.0, "rte_setup: sigma_T, sigma_a, q must be >= 0");
      double t = sT / e, sc = sT / e - e * sA;
      RTE_REQUIRE(sc >= 0.0, "rte_setup: sigma_T/eps < eps*sigma_a (negative scattering) in a cell");
      st64[k] = t;
      ss64[k] = sc;
      st[k] = (float)t;
      ss[k] = (float)sc;
      sd64[k] = e * sA;  // sigma_t - sigma_s, formed without the cancellation
      sd[k] = (float)sd64[k];
      ff[k] = (float)(e * (double)q[k]);
    }
    p->h_eps.assign(eps, eps + p->ncell);
    p->h_sa.assign(sigma_a, sigma_a + p->ncell);
    // scattering matrices per sample
    p->S.assign((size_t)B * M * M, 0.0);
    for (int b = 0; b < B; ++b) {
      RTE_REQUIRE(fabs((double)g[b]) < 1.0, "rte_setup: |g| must be < 1");
      hg_matrix(p->c, p->s, p->zeta, p->w, (double)g[b], p->S.data() + (size_t)b * M * M);
    }
    std::vector<float> S32((size_t)B * M * M), St32((size_t)B * M * M), Shi((size_t)B * M * M), Slo((size_t)B * M * M);
    std::vector<double> St64((size_t)B * M * M);
    for (int b = 0; b < B; ++b)
      for (int m = 0; m < M; ++m)
        for (int n = 0; n < M; ++n) {
          size_t o = (size_t)b * M * M;
          double v = p->S[o + (size_t)m * M + n];
          float v32 = (float)v;
          S32[o + (size_t)m * M + n] = v32;
          St32[o + (size_t)n * M + m] = v32;
          St64[o + (size_t)n * M + m] = v;
          float hi = tf32_rna(v32);
          Shi[o + (size_t)m * M + n] = hi;
          Slo[o + (size_t)m * M + n] = tf32_rna(v32 - hi);
        }
    std::vector<float> ax(M), ay(M);
    std::vector<double> ax64(M), ay64(M);
    std::vector<int8_t> sgx(M), sgy(M);
    for (int m = 0; m < M; ++m) {
      ax64[m] = fabs(p->c[m]) / h;
      ay64[m] = fabs(p->s[m]) / h;
      ax[m] = (float)ax64[m];
      ay[m] = (float)ay64[m];
      sgx[m] = p->c[m] > 0 ? 1 : -1;
      sgy[m] = p->s[m] > 0 ? 1 : -1;
    }
    // upload
    p->sig_t = dalloc<float>(p->ncell); upload(p->sig_t, st.data(), p->ncell);
    p->sig_s = dalloc<float>(p->ncell); upload(p->sig_s, ss.data(), p->ncell);
    p->f = dalloc<float>(p->ncell); upload(p->f, ff.data(), p->ncell);
    p->sig_t64 = dalloc<double>(p->ncell); upload(p->sig_t64, st64.data(), p->ncell);
    p->sig_s64 = dalloc<double>(p->ncell); upload(p->sig_s64, ss64.data(), p->ncell);
    p->sig_d = dalloc<float>(p->ncell); upload(p->sig_d, sd.data(), p->ncell);
    p->sig_d64 = dalloc<double>(p->ncell); upload(p->sig_d64, sd64.data(), p->ncell);
    size_t mm = (size_t)B * M * M;
    p->S32 = dalloc<float>(mm); upload(p->S32, S32.data(), mm);
    p->St32 = dalloc<float>(mm); upload(p->St32, St32.data(), mm);
    p->St64 = dalloc<double>(mm); upload(p->St64, St64.data(), mm);
    p->S_hi = dalloc<float>(mm); upload(p->S_hi, Shi.data(), mm);
    p->S_lo = dalloc<float>(mm); upload(p->S_lo, Slo.data(), mm);
    p->ax = dalloc<float>(M); upload(p->ax, ax.data(), M);
    p->ay = dalloc<float>(M); upload(p->ay, ay.data(), M);
    p->ax64 = dalloc<double>(M); upload(p->ax64, ax64.data(), M);
    p->ay64 = dalloc<double>(M); upload(p->ay64, ay64.data(), M);
    p->sgx = dalloc<int8_t>(M); upload(p->sgx, sgx.data(), M);
    p->sgy = dalloc<int8_t>(M); upload(p->sgy, sgy.data(), M);
    if (inflow) {
      size_t ni = (size_t)B * 4 * N * M;
      p->inflow = dalloc<float>(ni);
      upload(p->inflow, inflow, ni);
    }
    p->scratch64 = dalloc<double>(64);
    p->tc_apply = apply_tc_supported(M) && getenv("RTE_DISABLE_TC") == nullptr;
    *out = p;
    return RTE_OK;
  } catch (const Fail& f) {
    free_problem(p);
    return f.st;
  } catch (const std::exception& e) {
    free_problem(p);
    set_error(std::string("internal: ") + e.what());
    return RTE_EINTERNAL;
  }
}

rte_status rte_setup_tfps(const rte_grid* grid, const rte_ordinates* ord, const float* sigma_T, const float* sigma_a,
                          const float* q, const float* eps, const float* g, const float* inflow, rte_problem** out) {
  rte_problem* p = nullptr;
  try {
    RTE_REQUIRE(out, "rte_setup_tfps: NULL argument");
    *out = nullptr;
    // the psi-space setup validates the inputs and builds quadrature, S and the coefficient fields
    const rte_status st0 = rte_setup(grid, ord, sigma_T, sigma_a, q, eps, g, inflow, &p);
    if (st0 != RTE_OK) return st0;
    const int B = p->B, N = p->N, Md = p->M;
    const double h = 1.0 / N;
    // materials: distinct (sample, sigma_t, sigma_s) of the cells (R7); the TFPS
    // basis needs sigma_t - sigma_s = eps sigma_a > 0
    std::map<std::tuple<int, double, double>, int> index;
    std::vector<int> mat(p->ncell);
    std::vector<double> chis(p->ncell);
    std::vector<std::tuple<int, double, double>> keys;
    for (int64_t k = 0; k < p->ncell; ++k) {
      const double e = eps[k], sT = sigma_T[k], sA = sigma_a[k];
      const double t = sT / e, sc = sT / e - e * sA;
      RTE_REQUIRE(e * sA > 0.0, "rte_setup_tfps: TFPS needs eps sigma_a > 0 in every cell (PAPER.md:117)");
      const int b = (int)(k / ((int64_t)N * N));
      auto key = std::make_tuple(b, t, sc);
      auto it = index.find(key);
      if (it == index.end()) {
        RTE_REQUIRE(index.size() < 4096, "rte_setup_tfps: more than 4096 distinct materials (piecewise-constant "
                                         "media with few materials only)");
        it = index.emplace(key, (int)keys.size()).first;
        keys.push_back(key);
      }
      mat[k] = it->second;
      chis[k] = (e * (double)q[k]) / (e * sA);  // f / (sigma_t - sigma_s)
    }
    const int nmat = (int)keys.size();
    const int K = 2 * Md;
    std::vector<double> LT((size_t)nmat * K * Md), fac((size_t)nmat * 5 * K);
    p->tf_xi.assign((size_t)nmat * K, 0.0);
    p->tf_Lh.assign((size_t)nmat * Md * K, 0.0);
    for (int mi = 0; mi < nmat; ++mi) {
      const int b = std::get<0>(keys[mi]);
      const double t = std::get<1>(keys[mi]), sc = std::get<2>(keys[mi]);
      std::vector<double> xi, L;
      tfps_local_modes(p->S.data() + (size_t)b * Md * Md, p->c, p->s, sc / t, xi, L);
      for (int k = 0; k < K; ++k) {
        p->tf_xi[(size_t)mi * K + k] = xi[k];
        for (int m = 0; m < Md; ++m) {
          LT[((size_t)mi * K + k) * Md + m] = L[(size_t)m * K + k];
          p->tf_Lh[((size_t)mi * Md + m) * K + k] = L[(size_t)m * K + k];
        }
      }
      tfps_face_factors(xi, Md, t, h, fac.data() + (size_t)mi * 5 * K);
    }
    std::vector<float> LT32(LT.begin(), LT.end()), fac32(fac.begin(), fac.end()), chis32(chis.begin(), chis.end());
    p->kind = 1;
    p->Md = Md;
    p->M = K;
    p->n = p->ncell * K;
    p->nmat = nmat;
    p->tc_apply = false;
    p->tf_mat = dalloc<int>(p->ncell); upload(p->tf_mat, mat.data(), p->ncell);
    p->tf_L64 = dalloc<double>(LT.size()); upload(p->tf_L64, LT.data(), LT.size());
    p->tf_L32 = dalloc<float>(LT.size()); upload(p->tf_L32, LT32.data(), LT.size());
    p->tf_fac64 = dalloc<double>(fac.size()); upload(p->tf_fac64, fac.data(), fac.size());
    p->tf_fac32 = dalloc<float>(fac.size()); upload(p->tf_fac32, fac32.data(), fac.size());
    p->tf_chis64 = dalloc<double>(p->ncell); upload(p->tf_chis64, chis.data(), p->ncell);
    p->tf_chis32 = dalloc<float>(p->ncell); upload(p->tf_chis32, chis32.data(), p->ncell);
    *out = p;
    return RTE_OK;
  } catch (const Fail& f) {
    free_problem(p);
    return f.st;
  } catch (const std::exception& e) {
    free_problem(p);
    set_error(std::string("internal: ") + e.what());
    return RTE_EINTERNAL;
  }
}

rte_status rte_setup_atfps(const rte_grid* grid, const rte_ordinates* ord, const float* sigma_T,
                           const float* sigma_a, const float* q, const float* eps, const float* g, const float* inflow,
                           double delta, rte_problem** out) {
  rte_problem* p = nullptr;
  try {
    RTE_REQUIRE(out, "rte_setup_atfps: NULL argument");
    *out = nullptr;
    RTE_REQUIRE(delta > 0.0 && delta < 1.0, "rte_setup_atfps: delta must lie in (0, 1)");
    const rte_status st0 = rte_setup_tfps(grid, ord, sigma_T, sigma_a, q, eps, g, inflow, &p);
    if (st0 != RTE_OK) return st0;
    const int Md = p->Md, K = 2 * Md, H = Md / 2, nmat = p->nmat;
    RTE_REQUIRE(Md % 2 == 0, "rte_setup_atfps: the number of directions must be even");
    const double h = 1.0 / p->N;
    // selection (eq:def_V_delta): exp(-1/2 |xi| sigma_t h) > delta
    std::vector<uint8_t> sel((size_t)nmat * K);
    std::vector<double> st_of(nmat, 0.0);
    {
      std::vector<int> mat(p->ncell);
      RTE_CHECK_CUDA(cudaMemcpy(mat.data(), p->tf_mat, sizeof(int) * p->ncell, cudaMemcpyDeviceToHost));
      for (int64_t k = 0; k < p->ncell; ++k) st_of[mat[k]] = (double)sigma_T[k] / (double)eps[k];
      std::vector<int64_t> count(nmat, 0);
      for (int64_t k = 0; k < p->ncell; ++k) ++count[mat[k]];
      p->at_dim = 0;
      for (int m = 0; m < nmat; ++m)
        for (int k = 0; k < K; ++k) {
          sel[(size_t)m * K + k] = exp(-0.5 * fabs(p->tf_xi[(size_t)m * K + k]) * st_of[m] * h) > delta ? 1 : 0;
          p->at_dim += sel[(size_t)m * K + k] ? count[m] : 0;
        }
    }
    // interface bases and projections (R40): interior [2 orient][a][b], boundary [4 faces][a]
    const size_t nint = (size_t)2 * nmat * nmat, nbnd = (size_t)4 * nmat;
    std::vector<double> P(nint * Md * Md + nbnd * H * H, 0.0);
    std::vector<int> row((nint + nbnd) * 2 * K, -1);
    std::vector<int> alld(Md), dirs[4];
    std::iota(alld.begin(), alld.end(), 0);
    for (int m = 0; m < Md; ++m) {
      (p->c[m] > 0 ? dirs[0] : dirs[1]).push_back(m);  // incoming at x = 0 (L) / x = 1 (R)
      (p->s[m] > 0 ? dirs[2] : dirs[3]).push_back(m);  // incoming at y = 0 (B) / y = 1 (T)
    }
    for (int f = 0; f < 4; ++f) RTE_REQUIRE((int)dirs[f].size() == H, "rte_setup_atfps: unbalanced ordinate set");
    std::vector<double> Pt;
    for (int o = 0; o < 2; ++o)
      for (int a = 0; a < nmat; ++a)
        for (int b = 0; b < nmat; ++b) {
          const size_t t = ((size_t)o * nmat + a) * nmat + b;
          // C- contributes its R- (T-) centred modes, C+ its L- (B-) centred modes
          atfps_interface(p->tf_Lh, sel, Md, a, b, o == 0 ? 1 : 3, o == 0 ? 0 : 2, alld, Pt, row.data() + t * 2 * K);
          std::copy(Pt.begin(), Pt.end(), P.begin() + t * Md * Md);
        }
    for (int f = 0; f < 4; ++f)
      for (int a = 0; a < nmat; ++a) {
        const size_t t = (size_t)f * nmat + a;
        atfps_interface(p->tf_Lh, sel, Md, a, a, f, -1, dirs[f], Pt, row.data() + (nint + t) * 2 * K);
        std::copy(Pt.begin(), Pt.end(), P.begin() + nint * Md * Md + t * H * H);
      }
    std::vector<float> P32(P.begin(), P.end());
    std::vector<int> dflat;
    for (int f = 0; f < 4; ++f) dflat.insert(dflat.end(), dirs[f].begin(), dirs[f].end());
    p->kind = 2;
    p->at_delta = delta;
    p->at_sel = dalloc<uint8_t>(sel.size()); upload(p->at_sel, sel.data(), sel.size());
    p->at_P64 = dalloc<double>(P.size()); upload(p->at_P64, P.data(), P.size());
    p->at_P32 = dalloc<float>(P.size()); upload(p->at_P32, P32.data(), P.size());
    p->at_row = dalloc<int>(row.size()); upload(p->at_row, row.data(), row.size());
    p->at_dirs = dalloc<int>(dflat.size()); upload(p->at_dirs, dflat.data(), dflat.size());
    p->at_tmp32 = dalloc<float>(p->n);
    p->at_tmp64 = dalloc<double>(p->n);
    *out = p;
    return RTE_OK;
  } catch (const Fail& f) {
    free_problem(p);
    return f.st;
  } catch (const std::exception& e) {
    free_problem(p);
    set_error(std::string("internal: ") + e.what());
    return RTE_EINTERNAL;
  }
}

rte_status rte_atfps_info(const rte_problem* p, double* delta, int64_t* dim, uint8_t* sel) {
  RTE_API_BEGIN
  RTE_REQUIRE(p && p->kind == 2, "rte_atfps_info: not an ATFPS problem");
  if (delta) *delta = p->at_delta;
  if (dim) *dim = p->at_dim;
  if (sel) RTE_CHECK_CUDA(cudaMemcpy(sel, p->at_sel, (size_t)p->nmat * 2 * p->Md, cudaMemcpyDeviceToHost));
  RTE_API_END
}

rte_status rte_atfps_reconstruct(const rte_problem* p, const float* alpha_dev, float* psi_dev, float* full_dev,
                                 void* stream) {
  RTE_API_BEGIN
  RTE_REQUIRE(p && alpha_dev && psi_dev && p->kind == 2, "rte_atfps_reconstruct: NULL argument or not ATFPS");
  float* full = full_dev ? full_dev : p->at_tmp32;
  launch_atfps<float>(p, 2, alpha_dev, full, nullptr, 0, nullptr, as_stream(stream));
  launch_tfps_reconstruct<float>(p, full, psi_dev, as_stream(stream));
  RTE_API_END
}

rte_status rte_atfps_reconstruct_f64(const rte_problem* p, const double* alpha_dev, double* psi_dev, double* full_dev,
                                     void* stream) {
  RTE_API_BEGIN
  RTE_REQUIRE(p && alpha_dev && psi_dev && p->kind == 2, "rte_atfps_reconstruct_f64: NULL argument or not ATFPS");
  double* full = full_dev ? full_dev : p->at_tmp64;
  launch_atfps<double>(p, 2, alpha_dev, full, nullptr, 0, nullptr, as_stream(stream));
  launch_tfps_reconstruct<double>(p, full, psi_dev, as_stream(stream));
  RTE_API_END
}

rte_status rte_set_source(rte_problem* p, const float* q, const float* inflow) {
  RTE_API_BEGIN
  RTE_REQUIRE(p && q, "rte_set_source: NULL argument");
  const int64_t nc = p->ncell;
  std::vector<float> ff(nc);
  std::vector<double> chis(nc);
  for (int64_t k = 0; k < nc; ++k) {
    RTE_REQUIRE(q[k] >= 0.0f, "rte_set_source: q must be >= 0");
    const double e = p->h_eps[k];
    ff[k] = (float)(e * (double)q[k]);
    chis[k] = (e * (double)q[k]) / (e * (double)p->h_sa[k]);  // f / (sigma_t - sigma_s), as rte_setup_tfps
  }
  upload(p->f, ff.data(), nc);
  if (p->kind != 0) {
    std::vector<float> c32(chis.begin(), chis.end());
    upload(p->tf_chis64, chis.data(), nc);
    upload(p->tf_chis32, c32.data(), nc);
  }
  if (inflow) {
    const int Md = p->kind == 0 ? p->M : p->Md;
    const size_t ni = (size_t)p->B * 4 * p->N * Md;
    if (!p->inflow) p->inflow = dalloc<float>(ni);
    upload(p->inflow, inflow, ni);
  }
  RTE_API_END
}

rte_status rte_atfps_fit(const rte_problem* p, const float* psi_dev, float* alpha_dev, void* stream) {
  RTE_API_BEGIN
  RTE_REQUIRE(p && psi_dev && alpha_dev, "rte_atfps_fit: NULL argument");
  RTE_REQUIRE(p->kind == 2, "rte_atfps_fit: not an ATFPS problem (rte_setup_atfps)");
  atfps_fit<float>(p, psi_dev, alpha_dev, as_stream(stream));
  RTE_API_END
}

rte_status rte_atfps_fit_f64(const rte_problem* p, const double* psi_dev, double* alpha_dev, void* stream) {
  RTE_API_BEGIN
  RTE_REQUIRE(p && psi_dev && alpha_dev, "rte_atfps_fit_f64: NULL argument");
  RTE_REQUIRE(p->kind == 2, "rte_atfps_fit_f64: not an ATFPS problem (rte_setup_atfps)");
  atfps_fit<double>(p, psi_dev, alpha_dev, as_stream(stream));
  RTE_API_END
}

rte_status rte_atfps_loss(const rte_problem* p, const float* psi_dev, double* loss, float* grad_dev, void* stream) {
  RTE_API_BEGIN
  RTE_REQUIRE(p && psi_dev && loss, "rte_atfps_loss: NULL argument");
  RTE_REQUIRE(p->kind == 2, "rte_atfps_loss: not an ATFPS problem (rte_setup_atfps)");
  RTE_REQUIRE((const void*)psi_dev != (const void*)grad_dev, "rte_atfps_loss: psi and grad must not alias");
  atfps_loss<float>(p, psi_dev, loss, grad_dev, as_stream(stream));
  RTE_API_END
}

rte_status rte_atfps_loss_f64(const rte_problem* p, const double* psi_dev, double* loss, double* grad_dev,
                              void* stream) {
  RTE_API_BEGIN
  RTE_REQUIRE(p && psi_dev && loss, "rte_atfps_loss_f64: NULL argument");
  RTE_REQUIRE(p->kind == 2, "rte_atfps_loss_f64: not an ATFPS problem (rte_setup_atfps)");
  RTE_REQUIRE((const void*)psi_dev != (const void*)grad_dev, "rte_atfps_loss_f64: psi and grad must not alias");
  atfps_loss<double>(p, psi_dev, loss, grad_dev, as_stream(stream));
  RTE_API_END
}

rte_status rte_tfps_modes(int M, const double* c, const double* s, const double* S, double gamma, double* xi,
                          double* L) {
  RTE_API_BEGIN
  RTE_REQUIRE(M >= 2 && c && s && S && xi && L, "rte_tfps_modes: bad argument");
  std::vector<double> vc(c, c + M), vs(s, s + M), x, l;
  tfps_local_modes(S, vc, vs, gamma, x, l);
  memcpy(xi, x.data(), x.size() * sizeof(double));
  memcpy(L, l.data(), l.size() * sizeof(double));
  RTE_API_END
}

rte_status rte_tfps_info(const rte_problem* p, int* nmat, int* Md, double* xi, double* L) {
  if (!p || (p->kind != 1 && p->kind != 2)) { set_error("rte_tfps_info: not a TFPS problem"); return RTE_EINVAL; }
  if (nmat) *nmat = p->nmat;
  if (Md) *Md = p->Md;
  if (xi) memcpy(xi, p->tf_xi.data(), p->tf_xi.size() * sizeof(double));
  if (L) memcpy(L, p->tf_Lh.data(), p->tf_Lh.size() * sizeof(double));
  return RTE_OK;
}

rte_status rte_tfps_reconstruct(const rte_problem* p, const float* alpha_dev, float* psi_dev, void* stream) {
  RTE_API_BEGIN
  RTE_REQUIRE(p && alpha_dev && psi_dev && p->kind >= 1, "rte_tfps_reconstruct: NULL argument or not a TFPS problem");
  launch_tfps_reconstruct<float>(p, alpha_dev, psi_dev, as_stream(stream));
  RTE_API_END
}

rte_status rte_tfps_reconstruct_f64(const rte_problem* p, const double* alpha_dev, double* psi_dev, void* stream) {
  RTE_API_BEGIN
  RTE_REQUIRE(p && alpha_dev && psi_dev && p->kind >= 1, "rte_tfps_reconstruct_f64: NULL argument or not a TFPS problem");
  launch_tfps_reconstruct<double>(p, alpha_dev, psi_dev, as_stream(stream));
  RTE_API_END
}

rte_status rte_problem_info(const rte_problem* p, int* batch, int* N, int* M, int64_t* n) {
  if (!p) { set_error("rte_problem_info: NULL problem"); return RTE_EINVAL; }
  if (batch) *batch = p->B;
  if (N) *N = p->N;
  if (M) *M = p->M;
  if (n) *n = p->n;
  return RTE_OK;
}

rte_status rte_get_ordinates(const rte_problem* p, double* c, double* s, double* zeta, double* w) {
  if (!p) { set_error("rte_get_ordinates: NULL problem"); return RTE_EINVAL; }
  const size_t nd = p->c.size();  // directions (p->M counts unknowns per cell: 2 x directions for TFPS)
  if (c) memcpy(c, p->c.data(), nd * sizeof(double));
  if (s) memcpy(s, p->s.data(), nd * sizeof(double));
  if (zeta) memcpy(zeta, p->zeta.data(), nd * sizeof(double));
  if (w) memcpy(w, p->w.data(), nd * sizeof(double));
  return RTE_OK;
}

rte_status rte_quadrature(int n_polar, int n_azim, double* c, double* s, double* zeta, double* w) {
  RTE_API_BEGIN
  RTE_REQUIRE(n_polar >= 1 && n_azim >= 4 && n_azim % 4 == 0, "rte_quadrature: need n_polar >= 1, n_azim % 4 == 0");
  std::vector<double> vc, vs, vz, vw;
  product_quadrature(n_polar, n_azim, vc, vs, vz, vw);
  size_t M = vc.size();
  if (c) memcpy(c, vc.data(), M * sizeof(double));
  if (s) memcpy(s, vs.data(), M * sizeof(double));
  if (zeta) memcpy(zeta, vz.data(), M * sizeof(double));
  if (w) memcpy(w, vw.data(), M * sizeof(double));
  RTE_API_END
}

rte_status rte_hg_matrix(int M, const double* c, const double* s, const double* zeta, const double* w, double g,
                         double* S) {
  RTE_API_BEGIN
  RTE_REQUIRE(M >= 1 && c && s && zeta && w && S, "rte_hg_matrix: bad argument");
  RTE_REQUIRE(fabs(g) < 1.0, "rte_hg_matrix: |g| must be < 1");
  std::vector<double> vc(c, c + M), vs(s, s + M), vz(zeta, zeta + M), vw(w, w + M);
  hg_matrix(vc, vs, vz, vw, g, S);
  RTE_API_END
}

rte_status rte_rhs(const rte_problem* p, float* b_dev, void* stream) {
  RTE_API_BEGIN
  RTE_REQUIRE(p && b_dev, "rte_rhs: NULL argument");
  launch_rhs(p, b_dev, as_stream(stream));
  RTE_API_END
}

rte_status rte_apply(const rte_problem* p, const float* x_dev, float* y_dev, void* stream) {
  RTE_API_BEGIN
  RTE_REQUIRE(p && x_dev && y_dev, "rte_apply: NULL argument");
  RTE_REQUIRE((const void*)x_dev != (const void*)y_dev, "rte_apply: x and y must not alias");
  launch_apply_f32(p, x_dev, y_dev, nullptr, 0, as_stream(stream));
  RTE_API_END
}

rte_status rte_apply_f64(const rte_problem* p, const double* x_dev, double* y_dev, void* stream) {
  RTE_API_BEGIN
  RTE_REQUIRE(p && x_dev && y_dev, "rte_apply_f64: NULL argument");
  RTE_REQUIRE((const void*)x_dev != (const void*)y_dev, "rte_apply_f64: x and y must not alias");
  launch_apply_f64(p, x_dev, y_dev, nullptr, as_stream(stream));
  RTE_API_END
}

}  // extern "C"
