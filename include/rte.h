/* rte.h -- C ABI of the B200-native hot path of arXiv 2604.23265
 * ("A filtered MgNet solver for radiative transfer equations").
 *
 * The hot path is the inner loop of an MgNet-preconditioned restarted GMRES
 * solve of the discretised steady RTE in x-y geometry:
 *   one discrete-ordinates operator apply  (rte_apply: upwind stencil + dense
 *   M x M Henyey-Greenstein scattering contraction, PAPER.md:90-104 eq:DORTE_2d),
 *   one MgNet V-cycle (mgnet_vcycle), and the Arnoldi/Givens
 *   bookkeeping (gmres_solve).
 * Readings of the paper (R1..R30) are listed in DESIGN.md §3; the operator is
 * the psi-space discrete-ordinates operator (R1).
 *
 * Conventions
 *  - Every call returns rte_status; RTE_OK == 0.  On failure a thread-local
 *    message is available from rte_last_error().  No call aborts the process.
 *  - "host" pointers are ordinary CPU memory, read during the call only (the
 *    library copies what it keeps; the caller may free them on return).
 *  - "_dev" pointers are caller-owned CUDA device memory (e.g. PyTorch
 *    tensors), contiguous, 16-byte aligned, in the layout stated.  Input and
 *    output buffers of one call must not alias.
 *  - stream: a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Calls only enqueue work on it, except gmres_solve, which synchronises it
 *    once per inner iteration to read an 8-byte convergence flag.
 *  - Unknown layout: psi[b][j][i][m] (batch, y-index j, x-index i, ordinate m
 *    fastest), float32 unless stated; n = batch*N*N*M elements.  Cell (j,i)
 *    covers [i h,(i+1) h] x [j h,(j+1) h], h = 1/N.  Ordinates are ordered
 *    quadrant-major (+,+),(-,+),(-,-),(+,-), then polar, then azimuth
 *    (R3); rte_get_ordinates returns them.
 *  - A handle is not thread-safe: serialise calls on one handle (it owns
 *    scratch).  Distinct handles may run concurrently on distinct streams.
 */
#ifndef RTE_H
#define RTE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RTE_OK = 0,
  RTE_EINVAL = 1,    /* invalid argument (message says which) */
  RTE_ENOMEM = 2,    /* device or host allocation failed */
  RTE_ECUDA = 3,     /* CUDA error (message holds cudaGetErrorString) */
  RTE_EINTERNAL = 4,
  RTE_ENUMERIC = 5   /* gmres_solve: a non-finite (NaN/Inf) Arnoldi column stopped a sample; the
                        reports are filled and that sample's breakdown is 2 */
} rte_status;

/* Uniform grid on the unit square; nx == ny == N required; h = 1/N. */
typedef struct { int batch, nx, ny; } rte_grid;

/* Angular quadrature.  If c == NULL the built-in product set is
 * used: n_polar Gauss-Legendre zeta nodes on (0,1) x n_azim offset-uniform
 * azimuths, M = n_polar*n_azim, weights summing to 4 pi (R2, R3).
 * Otherwise c, s, zeta, w (host, length M) are taken as given: requires
 * sum w = 4 pi within 1e-12, c_m != 0, s_m != 0, M % 4 == 0. */
typedef struct {
  int M, n_polar, n_azim;
  const double *c, *s, *zeta, *w;
} rte_ordinates;

typedef struct rte_problem rte_problem;   /* opaque; immutable after setup except scratch */
typedef struct mgnet_net mgnet_net;       /* opaque */

/* rte_setup -- build the discrete problem (PAPER.md:23-37 eq:RTE + BCs, 69-74 eq:RTE_xy,
 * 90-104 eq:DORTE_2d, 113-117 cell values).
 *  sigma_T, sigma_a, q, eps : host float32 [batch][ny][nx] cell values.
 *  g                         : host float32 [batch], HG anisotropy, |g| < 1.
 *  inflow                    : host float32 [batch][4][N][M], faces in order
 *      L (x=0, indexed by j), R (x=1, by j), B (y=0, by i), T (y=1, by i);
 *      only incoming entries (u_m . n < 0) are read; may be NULL (zero inflow).
 * Computes (host, fp64): the quadrature, the row-normalised HG matrix
 * S = K W (R4, R5), per-cell sigma_t = sigma_T/eps,
 * sigma_s = sigma_T/eps - eps sigma_a, f = eps q (R7), and uploads them.
 * Errors (RTE_EINVAL): N < 1, nx != ny, batch < 1, bad ordinates, eps not in
 * (0,1], any sigma < 0, |g| >= 1, sigma_T/eps < eps sigma_a in a cell. */
rte_status rte_setup(const rte_grid* grid, const rte_ordinates* ord,
                     const float* sigma_T, const float* sigma_a, const float* q,
                     const float* eps, const float* g, const float* inflow,
                     rte_problem** out);
void rte_destroy(rte_problem* p);

/* rte_setup_tfps -- the TFPS alpha-space system of the same problem (NEXT-3; §2.2,
 * eq:2DTFPS_linear_sys; readings R37-R39 in DESIGN.md §3).  Same arguments and validation as rte_setup,
 * plus: every cell needs eps sigma_a > 0, and the medium must be piecewise constant with
 * at most 4096 distinct (sample, sigma_t, sigma_s) materials (RTE_EINVAL otherwise).
 * Per material it solves the local eigenproblems (gamma S - I) l = xi C l and (gamma S - I) l = xi S_y l,
 * gamma = sigma_s/sigma_t (eq:discretization_2D_eigenfunc_constraint; host fp64, symmetrised and solved
 * by Cholesky + Jacobi: all xi real), giving Md x-modes and Md y-modes per cell (Md = directions).
 * The problem's vectors then hold the basis coefficients alpha [batch][N][N][2 Md] (x-modes by
 * ascending xi, then y-modes), and on it
 *   rte_rhs   writes b (particular-solution jumps and inflow rows),
 *   rte_apply / rte_apply_f64 apply A alpha: the midpoint continuity rows of the faces x = i h
 *             (slots [0, Md) of cell (j, i)) and y = j h (slots [Md, 2Md)); the boundary rows of a
 *             row/column sit in the slots of its first cell (incoming directions only),
 *   gmres_solve solves A alpha = b (precond 0, or 1 with an MgNet created on this problem: 2 Md input
 *             channels; block Jacobi (2) is rejected),
 *   rte_problem_info reports M = 2 Md.  The ordinate set (rte_get_ordinates) keeps Md entries. */
rte_status rte_setup_tfps(const rte_grid* grid, const rte_ordinates* ord,
                          const float* sigma_T, const float* sigma_a, const float* q,
                          const float* eps, const float* g, const float* inflow,
                          rte_problem** out);
/* Host-only (no device work): the local modes of one material, as rte_setup_tfps computes them --
 * xi [2M] (x-modes ascending, then y-modes ascending) and L [M][2M] row-major (column k = l^k) for the
 * ordinates c, s, the row-stochastic S [M][M] (rte_hg_matrix) and gamma = sigma_s/sigma_t in [0, 1). */
rte_status rte_tfps_modes(int M, const double* c, const double* s, const double* S, double gamma, double* xi,
                          double* L);
/* Materials of a TFPS problem: nmat, Md, and (host, may be NULL) xi [nmat][2 Md] and the eigenvectors
 * L [nmat][Md][2 Md] (column k = l^k, ||l^k||_inf = 1, largest entry +1).  RTE_EINVAL if not TFPS. */
rte_status rte_tfps_info(const rte_problem* p, int* nmat, int* Md, double* xi, double* L);
/* psi at the cell centres from the coefficients (eq:2DTFPS_sol): psi_dev [batch][N][N][Md] =
 * sum_k alpha^k chi^k(z_c) + chi^s, alpha_dev [batch][N][N][2 Md] (float32 / float64). */
rte_status rte_tfps_reconstruct(const rte_problem* p, const float* alpha_dev, float* psi_dev, void* stream);
rte_status rte_tfps_reconstruct_f64(const rte_problem* p, const double* alpha_dev, double* psi_dev, void* stream);

/* rte_setup_atfps -- the ATFPS compressed system (NEXT-3b, eq:2DAdaptiveTFPS_linear_sys;
 * readings R40-R42 in DESIGN.md §3): the TFPS problem of rte_setup_tfps (same arguments, same checks)
 * compressed with the tolerance delta in (0, 1).  A mode k of a cell is kept iff
 * exp(-1/2 |xi_k| sigma_t h) > delta (eq:def_V_delta).  At every interface the kept centred eigenvectors
 * of both cells are orthonormalised (QR; each eta signed with its largest entry +1 and scaled to
 * ||eta||_inf = 1), the dropped ones follow, and P = [eta_kept | l_dropped]^-1 gives the projections;
 * the row of a kept mode is its P-row applied to the jump of the kept-mode traces at its interface
 * midpoint (eq:2DAdaptiveTFPS_continuity_cond), or to the incoming trace on a boundary face
 * (eq:2DAdaptiveTFPS_boundary_cond).  Vectors use the padded layout [batch][N][N][2 Md]: the row of a kept
 * mode sits at its own slot, dropped slots carry the identity row (b = 0 there), so the system is square
 * and its solution is 0 on dropped slots; rte_rhs / rte_apply / rte_apply_f64 / gmres_solve work on it as
 * on a TFPS problem.  Errors: RTE_EINVAL (delta, as rte_setup_tfps, linearly dependent kept modes at an
 * interface). */
rte_status rte_setup_atfps(const rte_grid* grid, const rte_ordinates* ord,
                           const float* sigma_T, const float* sigma_a, const float* q,
                           const float* eps, const float* g, const float* inflow, double delta,
                           rte_problem** out);
/* delta, the compressed dimension (kept unknowns over all cells) and (host, may be NULL) the kept mask
 * [nmat][2 Md] of an ATFPS problem. */
rte_status rte_atfps_info(const rte_problem* p, double* delta, int64_t* dim, uint8_t* sel);
/* Layer reconstruction (eq:2DAdaptive_TFPS_layer1/2): from the compressed solution alpha_dev (padded),
 * fills the dropped coefficients from the projected jumps of the smooth solution into full_dev (may be
 * NULL: problem scratch) and writes psi_delta at the cell centres to psi_dev [batch][N][N][Md]. */
rte_status rte_atfps_reconstruct(const rte_problem* p, const float* alpha_dev, float* psi_dev, float* full_dev,
                                 void* stream);
rte_status rte_atfps_reconstruct_f64(const rte_problem* p, const double* alpha_dev, double* psi_dev,
                                     double* full_dev, void* stream);

/* rte_set_source -- replace the source q (host [batch][N][N], >= 0) and, if inflow != NULL, the inflow
 * (host [batch][4][N][directions], layout of rte_setup) of an existing problem of any kind, keeping the
 * medium and everything derived from it: the right-hand side (rte_rhs; f = eps q, and chi^s = f / (eps sigma_a)
 * of a TFPS / ATFPS problem) changes, the operator does not.  For training over many right-hand sides per
 * medium (NEXT-4).  Synchronous.  Errors: RTE_EINVAL (NULL p or q, negative q). */
rte_status rte_set_source(rte_problem* p, const float* q, const float* inflow);

/* rte_atfps_fit -- D_delta of the filtered loss (NEXT-4, eq:loss / eq:loss_delta; reading
 * R43 in DESIGN.md §3): maps a discrete angular flux psi_dev [batch][N][N][Md] (cell centres, the
 * psi-space layout of rte_setup) to coefficients alpha_dev [batch][N][N][2 Md] (padded ATFPS layout) by a
 * per-cell least-squares fit: the samples at the centre and the four face midpoints (the average of the two
 * adjacent centre values; the cell's own value on a boundary face) minus the particular solution chi^s,
 * fitted by the cell's kept modes (minimum-norm solution); dropped slots get 0.  Device pointers, no
 * aliasing, asynchronous on `stream`.  The fit operators are built on the first call (host fp64).
 * Errors: RTE_EINVAL (NULL, not an ATFPS problem). */
rte_status rte_atfps_fit(const rte_problem* p, const float* psi_dev, float* alpha_dev, void* stream);
rte_status rte_atfps_fit_f64(const rte_problem* p, const double* psi_dev, double* alpha_dev, void* stream);
/* rte_atfps_loss -- the filtered loss loss_delta = ||b_bar - A_bar D_delta psi_d||_2 per sample (eq:loss_delta)
 * into the host array loss [batch] (the call synchronises `stream`), and, if grad_dev != NULL, its gradient
 * with respect to psi_d (sum over samples) into grad_dev [batch][N][N][Md]: D_lin^T A_bar^T (-r / ||r||)
 * (reading R45).  Reductions in fp64 (fixed order).  Errors: RTE_EINVAL (NULL psi/loss, aliasing, not an
 * ATFPS problem). */
rte_status rte_atfps_loss(const rte_problem* p, const float* psi_dev, double* loss, float* grad_dev, void* stream);
rte_status rte_atfps_loss_f64(const rte_problem* p, const double* psi_dev, double* loss, double* grad_dev,
                              void* stream);

/* Sizes of a problem: batch, N, M and n = batch*N*N*M. Any pointer may be NULL. */
rte_status rte_problem_info(const rte_problem* p, int* batch, int* N, int* M, int64_t* n);

/* Copy the ordinate set actually used (host arrays of length M directions; any may be NULL). */
rte_status rte_get_ordinates(const rte_problem* p, double* c, double* s, double* zeta, double* w);

/* Host-only setup helpers (no device work; usable without a GPU):
 * rte_quadrature fills the built-in product set (R2, R3; arrays of n_polar*n_azim);
 * rte_hg_matrix fills S = K W, [M][M] row-major, for ordinates c, s, zeta, w and anisotropy g
 * (PAPER.md:30-32 eq:hg; row normalisation sum_n K_mn w_n = 1, R4, R5). */
rte_status rte_quadrature(int n_polar, int n_azim, double* c, double* s, double* zeta, double* w);
rte_status rte_hg_matrix(int M, const double* c, const double* s, const double* zeta, const double* w,
                         double g, double* S);

/* b = eps q + inflow ghost terms: b_dev float32 [n]. */
rte_status rte_rhs(const rte_problem* p, float* b_dev, void* stream);

/* y = A x, the discrete-ordinates operator (R9):
 *  (A psi)_{jim} = (|c_m|/h + |s_m|/h + sigma_t) psi_{jim} - (|c_m|/h) psi_{j,i-sgn c_m,m}
 *                  - (|s_m|/h) psi_{j-sgn s_m,i,m} - sigma_s sum_n S_mn psi_{jin},
 * neighbours outside the grid are 0.  Fused upwind stencil + dense [cells x M].[M x M]
 * scattering GEMM (3xTF32 on tcgen05 tensor cores where M allows; fp32 accumulate).
 * x_dev, y_dev float32 [n]. */
rte_status rte_apply(const rte_problem* p, const float* x_dev, float* y_dev, void* stream);

/* Same operator in float64 (used for the fp64 restart residual; exported for tests). */
rte_status rte_apply_f64(const rte_problem* p, const double* x_dev, double* y_dev, void* stream);

/* mgnet_create -- linear MgNet V-cycle preconditioner (R12-R20).
 *  levels L >= 1, c0 = channels at level 0 (C_l = c0 2^l), nu = smoothing steps pre/post.
 *  weights: host float32, packed in the order of DESIGN.md R20 (PyTorch layouts):
 *    Lambda [c0][M][1][1]; for l = 0..L-1: A^l [C_l][C_l][3][3], pre B^{l,1..nu},
 *    post B'^{l,1..nu}; if l < L-1: R^l [C_{l+1}][C_l][3][3] (OIHW) and
 *    P^l [C_{l+1}][C_l][4][4] (conv_transpose IOHW); finally Theta [M][c0][1][1].
 *  n_floats must equal that count.  N must be divisible by 2^(L-1).
 * The net keeps its own device copies of the weights and its activation workspace. */
rte_status mgnet_create(const rte_problem* p, int levels, int c0, int nu,
                        const float* weights, size_t n_floats, mgnet_net** out);
void mgnet_destroy(mgnet_net* net);

/* z = [r +] V(r): one V-cycle on f^0 = Lambda r; z = Theta u^0 (+ r if add_identity).
 * r_dev, z_dev float32 [n], NHWC with M channels (the unknown layout). */
rte_status mgnet_vcycle(const mgnet_net* net, const float* r_dev, float* z_dev,
                        int add_identity, void* stream);

/* The same V-cycle entirely in float64 (SIMT kernels; fp64 weight copies and activation buffers are
 * created on first use).  Used by gmres_solve(precision=1) and as the fp64 parity reference of the
 * V-cycle's data flow.  r_dev, z_dev float64 [n]. */
rte_status mgnet_vcycle_f64(const mgnet_net* net, const double* r_dev, double* z_dev, int add_identity,
                            void* stream);

/* CoeffNet (NEXT-1; R31-R33): computes the modulation maps a^[l] and
 * abar^[l] = a^{-1,[l]} of every level from the medium (sigma_T, sigma_a, eps: host float32
 * [batch][N][N], the rte_setup arrays) and attaches them to `net`.  Every later V-cycle (fp32 and
 * fp64, and gmres_solve through it) then smooths with u <- u + abar (.) (B * (f - a (.) (A * u))).
 * Weights: host float32, packed per level l as trunk conv K_l [C_l][C_in][3][3] (C_in = 3 at l = 0,
 * else C_{l-1}; stride 1 at l = 0, 2 after), bias [C_l], a-head [C_l][C_l], bias [C_l], abar-head
 * [C_l][C_l], bias [C_l], C_l = c0 2^l; the trunk applies ReLU, the heads are linear (BatchNorm
 * folded).  n_floats must equal mgnet_coeffnet_weight_count(levels, c0).  weights == NULL removes
 * the maps (a = abar = 1).  Runs in fp64 at setup time and synchronises the device.  Must not run
 * concurrently with a V-cycle of the same net.  Errors: RTE_EINVAL (NULL field, count mismatch),
 * RTE_ENOMEM, RTE_ECUDA. */
size_t mgnet_coeffnet_weight_count(int levels, int c0);
rte_status mgnet_coeffnet(mgnet_net* net, const float* sigma_T, const float* sigma_a, const float* eps,
                          const float* weights, size_t n_floats);
/* Copies the fp64 map a^[level] (which = 0) or abar^[level] (which = 1), [batch][N_l][N_l][C_l]
 * NHWC, to host_out.  Errors: RTE_EINVAL (bad level/which, or no maps attached). */
rte_status mgnet_modulation(const mgnet_net* net, int level, int which, double* host_out);

/* Block-Jacobi preconditioner (NEXT-2; R35): z = A_cc^{-1} r per cell,
 * A_cc = diag((|c_m| + |s_m|)/h + sigma_t) - sigma_s S the restriction of A to the cell's M
 * ordinates.  r_dev, z_dev [n] (float32 / float64), must not alias.  Builds the inverse blocks on the
 * first call (fp64 Gauss-Jordan, kept by the problem).  Errors: RTE_EINVAL (sizes, see gmres_opts). */
rte_status rte_blockjacobi_apply(const rte_problem* p, const float* r_dev, float* z_dev, void* stream);
rte_status rte_blockjacobi_apply_f64(const rte_problem* p, const double* r_dev, double* z_dev, void* stream);

/* Restarted right-preconditioned GMRES(m) (R21, R22).
 * Preconditioner P = I + V (precond=1, requires net), P = I (precond=0), or block Jacobi
 * (precond=2, NEXT-2: P = A_cc^{-1} per cell, R35; the inverse blocks are built on the
 * first use and kept by the problem; RTE_EINVAL if cells x M^2 x 12 B > 24 GiB or M > 128).
 * Iterate x is float64; the Krylov basis is float32 (precision=0) or float64 (precision=1); dot
 * products accumulate in float64; every restart recomputes r = b - A x in float64.  The batch's
 * samples are independent solves with their own Arnoldi/Givens state. */
typedef struct {
  int restart;       /* m, 1..32 (gmres_prepare, gmres_solve and gmres_solve_host alike; a call
                        with another m than the cached workspace's re-allocates it) */
  int maxit;         /* cap on total inner iterations per sample */
  double rtol;       /* stop when ||b - A x|| <= rtol ||b|| */
  int precond;       /* 0 none, 1 MgNet (I + V), 2 block Jacobi */
  int reorth;        /* Gram-Schmidt of the Arnoldi step (all equal MGS in exact arithmetic):
                        3 = DCGS2 (recommended): delayed CGS2 -- the second CGS pass of the candidate
                            vector is deferred to the next step and fused with the first pass of the
                            new vector, so each step streams the basis twice (CGS1's traffic) with
                            CGS2's orthogonality; the Hessenberg column it corrects is finalised then
                            (the last one at the cycle end);
                        0 = CGS2: two classical Gram-Schmidt passes (three basis streams);
                        1 = one CGS pass;
                        2 = selective (DGKS): the second pass runs only when ||v'|| < ||w||/sqrt(2),
                            decided on the device (its fp32 orthogonality is too loose for
                            iteration-count parity on diffusive problems) */
  int precision;     /* 0 = mixed (default): float32 Krylov basis, operator apply and V-cycle, float64
                        iterate, reductions and restart residual;  1 = everything in float64 (basis,
                        apply, V-cycle on SIMT kernels): for tight tolerances and iteration-count
                        parity with an fp64 reference; not the fast path */
  int x0_zero;       /* 1 = the initial guess is zero: x is set to 0 by the call (its contents are not
                        read) and the first restart residual is b itself, so A x0 is not applied (same
                        result bits as passing x0 = 0 with x0_zero = 0); 0 = x holds x0 on entry */
} gmres_opts;

typedef struct {
  int iterations;    /* total inner iterations */
  int restarts;      /* cycles started */
  int converged;     /* true residual <= rtol ||b|| at exit */
  int breakdown;     /* 0 none; 1 lucky breakdown (h_{j+1,j} <= 1e-14 |col|: the Krylov space is
                        invariant, the solve ends); 2 a non-finite Arnoldi column stopped the
                        sample (x keeps the update of the finite columns; RTE_ENUMERIC) */
  double relres_true;/* ||b - A x|| / ||b|| in float64 at exit */
  double relres_est; /* last Arnoldi estimate |g_{j+1}| / ||b|| */
  double* history;   /* optional caller buffer, >= maxit doubles: estimate after each iteration */
  double* hessenberg;/* optional caller buffer, (restart+1)*restart doubles: the first cycle's
                        unrotated Hessenberg matrix H[i][j], row-major */
} gmres_report;

/* Optional setup for gmres_solve with these options (fp32 basis): captures, once, one CUDA graph per
 * Arnoldi step j of the step's operator part w = A P(alpha_j V_j) (preconditioner + apply, ~90
 * launches at config 5; the Krylov workspace is cached per problem, so every pointer of that part
 * is fixed per j) -- later solves replay them instead of launching each kernel (measured 5.9% on
 * apply + V-cycle).  Without it gmres_solve captures lazily (step seen once eagerly, captured on
 * the next use).  Graphs are dropped by mgnet_coeffnet, mgnet_destroy and rte_destroy; none are
 * used while per-launch timing records a class inside them, or with RTE_NO_GRAPHS set.  Runs
 * the operator once (results discarded).  Errors: RTE_EINVAL (options), RTE_ECUDA. */
rte_status gmres_prepare(const rte_problem* p, const mgnet_net* net, const gmres_opts* opts, void* stream);

/* b_dev float32 [n]; x_dev float64 [n] (in: x0, out: x); rep: array of `batch` reports. */
rte_status gmres_solve(const rte_problem* p, const mgnet_net* net, const float* b_dev,
                       double* x_dev, const gmres_opts* opts, gmres_report* rep, void* stream);

/* gmres_solve with HOST buffers (the end-to-end call): b_host float32 [n], x_host float64 [n]
 * (in: x0 unless opts->x0_zero, out: x); page-locked memory gives full-rate copies, pageable works.
 * b (and x0) are copied into problem-owned device buffers on `stream` (allocated on the first call,
 * 12 B per unknown, freed by rte_destroy); x is copied back as soon as the host knows the last cycle
 * has ended (budget spent, or every sample's Arnoldi estimate converged or broke down), on an
 * internal copy stream overlapping the closing fp64 true-residual apply -- if that residual starts
 * another cycle, x is copied again at exit.  Returns after x_host and rep are written.  Errors: as
 * gmres_solve. */
rte_status gmres_solve_host(const rte_problem* p, const mgnet_net* net, const float* b_host, double* x_host,
                            const gmres_opts* opts, gmres_report* rep, void* stream);

/* Kernel launches issued by this thread since the last call (reset to 0). */
int64_t rte_launch_count(int reset);

/* Per-launch device timing (measurement only; not on the product path unless enabled).
 * rte_timing_enable(1): every kernel launch of this thread is bracketed by a CUDA-event pair
 * recorded on the stream it is launched on, and tagged with its ALGORITHMIC flops and bytes
 * (DESIGN.md §5 states the per-unit figures).  rte_timing_get resolves the events (it
 * synchronises on the last one) and returns the aggregate of kernel class `idx`:
 * name (NUL-terminated, truncated to name_len), kind (0 HBM streaming, 1 3xTF32 tensor-core
 * contraction, 2 fp32 SIMT contraction, 3 fp64 SIMT, 4 latency-bound tiny kernel), launches,
 * total device ms, total algorithmic flops and bytes; *count receives the number of classes
 * (idx = -1 only queries the count).  rte_timing_reset clears the aggregates.  Any output
 * pointer may be NULL.  Errors: RTE_EINVAL (idx out of range), RTE_ECUDA. */
rte_status rte_timing_enable(int on);
/* Restrict per-launch timing to the class named `name` (NULL or "" = every class): the other
 * launches record no events (the event pairs of every launch cost ~10% of a GMRES step at
 * config 5, so bench.py times its headline solve with only the dominant class instrumented).
 * Errors: none. */
rte_status rte_timing_filter(const char* name);
/* Experiments only: per-role cycle counters of the tensor-core GEMM (collected when the
 * environment variable RTE_TC_DBG has bit 6 set); copies min(n, 24) counters, then zeroes them
 * if reset != 0.  Slot meanings are listed in csrc/tc_gemm.cuh (g_tc_prof). */
rte_status rte_debug_counters(uint64_t* out, int n, int reset);
rte_status rte_timing_reset(void);
rte_status rte_timing_get(int idx, char* name, int name_len, int* kind, int64_t* launches, double* ms,
                          double* flops, double* bytes, int* count);

const char* rte_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* RTE_H */
