"""fp64 CPU oracle for the MgNet-preconditioned GMRES hot path (TEST INFRASTRUCTURE).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module.  The product path
(``paper_2604_23265_b200``) never imports it and shares no code with it; the
only common dependency is the input generator ``workloads``.

Everything is plain numpy in float64, written in the paper's order and notation
(PAPER.md = /root/reference/PAPER.md, line numbers; readings Q1-Q30 are
SURVEY.md §8(c), restated in DESIGN.md §3).  Library primitives used as single
steps: ``numpy.polynomial.legendre.leggauss`` (Gauss-Legendre rule), matmul,
``numpy.linalg.norm``/``solve``.  No blocking, fusion or reordering beyond the
definitions.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): sphere-moment closed forms for
the quadrature, closed-form HG integrals (scipy quad), discrete conservation,
isotropic limit, manufactured constant solution, pure-absorber sweep, N=1 closed
form, D4 symmetry, torch-fp64 conv routines, adjoint identity, dense LU vs
GMRES, scipy GMRES iteration counts.  Every function below is pinned by at
least one of them (see DESIGN.md §4 pin table); nothing here is "parity unpinned".
"""
from __future__ import annotations

import dataclasses
import math
from typing import Callable, List, Optional

import numpy as np

FOUR_PI = 4.0 * math.pi


# ---------------------------------------------------------------------------
# 1. Angular discretisation  (§2.1 DOM; readings Q2, Q3)
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class Quadrature:
    c: np.ndarray      # [M] x-direction cosine  sqrt(1-zeta^2) cos(theta)
    s: np.ndarray      # [M] y-direction cosine  sqrt(1-zeta^2) sin(theta)
    zeta: np.ndarray   # [M] |z-component|, zeta in [0,1]
    w: np.ndarray      # [M] weights, sum = 4 pi (each node stands for +zeta and -zeta)


def quadrature(n_polar: int, n_azim: int) -> Quadrature:
    """Product quadrature {u_m, omega_m}.

    zeta_p, a_p: the n_polar-point Gauss-Legendre rule mapped to (0,1) (sum a_p = 1);
    theta_k = (k + 1/2) 2 pi / n_azim;  c = sqrt(1-zeta^2) cos theta,
    s = sqrt(1-zeta^2) sin theta,  w = 4 pi a_p / n_azim.
    Ordinates are ordered quadrant-major -- quadrants (+,+), (-,+), (-,-), (+,-) --
    then polar-major, then azimuth within the quadrant (reading R3).
    """
    if n_azim % 4 != 0 or n_polar < 1:
        raise ValueError("n_azim must be a multiple of 4 and n_polar >= 1")
    x, a = np.polynomial.legendre.leggauss(n_polar)       # rule on [-1, 1], sum a = 2
    zeta_p = 0.5 * (x + 1.0)
    a_p = 0.5 * a
    nq = n_azim // 4
    c, s, z, w = [], [], [], []
    for quad in range(4):
        for p in range(n_polar):
            for kk in range(nq):
                k = quad * nq + kk
                theta = (k + 0.5) * 2.0 * math.pi / n_azim
                r = math.sqrt(1.0 - zeta_p[p] ** 2)
                c.append(r * math.cos(theta))
                s.append(r * math.sin(theta))
                z.append(zeta_p[p])
                w.append(FOUR_PI * a_p[p] / n_azim)
    return Quadrature(np.array(c), np.array(s), np.array(z), np.array(w))


def hg(g: float, mu: np.ndarray) -> np.ndarray:
    """Henyey-Greenstein kernel (eq:hg): (1-g^2)/(1+g^2-2 g mu)^{3/2}."""
    return (1.0 - g * g) / (1.0 + g * g - 2.0 * g * mu) ** 1.5


def kappa_hat(qd: Quadrature, g: float) -> np.ndarray:
    """Pointwise HG at node pairs, averaged over the two 3-D directions (+-zeta') that a
    projected node stands for (Q4): 1/2 [HG(u_m.u_n^+) + HG(u_m.u_n^-)]."""
    planar = np.outer(qd.c, qd.c) + np.outer(qd.s, qd.s)
    zz = np.outer(qd.zeta, qd.zeta)
    return 0.5 * (hg(g, planar + zz) + hg(g, planar - zz))


def scattering_matrix(qd: Quadrature, g: float):
    """Discrete kernel (PAPER.md:92-94 kappa_mn; readings Q4, Q5).

    kappa_hat_mn = 1/2 [HG(c_m c_n + s_m s_n + zeta_m zeta_n) + HG(c_m c_n + s_m s_n - zeta_m zeta_n)]
    K_mn = kappa_hat_mn / sum_n' kappa_hat_mn' w_n'            (row normalisation)
    S_mn = K_mn w_n                                             (row-stochastic)
    Returns (K, S).
    """
    kh = kappa_hat(qd, g)
    K = kh / (kh @ qd.w)[:, None]
    S = K * qd.w[None, :]
    return K, S


# ---------------------------------------------------------------------------
# 2. Problem: coefficients, operator, right-hand side
#    (PAPER.md:23-27 eq:RTE, 69-74 eq:RTE_xy, 90-104 eq:DORTE_2d + BCs,
#     113-117 cell values; readings Q1, Q7-Q11)
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class Problem:
    N: int
    qd: Quadrature
    sig_t: np.ndarray    # [B][N][N] sigma_T / eps
    sig_s: np.ndarray    # [B][N][N] sigma_T / eps - eps sigma_a
    f: np.ndarray        # [B][N][N] eps q
    S: np.ndarray        # [B][M][M] row-stochastic K W per sample (g per sample)
    inflow: np.ndarray   # [B][4][N][M]

    @property
    def B(self):
        return self.sig_t.shape[0]

    @property
    def M(self):
        return self.qd.c.size

    @property
    def h(self):
        return 1.0 / self.N

    @property
    def shape(self):
        return (self.B, self.N, self.N, self.M)


def coefficients(sigma_T, sigma_a, q, eps):
    """Per-cell scaled coefficients (Q7):
    sigma_t = sigma_T/eps, sigma_s = sigma_T/eps - eps sigma_a, f = eps q."""
    sigma_T = np.asarray(sigma_T, np.float64); sigma_a = np.asarray(sigma_a, np.float64)
    q = np.asarray(q, np.float64); eps = np.asarray(eps, np.float64)
    return sigma_T / eps, sigma_T / eps - eps * sigma_a, eps * q


def setup(N, n_polar, n_azim, sigma_T, sigma_a, q, eps, g, inflow, qd: Optional[Quadrature] = None) -> Problem:
    qd = qd if qd is not None else quadrature(n_polar, n_azim)
    sig_t, sig_s, f = coefficients(sigma_T, sigma_a, q, eps)
    g = np.atleast_1d(np.asarray(g, np.float64))
    S = np.stack([scattering_matrix(qd, float(gb))[1] for gb in g])
    return Problem(N, qd, sig_t, sig_s, f, S, np.asarray(inflow, np.float64))


def setup_from_media(cfg, media, qd: Optional[Quadrature] = None) -> Problem:
    return setup(cfg.N, cfg.n_polar, cfg.n_azim, media.sigma_T, media.sigma_a, media.q,
                 media.eps, media.g, media.inflow, qd)


def _upwind_neighbours(psi: np.ndarray, qd: Quadrature):
    """psi at (j, i - sgn c_m) and (j - sgn s_m, i) with zero outside the grid (Q9)."""
    B, N, _, M = psi.shape
    px = np.zeros_like(psi)
    py = np.zeros_like(psi)
    cp, cn = qd.c > 0, qd.c < 0
    sp, sn = qd.s > 0, qd.s < 0
    px[:, :, 1:, cp] = psi[:, :, :-1, cp]        # c_m > 0: upwind cell is i-1
    px[:, :, :-1, cn] = psi[:, :, 1:, cn]        # c_m < 0: upwind cell is i+1
    py[:, 1:, :, sp] = psi[:, :-1, :, sp]        # s_m > 0: upwind cell is j-1
    py[:, :-1, :, sn] = psi[:, 1:, :, sn]        # s_m < 0: upwind cell is j+1
    return px, py


def apply(prob: Problem, psi: np.ndarray) -> np.ndarray:
    """y = A psi, the discrete-ordinates operator (PAPER.md:91-93 eq:DORTE_2d):

    (A psi)_{b,j,i,m} = (|c_m|/h + |s_m|/h + sigma_t) psi_{jim}
                        - (|c_m|/h) psi_{j,i-sgn c_m,m} - (|s_m|/h) psi_{j-sgn s_m,i,m}
                        - sigma_s sum_n S_mn psi_{jin}
    """
    psi = np.asarray(psi, np.float64).reshape(prob.shape)
    h = prob.h
    ax = np.abs(prob.qd.c) / h
    ay = np.abs(prob.qd.s) / h
    px, py = _upwind_neighbours(psi, prob.qd)
    B, N, _, M = psi.shape
    scatter = (psi.reshape(B, N * N, M) @ np.transpose(prob.S, (0, 2, 1))).reshape(psi.shape)  # sum_n S_mn psi_n
    return ((ax + ay)[None, None, None, :] + prob.sig_t[..., None]) * psi \
        - ax * px - ay * py - prob.sig_s[..., None] * scatter


def rhs(prob: Problem) -> np.ndarray:
    """b = eps q + inflow ghost terms (eq:boundary_condition_2d).

    b_{jim} = f_{ji} + (|c_m|/h) Psi_m on the inflow x-face when i - sgn c_m is outside
    the grid, + (|s_m|/h) Psi_m on the inflow y-face when j - sgn s_m is outside.
    Inflow layout [B][face L(x=0), R(x=1), B(y=0), T(y=1)][position along face][M].
    """
    B, N, M = prob.B, prob.N, prob.M
    h = prob.h
    ax = np.abs(prob.qd.c) / h
    ay = np.abs(prob.qd.s) / h
    b = np.repeat(prob.f[..., None], M, axis=-1).astype(np.float64)
    inf = prob.inflow
    for m in range(M):
        if prob.qd.c[m] > 0:
            b[:, :, 0, m] += ax[m] * inf[:, 0, :, m]          # left face x = 0, indexed by j
        elif prob.qd.c[m] < 0:
            b[:, :, N - 1, m] += ax[m] * inf[:, 1, :, m]      # right face x = 1
        if prob.qd.s[m] > 0:
            b[:, 0, :, m] += ay[m] * inf[:, 2, :, m]          # bottom face y = 0, indexed by i
        elif prob.qd.s[m] < 0:
            b[:, N - 1, :, m] += ay[m] * inf[:, 3, :, m]      # top face y = 1
    return b


# ---------------------------------------------------------------------------
# 3. MgNet V-cycle (§3.3; readings Q12-Q20)
# ---------------------------------------------------------------------------
def conv3x3(x: np.ndarray, W: np.ndarray, stride: int = 1) -> np.ndarray:
    """Cross-correlation, 3x3 kernel, zero padding 1 (Q18), NHWC x, OIHW W.

    out[b,y,x,o] = sum_{ky,kx,c} W[o,c,ky,kx] x_pad[b, stride*y+ky, stride*x+kx, c]
    """
    Bn, H, Wd, C = x.shape
    xp = np.zeros((Bn, H + 2, Wd + 2, C))
    xp[:, 1:H + 1, 1:Wd + 1, :] = x
    Ho, Wo = (H - 1) // stride + 1, (Wd - 1) // stride + 1
    out = np.zeros((Bn, Ho, Wo, W.shape[0]))
    for ky in range(3):
        for kx in range(3):
            patch = xp[:, ky:ky + stride * (Ho - 1) + 1:stride, kx:kx + stride * (Wo - 1) + 1:stride, :]
            out += patch @ W[:, :, ky, kx].T
    return out


def conv_transpose4x4_s2(x: np.ndarray, W: np.ndarray) -> np.ndarray:
    """Transposed conv, kernel 4, stride 2, padding 1 (Q18): the adjoint of
    the stride-2 pad-1 4x4 conv.  W is IOHW [C_in][C_out][4][4], x NHWC [.., H, W, C_in];
    out[b, 2y-1+ky, 2x-1+kx, o] += sum_c x[b,y,x,c] W[c,o,ky,kx]  (H -> 2H)."""
    Bn, H, Wd, _ = x.shape
    Co = W.shape[1]
    outp = np.zeros((Bn, 2 * H + 2, 2 * Wd + 2, Co))
    for ky in range(4):
        for kx in range(4):
            outp[:, ky:ky + 2 * H:2, kx:kx + 2 * Wd:2, :] += x @ W[:, :, ky, kx]
    return outp[:, 1:2 * H + 1, 1:2 * Wd + 1, :]


def conv1x1(x: np.ndarray, W: np.ndarray) -> np.ndarray:
    """1x1 conv (lift Lambda / head Theta, Q17): out[..., o] = sum_c W[o,c] x[..., c]."""
    return x @ W[:, :, 0, 0].T


def unpack_weights(w: np.ndarray, M: int, L: int, C0: int, nu: int) -> dict:
    """Read the packed weight vector in the order of SURVEY Q20 (fp32 -> fp64)."""
    w = np.asarray(w, np.float64)
    shapes = [("Lambda", (C0, M, 1, 1))]
    for l in range(L):
        C = C0 << l
        shapes.append((f"A{l}", (C, C, 3, 3)))
        shapes += [(f"Bpre{l}_{i}", (C, C, 3, 3)) for i in range(nu)]
        shapes += [(f"Bpost{l}_{i}", (C, C, 3, 3)) for i in range(nu)]
        if l < L - 1:
            shapes.append((f"R{l}", (2 * C, C, 3, 3)))
            shapes.append((f"P{l}", (2 * C, C, 4, 4)))
    shapes.append(("Theta", (M, C0, 1, 1)))
    out, off = {}, 0
    for name, shp in shapes:
        n = int(np.prod(shp))
        out[name] = w[off:off + n].reshape(shp)
        off += n
    if off != w.size:
        raise ValueError(f"weight count mismatch: expected {off}, got {w.size}")
    return out


@dataclasses.dataclass
class MgNet:
    W: dict
    M: int
    L: int
    C0: int
    nu: int


def make_mgnet(w, M, L, C0, nu) -> MgNet:
    return MgNet(unpack_weights(w, M, L, C0, nu), M, L, C0, nu)


def vcycle(net: MgNet, r: np.ndarray, add_identity: bool = True, mod: Optional[dict] = None) -> np.ndarray:
    """z = [r +] Theta u^0 after one MgNet V-cycle on f^0 = Lambda r (Q13-Q17).

    Smoothing step (Q13; "update the current solution based on the discrete operator
    information a[l] and the solution operator information a^{-1}[l]"):
        u <- u + abar^[l] (.) (B * (f - a^[l] (.) (A^l * u)))       ((.) = elementwise)
    with a = mod["a"][l], abar = mod["abar"][l] from CoeffNet (R31-R33); mod=None means
    a = abar = 1 (v1).  The restriction residual uses the same modulated operator.
    Down (l < L-1): nu pre-steps with B^{l,i}; f^{l+1} = R^l *_2 (f - a (.) A^l * u); u^{l+1} = 0 (Q16).
    Coarsest: 2 nu steps, pre then post B (Q15).
    Up: u^l += P^l^T *_2 u^{l+1}; nu post-steps with B'^{l,i}.
    """
    W = net.W
    r = np.asarray(r, np.float64)
    L, nu = net.L, net.nu
    a = (lambda l: mod["a"][l]) if mod is not None else (lambda l: 1.0)
    ab = (lambda l: mod["abar"][l]) if mod is not None else (lambda l: 1.0)
    f = [None] * L
    u = [None] * L
    f[0] = conv1x1(r, W["Lambda"])
    for l in range(L):
        u[l] = np.zeros_like(f[l])
        steps = [W[f"Bpre{l}_{i}"] for i in range(nu)]
        if l == L - 1:
            steps += [W[f"Bpost{l}_{i}"] for i in range(nu)]
        for Bw in steps:
            u[l] = u[l] + ab(l) * conv3x3(f[l] - a(l) * conv3x3(u[l], W[f"A{l}"]), Bw)
        if l < L - 1:
            f[l + 1] = conv3x3(f[l] - a(l) * conv3x3(u[l], W[f"A{l}"]), W[f"R{l}"], stride=2)
    for l in range(L - 2, -1, -1):
        u[l] = u[l] + conv_transpose4x4_s2(u[l + 1], W[f"P{l}"])
        for i in range(nu):
            u[l] = u[l] + ab(l) * conv3x3(f[l] - a(l) * conv3x3(u[l], W[f"A{l}"]), W[f"Bpost{l}_{i}"])
    z = conv1x1(u[0], W["Theta"])
    return r + z if add_identity else z


# ---------------------------------------------------------------------------
# 3b. CoeffNet (§3.2; readings R31-R33 in DESIGN.md)
# ---------------------------------------------------------------------------
def coeffnet_weight_shapes(L: int, C0: int):
    """Packed CoeffNet weight order (R33): per level l, the trunk conv K_l (C_l x C_in x 3 x 3,
    C_in = 3 at l = 0 else C_{l-1}; stride 1 at l = 0, 2 after) and its bias beta_l (C_l), then
    the two 1x1 heads G^a_l, g^a_l and G^abar_l, g^abar_l (C_l x C_l and C_l).  C_l = C0 2^l."""
    shapes = []
    for l in range(L):
        C = C0 << l
        Cin = 3 if l == 0 else (C0 << (l - 1))
        shapes += [(f"K{l}", (C, Cin, 3, 3)), (f"beta{l}", (C,)), (f"Ga{l}", (C, C, 1, 1)), (f"ga{l}", (C,)),
                   (f"Gb{l}", (C, C, 1, 1)), (f"gb{l}", (C,))]
    return shapes


def coeffnet(sigma_T, sigma_a, eps, w, L: int, C0: int) -> dict:
    """CoeffNet forward: x = [sigma_T, sigma_a, eps] along channels (NHWC
    [B][N][N][3]); trunk h^0 = ReLU(K_0 * x + beta_0), h^{l+1} = ReLU(K_{l+1} *_2 h^l + beta_{l+1})
    (conv + batch normalisation folded into (K, beta) + activation, strided for the pyramid);
    heads a^[l] = G^a_l h^l + g^a_l, abar^[l] = G^abar_l h^l + g^abar_l (1x1, linear), each
    [B][N/2^l][N/2^l][C0 2^l].  Returns {"a": [...], "abar": [...]}."""
    w = np.asarray(w, np.float64)
    P, off = {}, 0
    for name, shp in coeffnet_weight_shapes(L, C0):
        n = int(np.prod(shp))
        P[name] = w[off:off + n].reshape(shp)
        off += n
    if off != w.size:
        raise ValueError(f"CoeffNet weight count mismatch: expected {off}, got {w.size}")
    x = np.stack([np.asarray(sigma_T, np.float64), np.asarray(sigma_a, np.float64),
                  np.asarray(eps, np.float64)], axis=-1)
    out = {"a": [], "abar": []}
    h = x
    for l in range(L):
        h = np.maximum(conv3x3(h, P[f"K{l}"], stride=1 if l == 0 else 2) + P[f"beta{l}"], 0.0)
        out["a"].append(conv1x1(h, P[f"Ga{l}"]) + P[f"ga{l}"])
        out["abar"].append(conv1x1(h, P[f"Gb{l}"]) + P[f"gb{l}"])
    return out


# ---------------------------------------------------------------------------
# 4. Restarted right-preconditioned GMRES (Q21, Q22)
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class GmresResult:
    x: np.ndarray
    iterations: int
    converged: bool
    history: List[float]          # |g_{j+1}| / ||b|| after every inner iteration
    relres_true: float
    hessenberg: List[np.ndarray]  # per cycle, the (k+1) x k Hessenberg matrix
    breakdown: bool = False


def gmres(A: Callable[[np.ndarray], np.ndarray], b: np.ndarray,
          P: Optional[Callable[[np.ndarray], np.ndarray]] = None,
          restart: int = 30, rtol: float = 1e-8, maxit: int = 1000,
          x0: Optional[np.ndarray] = None) -> GmresResult:
    """GMRES(m) with right preconditioning, modified Gram-Schmidt and Givens rotations in fp64.

    x0 = 0 by default.  Inside a cycle the Arnoldi estimate |g_{j+1}| <= rtol ||b|| stops
    the cycle; at every restart the true residual ||b - A x|| is recomputed and decides
    convergence (Q22).  Cycle end: x <- x + P(V_k y_k).  Iterations = total inner steps.
    """
    shape = b.shape
    b = np.asarray(b, np.float64).ravel()
    n = b.size
    Pf = (lambda v: v) if P is None else (lambda v: np.asarray(P(v.reshape(shape)), np.float64).ravel())
    Af = lambda v: np.asarray(A(v.reshape(shape)), np.float64).ravel()
    x = np.zeros(n) if x0 is None else np.asarray(x0, np.float64).ravel().copy()
    bnorm = np.linalg.norm(b)
    total = 0
    history: List[float] = []
    hess: List[np.ndarray] = []
    breakdown = False
    if bnorm == 0.0:
        return GmresResult(np.zeros(shape), 0, True, [], 0.0, [])
    while True:
        r = b - Af(x)
        beta = np.linalg.norm(r)
        if beta <= rtol * bnorm or total >= maxit or breakdown:
            break
        m = restart
        V = np.zeros((m + 1, n))
        H = np.zeros((m + 1, m))
        cs = np.zeros(m); sn = np.zeros(m)
        g = np.zeros(m + 1); g[0] = beta
        V[0] = r / beta
        k = 0
        for j in range(m):
            w = Af(Pf(V[j]))
            for i in range(j + 1):                 # modified Gram-Schmidt
                H[i, j] = np.dot(w, V[i])
                w = w - H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            for i in range(j):                     # previous rotations
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            hjj, hj1 = H[j, j], H[j + 1, j]
            den = math.hypot(hjj, hj1)
            cs[j], sn[j] = hjj / den, hj1 / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            k = j + 1
            history.append(abs(g[j + 1]) / bnorm)
            if hj1 <= 1e-14 * den:                 # lucky breakdown
                breakdown = True
                break
            V[j + 1] = w / hj1
            if abs(g[j + 1]) <= rtol * bnorm or total >= maxit:
                break
        hess.append(H[:k + 1, :k].copy())
        y = np.zeros(k)                            # back substitution R y = g
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:k] @ y[i + 1:k]) / H[i, i]
        x = x + Pf(V[:k].T @ y)
    relres = np.linalg.norm(b - Af(x)) / bnorm
    return GmresResult(x.reshape(shape), total, bool(relres <= rtol), history, float(relres), hess, breakdown)


def arnoldi_columns(A, b, P, steps: int):
    """First ``steps`` Arnoldi columns of the right-preconditioned Krylov process from x0=0
    (classical definition h_ij = <A P v_j, v_i>, MGS); returns the unrotated (steps+1) x steps H."""
    shape = b.shape
    b = np.asarray(b, np.float64).ravel()
    Pf = (lambda v: v) if P is None else (lambda v: np.asarray(P(v.reshape(shape)), np.float64).ravel())
    Af = lambda v: np.asarray(A(v.reshape(shape)), np.float64).ravel()
    V = [b / np.linalg.norm(b)]
    H = np.zeros((steps + 1, steps))
    for j in range(steps):
        w = Af(Pf(V[j]))
        for i in range(j + 1):
            H[i, j] = np.dot(w, V[i])
            w = w - H[i, j] * V[i]
        H[j + 1, j] = np.linalg.norm(w)
        V.append(w / H[j + 1, j])
    return H


# ---------------------------------------------------------------------------
# 5. Dense reference (tests only; PAPER.md:44 direct LU)
# ---------------------------------------------------------------------------
def cell_blocks(prob: Problem) -> np.ndarray:
    """The per-cell diagonal blocks of A (NEXT-2 block Jacobi; "the standard Block
    Jacobi preconditioner"; SPEC.md:380 cell blocks): the terms of apply() that couple ordinates of
    one cell,  A_cc = diag(|c_m|/h + |s_m|/h + sigma_t) - sigma_s S.  [B][N][N][M][M]."""
    h = prob.h
    lam = (np.abs(prob.qd.c) + np.abs(prob.qd.s)) / h
    eye = np.eye(prob.M)
    return (lam[None, None, None, :, None] * eye + prob.sig_t[..., None, None] * eye
            - prob.sig_s[..., None, None] * prob.S[:, None, None, :, :])


def block_jacobi(prob: Problem) -> Callable[[np.ndarray], np.ndarray]:
    """P r = A_cc^{-1} r_c for every cell c (numpy.linalg.solve per block, one library step)."""
    Acc = cell_blocks(prob)

    def P(r):
        r = np.asarray(r, np.float64).reshape(prob.shape)
        return np.linalg.solve(Acc, r[..., None])[..., 0]
    return P


def dense_matrix(prob: Problem) -> np.ndarray:
    """Assemble A column by column via apply(e_k) (small problems only)."""
    n = int(np.prod(prob.shape))
    Ad = np.zeros((n, n))
    e = np.zeros(n)
    for k in range(n):
        e[k] = 1.0
        Ad[:, k] = apply(prob, e.reshape(prob.shape)).ravel()
        e[k] = 0.0
    return Ad
