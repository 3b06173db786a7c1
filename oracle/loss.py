"""fp64 CPU oracle of the filtered loss loss_delta (NEXT-4; TEST INFRASTRUCTURE).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference``
legs may import this module; the product path never imports it and shares no code with it.

The physics-informed loss of PAPER.md:492-507 (§3.4) on the ATFPS system of oracle/atfps.py, with the
readings R43-R45 of DESIGN.md §3:

* eq:loss_delta:  loss_delta = || b_bar_delta - A_bar_delta D_delta psi_d ||_2 per
  sample, on the padded [cells][2M] layout of oracle/atfps.py (its dropped rows vanish: A_bar is the
  identity there and D_delta puts 0 there, b_bar is 0 there).
* D_delta (R43; "D maps the discrete angular flux psi_d to the coefficients of the TFPS
  basis functions", constructed in SPEC.md:224-233): per cell C, psi_d is sampled at 5 collocation
  points -- the centre (psi_d[C] itself) and the midpoints of the faces L, R, B, T, where the value is
  the average of the two adjacent cell-centre values (psi_d[C] alone at a boundary face).  The samples
  minus the particular solution chi^s_C are fitted in least squares by sum_k alpha_k chi^k_C over the
  cell's SELECTED modes (eq:def_V_delta) -- the minimum-norm solution (numpy.linalg.lstsq, one library
  step); the dropped modes get 0.  The fit matrix of material m is G_m[p M + i][k] = chi^k(z_p)_i,
  p = C, L, R, B, T (oracle/tfps.py face_matrices).
* The gradient of loss_delta with respect to psi_d (what training back-propagates, R45):
  -D_lin^T A_bar^T r / ||r|| per sample, r = b_bar - A_bar D psi_d, with D_lin the linear part of the
  affine map D and both linear maps assembled column by column from unit vectors (small problems only).

Pins (tests/test_oracle_loss.py): psi_d = chi^s gives alpha = 0 and loss = ||b_bar|| (the particular
solution absorbs everything); the fit satisfies its normal equations G^T (G alpha - y) = 0; a field
that IS a single selected basis function at the 5 collocation points of one cell is recovered exactly;
D is affine; the exact ATFPS solution's own collocation samples give loss 0 when the samples are taken
from the solution's traces; the gradient matches central finite differences.
"""
from __future__ import annotations

import numpy as np

from . import atfps as A
from . import tfps as T

POINTS = ("C", "L", "R", "B", "T")
_OPP = {"L": "R", "R": "L", "B": "T", "T": "B"}


def fit_matrix(at: A.ATFPS, m: int) -> np.ndarray:
    """G_m restricted to the selected modes: [5M][n_sel] (rows: point-major C, L, R, B, T)."""
    E = T.face_matrices(at.tp, m)
    G = np.concatenate([E[p] for p in POINTS], axis=0)
    return G[:, at.sel[m]]


def samples(tp: T.TFPS, psi) -> np.ndarray:
    """Collocation samples of psi_d, [B][N][N][5][M] in the order C, L, R, B, T (R43)."""
    psi = np.asarray(psi, np.float64).reshape(tp.B, tp.N, tp.N, tp.M)
    N = tp.N
    out = np.empty(psi.shape[:3] + (5, tp.M))
    out[..., 0, :] = psi
    for p, (dj, di) in zip(range(1, 5), ((0, -1), (0, 1), (-1, 0), (1, 0))):
        for j in range(N):
            for i in range(N):
                jn, jn_i = j + dj, i + di
                if 0 <= jn < N and 0 <= jn_i < N:
                    out[:, j, i, p] = 0.5 * (psi[:, j, i] + psi[:, jn, jn_i])
                else:
                    out[:, j, i, p] = psi[:, j, i]
    return out


def D(at: A.ATFPS, psi) -> np.ndarray:
    """D_delta psi_d on the padded layout (R43)."""
    tp = at.tp
    Y = samples(tp, psi)
    alpha = np.zeros(at.shape)
    Gs = {}
    for b in range(tp.B):
        for j in range(tp.N):
            for i in range(tp.N):
                m = tp.mat[b, j, i]
                if m not in Gs:
                    Gs[m] = fit_matrix(at, m)
                y = (Y[b, j, i] - tp.chi_s[b, j, i]).ravel()
                a = np.linalg.lstsq(Gs[m], y, rcond=None)[0]
                alpha[b, j, i, at.sel[m]] = a
    return alpha


def residual(at: A.ATFPS, psi) -> np.ndarray:
    """r = b_bar - A_bar D psi_d (padded layout)."""
    return A.rhs(at) - A.apply(at, D(at, psi))


def loss(at: A.ATFPS, psi) -> np.ndarray:
    """eq:loss_delta per sample: [B]."""
    r = residual(at, psi)
    return np.sqrt(np.sum(r.reshape(at.tp.B, -1) ** 2, axis=1))


def _dense_linear(fn, n_in: int) -> np.ndarray:
    e = np.zeros(n_in)
    cols = []
    for k in range(n_in):
        e[k] = 1.0
        cols.append(np.ravel(fn(e)))
        e[k] = 0.0
    return np.stack(cols, axis=1)


def loss_grad(at: A.ATFPS, psi) -> np.ndarray:
    """d loss_delta / d psi_d (the sum over samples' losses), [B][N][N][M]; dense assembly of the
    linear parts of D and A_bar (small problems only)."""
    tp = at.tp
    psi = np.asarray(psi, np.float64).reshape(tp.B, tp.N, tp.N, tp.M)
    n_psi, n_al = psi.size, int(np.prod(at.shape))
    d0 = D(at, np.zeros_like(psi)).ravel()
    Dl = _dense_linear(lambda v: D(at, v.reshape(psi.shape)).ravel() - d0, n_psi)
    Al = _dense_linear(lambda v: A.apply(at, v.reshape(at.shape)), n_al)
    r = (A.rhs(at).ravel() - Al @ (Dl @ psi.ravel() + d0)).reshape(tp.B, -1)
    nr = np.sqrt(np.sum(r ** 2, axis=1))
    w = (r / nr[:, None]).ravel()
    return (-(Dl.T @ (Al.T @ w))).reshape(psi.shape)
