"""fp64 CPU oracle of the TFPS alpha-space operator (NEXT-3; TEST INFRASTRUCTURE).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference``
legs may import this module; the product path never imports it and shares no code with it.

The tailored finite point scheme of PAPER.md:111-225 (§2.2), written out in the paper's order and
notation with the readings of DESIGN.md §3 (R7 scaling, R5 row-normalised kernel, R37-R40 below):

* Cell-wise constant coefficients: sigma_t = sigma_T/eps, sigma_s = sigma_T/eps -
  eps sigma_a, f = eps q (R7); the scheme assumes sigma_t - sigma_s = eps sigma_a > 0.
* Local eigenproblems (eq:discretization_2D_eigenfunc_constraint), with the
  discrete kernel K W read as the row-stochastic S = K~ W of R5 and gamma = sigma_s / sigma_t:
      x-modes: (gamma S - I) l = xi C l,   y-modes: (gamma S - I) l = xi S_y l,
  C = diag(c_m), S_y = diag(s_m).  M real eigenpairs per axis (numpy.linalg.eig as one library step),
  sorted ascending; M/2 negative and M/2 positive.  Eigenvectors normalised ||l||_inf = 1 with the
  largest-|.| entry positive (R37).
* Basis functions (eq:2D_eigenfunc): chi^k(z) = l^k exp(sigma_t xi^k . (z - z^k))
  with the reference point on the face the mode decays from, so |chi^k| <= 1 in the cell: x-modes
  with xi < 0 at x_l, xi > 0 at x_r; y-modes with xi < 0 at y_b, xi > 0 at y_t; the other coordinate
  at the cell centre (the garbled index map, read this way: R38).
  The 2M unknowns of a cell are ordered [x-modes by ascending xi, y-modes by ascending xi].
* Particular solution chi^s = f / (sigma_t - sigma_s) 1 (S 1 = 1).
* Equations (eq:2DTFPS_continuity_cond, eq:2DTFPS_boundary_cond), laid out per cell
  (R39) so that the system is square on the [cells][2M] layout of alpha:
    slots [0, M)  : the vertical face x = i h of cell (j, i): for i > 0 the midpoint continuity
                    psi_{(j,i-1)}(x_r) - psi_{(j,i)}(x_l) = 0 (all M directions); for i = 0 the
                    incoming boundary rows: c_m > 0 from the face x = 0 of cell (j, 0) and c_m < 0
                    from the face x = 1 of cell (j, N-1):  psi_C(face mid)_m = Psi_in.
    slots [M, 2M) : the horizontal face y = j h, likewise (s_m > 0 from y = 0 of cell (0, i), s_m < 0
                    from y = 1 of cell (N-1, i)).
  A alpha collects the basis-function terms; b = the inflow and particular-solution terms moved to
  the right (eq:2DTFPS_linear_sys).
* Reconstruction (eq:2DTFPS_sol): psi at the cell centre = sum_k alpha^k chi^k(z_c) + chi^s.

Pins (tests/test_oracle_tfps.py): pure absorber eigenpairs in closed form (xi = -1/c_m, unit vectors);
+-pairing of the spectrum; the basis functions solve the local homogeneous equation (finite-difference
derivatives) and are bounded by 1 in the cell; exact reproduction of global single-mode and constant
solutions on a homogeneous medium (closed-form alpha); dense LU solve == oracle GMRES; TFPS and the
psi-space upwind scheme converge to the same solution under refinement.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, Tuple

import numpy as np

from . import rte as R


@dataclasses.dataclass
class Modes:
    xi: np.ndarray      # [2M]  x-mode xi (ascending) then y-mode xi (ascending)
    L: np.ndarray       # [M][2M] eigenvectors as columns, same order
    axis: np.ndarray    # [2M]  0 = x-mode, 1 = y-mode


def local_modes(qd: R.Quadrature, S: np.ndarray, gamma: float) -> Modes:
    """Eigenpairs of eq:discretization_2D_eigenfunc_constraint for one material (R37)."""
    M = qd.c.size
    T = gamma * S - np.eye(M)
    xis, Ls, ax = [], [], []
    for axis, d in ((0, qd.c), (1, qd.s)):
        ev, V = np.linalg.eig(np.linalg.solve(np.diag(d), T))     # (gamma S - I) l = xi D l
        if np.max(np.abs(ev.imag)) > 1e-9 * np.max(np.abs(ev.real)):
            raise ValueError("complex TFPS eigenvalue")
        ev, V = ev.real, V.real
        order = np.argsort(ev)
        ev, V = ev[order], V[:, order]
        for k in range(M):
            v = V[:, k]
            a = np.abs(v)                                         # ties (within 1e-9, e.g. the +-1 pairs of
            big = int(np.nonzero(a >= a.max() * (1 - 1e-9))[0][0])   # the symmetric quadrature): lowest index
            V[:, k] = v / v[big]                                  # ||l||_inf = 1, largest entry +1
        xis.append(ev)
        Ls.append(V)
        ax.append(np.full(M, axis))
    return Modes(np.concatenate(xis), np.concatenate(Ls, axis=1), np.concatenate(ax))


@dataclasses.dataclass
class TFPS:
    N: int
    qd: R.Quadrature
    sig_t: np.ndarray        # [B][N][N]
    sig_s: np.ndarray
    f: np.ndarray
    S: np.ndarray            # [B][M][M]
    inflow: np.ndarray       # [B][4][N][M]
    mat: np.ndarray          # [B][N][N] material index into `modes`
    modes: list              # per material: Modes
    mat_key: list            # per material: (b, sigma_t, sigma_s)

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
        return (self.B, self.N, self.N, 2 * self.M)

    @property
    def chi_s(self):
        """Particular solution value per cell, f / (sigma_t - sigma_s)."""
        return self.f / (self.sig_t - self.sig_s)


def setup(N, n_polar, n_azim, sigma_T, sigma_a, q, eps, g, inflow) -> TFPS:
    """Cell coefficients (R7), scattering matrices (R4-R5) and the per-material local modes."""
    qd = R.quadrature(n_polar, n_azim)
    prob = R.setup(N, n_polar, n_azim, sigma_T, sigma_a, q, eps, g, inflow, qd)
    if np.any(prob.sig_t - prob.sig_s <= 0):
        raise ValueError("TFPS needs sigma_t > sigma_s (eps sigma_a > 0) in every cell (PAPER.md:117)")
    B = prob.B
    mat = np.zeros((B, N, N), np.int64)
    modes, keys, index = [], [], {}
    for b in range(B):
        for j in range(N):
            for i in range(N):
                key = (b, float(prob.sig_t[b, j, i]), float(prob.sig_s[b, j, i]))
                if key not in index:
                    index[key] = len(modes)
                    modes.append(local_modes(qd, prob.S[b], key[2] / key[1]))
                    keys.append(key)
                mat[b, j, i] = index[key]
    return TFPS(N, qd, prob.sig_t, prob.sig_s, prob.f, prob.S, prob.inflow, mat, modes, keys)


def setup_from_media(cfg, media) -> TFPS:
    return setup(cfg.N, cfg.n_polar, cfg.n_azim, media.sigma_T, media.sigma_a, media.q, media.eps, media.g,
                 media.inflow)


def basis_value(tp: TFPS, b: int, j: int, i: int, k: int, x: float, y: float) -> np.ndarray:
    """chi^k_C(x, y) of cell C = (j, i) (eq:2D_eigenfunc) with the R38 reference points."""
    h = tp.h
    md = tp.modes[tp.mat[b, j, i]]
    xi, l = md.xi[k], md.L[:, k]
    st = tp.sig_t[b, j, i]
    xl, xr, yb, yt = i * h, (i + 1) * h, j * h, (j + 1) * h
    if md.axis[k] == 0:
        ref = xl if xi < 0 else xr
        return l * np.exp(st * xi * (x - ref))
    ref = yb if xi < 0 else yt
    return l * np.exp(st * xi * (y - ref))


def _face_points(h, j, i):
    """Midpoints of the faces L, R, B, T of cell (j, i), and its centre."""
    xc, yc = (i + 0.5) * h, (j + 0.5) * h
    return {"L": (i * h, yc), "R": ((i + 1) * h, yc), "B": (xc, j * h), "T": (xc, (j + 1) * h), "C": (xc, yc)}


def face_matrices(tp: TFPS, m: int) -> Dict[str, np.ndarray]:
    """E_f [M][2M] for material m: column k = chi^k at the midpoint of face f in {L, R, B, T} (and the
    centre C) of a cell of that material.  The values depend on the material and h only (translation
    invariance of eq:2D_eigenfunc with cell-relative reference points), so they are evaluated on the
    first cell of the material with basis_value."""
    b, j, i = (int(v[0]) for v in np.nonzero(tp.mat == m))
    pts = _face_points(tp.h, j, i)
    return {f: np.stack([basis_value(tp, b, j, i, k, x, y) for k in range(2 * tp.M)], axis=1)
            for f, (x, y) in pts.items()}


def local_values(tp: TFPS, alpha: np.ndarray) -> Dict[str, np.ndarray]:
    """sum_k alpha^k_C chi^k_C at the face midpoints L, R, B, T and the centre C of every cell
    ([B][N][N][M] each); the particular solution is not included."""
    alpha = np.asarray(alpha, np.float64).reshape(tp.shape)
    B, N, M = tp.B, tp.N, tp.M
    out = {f: np.zeros((B, N, N, M)) for f in "LRBTC"}
    for m in range(len(tp.modes)):
        E = face_matrices(tp, m)
        sel = tp.mat == m
        for f in out:
            out[f][sel] = alpha[sel] @ E[f].T
    return out


def apply(tp: TFPS, alpha: np.ndarray) -> np.ndarray:
    """A alpha: the basis-function terms of the R39 equation rows (eq:2DTFPS_linear_sys)."""
    F = local_values(tp, alpha)
    B, N, M = tp.B, tp.N, tp.M
    c, s = tp.qd.c, tp.qd.s
    y = np.zeros(tp.shape)
    for b in range(B):
        for j in range(N):
            for i in range(N):
                if i > 0:                                     # continuity on x = i h
                    y[b, j, i, :M] = F["R"][b, j, i - 1] - F["L"][b, j, i]
                else:                                         # boundary rows of the row j
                    y[b, j, 0, :M] = np.where(c > 0, F["L"][b, j, 0], F["R"][b, j, N - 1])
                if j > 0:                                     # continuity on y = j h
                    y[b, j, i, M:] = F["T"][b, j - 1, i] - F["B"][b, j, i]
                else:
                    y[b, 0, i, M:] = np.where(s > 0, F["B"][b, 0, i], F["T"][b, N - 1, i])
    return y


def rhs(tp: TFPS) -> np.ndarray:
    """b of eq:2DTFPS_linear_sys: particular-solution jumps on interior faces, inflow minus the
    particular solution on boundary faces (eq:2DTFPS_continuity_cond, eq:2DTFPS_boundary_cond)."""
    B, N, M = tp.B, tp.N, tp.M
    c, s = tp.qd.c, tp.qd.s
    cs = tp.chi_s
    inf = tp.inflow
    y = np.zeros(tp.shape)
    for b in range(B):
        for j in range(N):
            for i in range(N):
                if i > 0:
                    y[b, j, i, :M] = cs[b, j, i] - cs[b, j, i - 1]
                else:
                    y[b, j, 0, :M] = np.where(c > 0, inf[b, 0, j] - cs[b, j, 0], inf[b, 1, j] - cs[b, j, N - 1])
                if j > 0:
                    y[b, j, i, M:] = cs[b, j, i] - cs[b, j - 1, i]
                else:
                    y[b, 0, i, M:] = np.where(s > 0, inf[b, 2, i] - cs[b, 0, i], inf[b, 3, i] - cs[b, N - 1, i])
    return y


def reconstruct(tp: TFPS, alpha: np.ndarray) -> np.ndarray:
    """psi at the cell centres (eq:2DTFPS_sol): [B][N][N][M]."""
    return local_values(tp, alpha)["C"] + tp.chi_s[..., None]


def dense_matrix(tp: TFPS) -> np.ndarray:
    """A assembled column by column from apply(e_k) (small problems only)."""
    n = int(np.prod(tp.shape))
    Ad = np.zeros((n, n))
    e = np.zeros(n)
    for k in range(n):
        e[k] = 1.0
        Ad[:, k] = apply(tp, e).ravel()
        e[k] = 0.0
    return Ad


def material_tables(tp: TFPS) -> Tuple[np.ndarray, np.ndarray]:
    """(xi [nmat][2M], L [nmat][M][2M]) for tests."""
    return np.stack([m.xi for m in tp.modes]), np.stack([m.L for m in tp.modes])
