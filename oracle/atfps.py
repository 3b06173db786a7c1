"""fp64 CPU oracle of the ATFPS compressed alpha-space system (NEXT-3b; TEST INFRASTRUCTURE).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference``
legs may import this module; the product path never imports it and shares no code with it.

The adaptive tailored finite point scheme of PAPER.md:228-412 (§2.3), on top of oracle/tfps.py, in the
paper's order with the readings R40-R42 of DESIGN.md §3:

* Selection (eq:def_V_delta): mode k of cell C is kept iff exp(-1/2 |xi^k| sigma_t h) > delta.
* Centring: a mode is centred at the face its reference point lies on (R38): x-modes
  with xi < 0 at L, xi > 0 at R; y-modes with xi < 0 at B, xi > 0 at T.  An interior interface i between
  C- (left / below) and C+ (right / above) collects C-'s R- (T-) centred modes and C+'s L- (B-) centred
  modes: M vectors in R^M.  A boundary face collects its cell's centred modes restricted to the M/2
  incoming directions: M/2 vectors in R^(M/2).
* Interface bases (R40): the selected centred eigenvectors, ordered [C- modes by k,
  C+ modes by k], are orthonormalised by QR (numpy.linalg.qr, one library step); each eta is then signed
  so its largest-|.| entry is positive (lowest index on ties within 1e-9) and scaled to ||eta||_inf = 1.
  The unselected centred eigenvectors follow unchanged, in the same order (they already have
  ||l||_inf = 1 on interior faces; on boundary faces the restriction is kept unscaled, so that
  P^k l^k = 1 holds exactly as eq:2DAdaptive_TFPS_layer2 uses it).  P = [eta_sel | eta_unsel]^-1 (the
  projection operators P^k of PAPER.md:313-323 are its rows).
* Compressed system (eq:2DAdaptiveTFPS_continuity_cond, eq:2DAdaptiveTFPS_boundary_cond,
  eq:2DAdaptiveTFPS_linear_sys; R41): one row per selected mode, the P-row of that mode's eta applied to
  the trace jump psi_sel|C- - psi_sel|C+ at the interface midpoint (selected modes only), or to the
  incoming trace on a boundary face.  The row of mode k of cell C is stored at slot (C, k) of the padded
  [cells][2M] layout (each selected mode is centred at exactly one face, so rows and unknowns pair up);
  the slots of unselected modes carry the identity row (y = alpha there, b = 0) and stay 0 in solutions.
* Layer reconstruction (eq:2DAdaptive_TFPS_layer1/2): unselected coefficients from the projected jumps
  of the smooth solution psi_bar = sum_sel alpha chi + chi^s; psi_delta = all modes + chi^s.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, Tuple

import numpy as np

from . import tfps as T

# the face a mode is centred at, and the neighbour across it
_FACE_OF = {(0, False): "L", (0, True): "R", (1, False): "B", (1, True): "T"}


def centre_faces(md: T.Modes):
    """Face (L, R, B, T) each of the 2M modes is centred at (R38 reference points)."""
    return [_FACE_OF[(int(md.axis[k]), bool(md.xi[k] > 0))] for k in range(md.xi.size)]


def select(tp: T.TFPS, m: int, delta: float) -> np.ndarray:
    """eq:def_V_delta for material m: exp(-1/2 |xi| sigma_t h) > delta."""
    st = tp.mat_key[m][1]
    return np.exp(-0.5 * np.abs(tp.modes[m].xi) * st * tp.h) > delta


def _sign_and_scale(v: np.ndarray) -> np.ndarray:
    a = np.abs(v)
    big = int(np.nonzero(a >= a.max() * (1 - 1e-9))[0][0])
    return v / v[big]                       # largest entry +1, ||.||_inf = 1


@dataclasses.dataclass
class Interface:
    cols: list          # [(side, k)] in basis order: selected (QR'd) first, then unselected
    nsel: int
    P: np.ndarray       # [d][d] = [eta_sel | eta_unsel]^-1
    dirs: np.ndarray    # direction indices of the d components (all M, or the incoming M/2)


@dataclasses.dataclass
class ATFPS:
    tp: T.TFPS
    delta: float
    sel: np.ndarray                    # [nmat][2M] bool
    faces: list                        # [nmat] list of centre faces
    inter: Dict[Tuple, Interface]      # (orient, m_minus, m_plus) for interior, (face, m) for boundary

    @property
    def shape(self):
        return self.tp.shape


def _interface(tp, faces, sel, mats, minus_face, plus_face, dirs) -> Interface:
    """Build the basis and projection of one interface type.  mats = (m_minus, m_plus) or (m,) for a
    boundary face; the centred modes of C- at `minus_face` and of C+ at `plus_face`."""
    cols_s, cols_u = [], []
    for side, m, f in ((0, mats[0], minus_face), (1, mats[-1], plus_face)):
        if f is None:
            continue
        for k in range(2 * tp.M):
            if faces[m][k] == f:
                (cols_s if sel[m][k] else cols_u).append((side, k))
    vec = lambda side, k: tp.modes[mats[side] if len(mats) > 1 else mats[0]].L[dirs, k]
    S = np.stack([vec(s, k) for s, k in cols_s], axis=1) if cols_s else np.zeros((dirs.size, 0))
    U = np.stack([vec(s, k) for s, k in cols_u], axis=1) if cols_u else np.zeros((dirs.size, 0))
    if cols_s:
        Q, _ = np.linalg.qr(S)
        Q = np.stack([_sign_and_scale(Q[:, j]) for j in range(Q.shape[1])], axis=1)
    else:
        Q = S
    E = np.concatenate([Q, U], axis=1)
    assert E.shape == (dirs.size, dirs.size), "interface basis is not square"
    return Interface(cols_s + cols_u, len(cols_s), np.linalg.inv(E), dirs)


def setup(tp: T.TFPS, delta: float) -> ATFPS:
    nmat = len(tp.modes)
    M = tp.M
    sel = np.stack([select(tp, m, delta) for m in range(nmat)])
    faces = [centre_faces(tp.modes[m]) for m in range(nmat)]
    c, s = tp.qd.c, tp.qd.s
    alld = np.arange(M)
    inter = {}
    for a in range(nmat):
        for b in range(nmat):
            inter[("x", a, b)] = _interface(tp, faces, sel, (a, b), "R", "L", alld)
            inter[("y", a, b)] = _interface(tp, faces, sel, (a, b), "T", "B", alld)
        for f, inc in (("L", c > 0), ("R", c < 0), ("B", s > 0), ("T", s < 0)):
            inter[(f, a)] = _interface(tp, faces, sel, (a,), f, None, np.nonzero(inc)[0])
    return ATFPS(tp, delta, sel, faces, inter)


def _masked(at: ATFPS, alpha):
    alpha = np.asarray(alpha, np.float64).reshape(at.shape)
    return alpha * at.sel[at.tp.mat]


def _rows(at: ATFPS, alpha, mode: str):
    """Projected interface rows.  mode 'apply': jumps of the selected traces (A alpha); 'rhs': the
    particular-solution / inflow terms (b); 'layer': the unselected coefficients of eq:2DAdaptive_TFPS_layer1/2
    from the smooth solution psi_bar."""
    tp = at.tp
    B, N, M = tp.B, tp.N, tp.M
    F = T.local_values(tp, _masked(at, alpha)) if mode != "rhs" else None
    cs = tp.chi_s
    out = np.zeros(at.shape)
    for b in range(B):
        for j in range(N):
            for i in range(N):
                m = tp.mat[b, j, i]
                for k in range(2 * M):
                    if (mode == "layer") == bool(at.sel[m][k]):
                        continue
                    f = at.faces[m][k]
                    nb = {"L": (j, i - 1), "R": (j, i + 1), "B": (j - 1, i), "T": (j + 1, i)}[f]
                    interior = 0 <= nb[0] < N and 0 <= nb[1] < N
                    if interior:
                        if f in ("L", "B"):
                            (jm, im), (jp, ip), side = nb, (j, i), 1
                        else:
                            (jm, im), (jp, ip), side = (j, i), nb, 0
                        orient = "x" if f in ("L", "R") else "y"
                        I = at.inter[(orient, tp.mat[b, jm, im], tp.mat[b, jp, ip])]
                        fm, fp = ("R", "L") if orient == "x" else ("T", "B")
                        if mode == "apply":
                            v = F[fm][b, jm, im] - F[fp][b, jp, ip]
                        elif mode == "rhs":
                            v = np.full(M, cs[b, jp, ip] - cs[b, jm, im])
                        else:  # layer: P^k(psi_bar|other) - P^k(psi_bar|own)
                            pm = F[fm][b, jm, im] + cs[b, jm, im]
                            pp = F[fp][b, jp, ip] + cs[b, jp, ip]
                            v = (pp - pm) if side == 0 else (pm - pp)
                    else:
                        I = at.inter[(f, m)]
                        own = F[f][b, j, i][I.dirs] if F is not None else None
                        face_in = {"L": (0, j), "R": (1, j), "B": (2, i), "T": (3, i)}[f]
                        psi_in = tp.inflow[b, face_in[0], face_in[1]][I.dirs]
                        side = 0
                        if mode == "apply":
                            v = own
                        elif mode == "rhs":
                            v = psi_in - cs[b, j, i]
                        else:
                            v = psi_in - (own + cs[b, j, i])
                    r = I.cols.index((side, k))
                    out[b, j, i, k] = I.P[r] @ v
    return out


def apply(at: ATFPS, alpha) -> np.ndarray:
    """The compressed operator on the padded layout (identity on the dropped slots, R41)."""
    alpha = np.asarray(alpha, np.float64).reshape(at.shape)
    y = _rows(at, alpha, "apply")
    drop = ~at.sel[at.tp.mat]
    y[drop] = alpha[drop]
    return y


def rhs(at: ATFPS) -> np.ndarray:
    return _rows(at, np.zeros(at.shape), "rhs")


def reconstruct(at: ATFPS, alpha) -> Tuple[np.ndarray, np.ndarray]:
    """(psi_delta at the cell centres, the full coefficient vector with the layer part filled in)."""
    a = _masked(at, alpha)
    full = a + _rows(at, a, "layer")
    return T.reconstruct(at.tp, full), full


def dimension(at: ATFPS) -> int:
    """Number of unknowns of the compressed system (selected modes over all cells)."""
    return int(at.sel[at.tp.mat].sum())
