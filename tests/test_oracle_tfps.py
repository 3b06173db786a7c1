"""Pins for the TFPS alpha-space oracle (oracle/tfps.py; §2.2; readings R37-R39).

Each pin fixes the oracle against something other than itself: closed forms (pure absorber spectrum,
exact single-mode and constant solutions of a homogeneous medium), properties the mathematics fixes
(+-pairing of the spectrum, boundedness of the basis in its cell, the basis solving the local PDE
checked by finite differences), a library routine (dense LU vs GMRES), and consistency with the
independent psi-space discretisation under refinement.
"""
import numpy as np
import pytest

import workloads as W
from oracle import rte as O
from oracle import tfps as T


def _homogeneous(N, n_polar, n_azim, sT, sA, eps, g, q=0.0, inflow=None):
    M = n_polar * n_azim
    f = lambda v: np.full((1, N, N), v, np.float64)
    inf = np.zeros((1, 4, N, M)) if inflow is None else inflow
    return T.setup(N, n_polar, n_azim, f(sT), f(sA), f(q), f(eps), [g], inf)


def test_pure_absorber_spectrum_closed_form():
    """gamma = 0: (0 S - I) l = xi C l gives xi = -1/c_m with eigenvectors supported on the directions
    of that c_m (SPEC.md tfps: 'eigenvalues {-1/c_m}')."""
    qd = O.quadrature(2, 8)
    _, S = O.scattering_matrix(qd, 0.5)
    md = T.local_modes(qd, S, 0.0)
    M = qd.c.size
    for axis, d in ((0, qd.c), (1, qd.s)):
        xi = md.xi[axis * M:(axis + 1) * M]
        assert np.allclose(xi, np.sort(-1.0 / d), rtol=1e-13)
        for k in range(M):
            l = md.L[:, axis * M + k]
            off = np.abs(-1.0 / d - xi[k]) > 1e-9 * abs(xi[k])
            assert np.max(np.abs(l[off])) < 1e-12 and np.isclose(np.max(l), 1.0)


@pytest.mark.parametrize("g,gamma", [(0.5, 0.99), (0.9, 0.5), (0.0, 0.999999)])
def test_spectrum_is_real_and_paired(g, gamma):
    """The sign-flip symmetry of the product quadrature pairs xi with -xi; M/2 modes decay each way."""
    qd = O.quadrature(2, 16)
    _, S = O.scattering_matrix(qd, g)
    md = T.local_modes(qd, S, gamma)
    M = qd.c.size
    for axis in (0, 1):
        xi = md.xi[axis * M:(axis + 1) * M]
        assert np.allclose(xi, -xi[::-1], rtol=1e-9, atol=1e-12)
        assert np.sum(xi < 0) == M // 2
        assert np.allclose(np.max(np.abs(md.L[:, axis * M:(axis + 1) * M]), axis=0), 1.0)


def test_basis_solves_the_local_equation_and_is_bounded():
    """Each chi^k solves c_m d_x psi + s_m d_y psi + sigma_t psi = sigma_s S psi in its cell
    (eq:discretization_2D_TFPS_local_homo), with the derivatives taken by central finite differences,
    and |chi^k| <= 1 in the cell (the reference points of PAPER.md:178)."""
    N = 4
    tp = _homogeneous(N, 2, 8, 3.0, 0.4, 0.5, 0.6)
    h = tp.h
    qd = tp.qd
    st, ss = tp.sig_t[0, 1, 2], tp.sig_s[0, 1, 2]
    rng = np.random.default_rng(0)
    d = 1e-6 * h
    for k in range(2 * tp.M):
        for _ in range(3):
            x = (2 + rng.uniform(0.1, 0.9)) * h
            y = (1 + rng.uniform(0.1, 0.9)) * h
            v = T.basis_value(tp, 0, 1, 2, k, x, y)
            dx = (T.basis_value(tp, 0, 1, 2, k, x + d, y) - T.basis_value(tp, 0, 1, 2, k, x - d, y)) / (2 * d)
            dy = (T.basis_value(tp, 0, 1, 2, k, x, y + d) - T.basis_value(tp, 0, 1, 2, k, x, y - d)) / (2 * d)
            res = qd.c * dx + qd.s * dy + st * v - ss * (tp.S[0] @ v)
            assert np.max(np.abs(res)) <= 1e-5 * st * max(np.max(np.abs(v)), 1e-3), k
            assert np.max(np.abs(v)) <= 1.0 + 1e-12
        for (x, y) in ((2 * h, 1 * h), (3 * h, 2 * h), (2 * h, 2 * h), (3 * h, 1 * h)):   # the corners
            assert np.max(np.abs(T.basis_value(tp, 0, 1, 2, k, x, y))) <= 1.0 + 1e-12


def _inflow_of(psi_fn, N, M):
    """Inflow array [1][4][N][M] holding psi at the boundary face midpoints (faces L, R, B, T)."""
    h = 1.0 / N
    inf = np.zeros((1, 4, N, M))
    for t in range(N):
        c = (t + 0.5) * h
        inf[0, 0, t] = psi_fn(0.0, c)
        inf[0, 1, t] = psi_fn(1.0, c)
        inf[0, 2, t] = psi_fn(c, 0.0)
        inf[0, 3, t] = psi_fn(c, 1.0)
    return inf


@pytest.mark.parametrize("axis,which", [(0, 0), (0, -1), (1, 3), (1, -2)])
def test_global_mode_is_reproduced_exactly(axis, which):
    """On a homogeneous medium, psi(x, y) = C + l exp(sigma_t xi (x or y)) (one global mode plus the
    particular solution C = q / sigma_a) solves the RTE exactly, so the TFPS solution must be it: every
    cell's coefficient of that mode is exp(sigma_t xi (ref - 0)) in closed form, all others 0, and the
    reconstruction equals psi at the cell centres."""
    N, npol, naz = 4, 1, 8
    sT, sA, eps, g, q = 2.0, 0.3, 0.5, 0.4, 0.7
    probe = _homogeneous(N, npol, naz, sT, sA, eps, g)
    M = probe.M
    md = probe.modes[0]
    k = axis * M + (which % M)
    xi, l = md.xi[k], md.L[:, k]
    st = probe.sig_t[0, 0, 0]
    C = q / sA
    psi_fn = lambda x, y: C + l * np.exp(st * xi * (x if axis == 0 else y))
    tp = _homogeneous(N, npol, naz, sT, sA, eps, g, q=q, inflow=_inflow_of(psi_fn, N, M))
    alpha = np.linalg.solve(T.dense_matrix(tp), T.rhs(tp).ravel()).reshape(tp.shape)
    h = tp.h
    expect = np.zeros(tp.shape)
    for j in range(N):
        for i in range(N):
            lo, hi = (i * h, (i + 1) * h) if axis == 0 else (j * h, (j + 1) * h)
            ref = lo if xi < 0 else hi
            expect[0, j, i, k] = np.exp(st * xi * ref)
    assert np.allclose(alpha, expect, rtol=1e-9, atol=1e-11)
    psi = T.reconstruct(tp, alpha)
    for j in range(N):
        for i in range(N):
            assert np.allclose(psi[0, j, i], psi_fn((i + 0.5) * h, (j + 0.5) * h), rtol=1e-9, atol=1e-11)


def test_constant_solution_on_piecewise_media():
    """q = C sigma_a per cell and inflow C on every face: psi = C everywhere across material
    interfaces, so b = 0 and alpha = 0 (eq:2DTFPS_linear_sys)."""
    N, M, C = 6, 8, 1.7
    rng = np.random.default_rng(1)
    sT = np.where(rng.random((1, N, N)) < 0.5, 2.0, 9.0)
    sA = np.where(rng.random((1, N, N)) < 0.5, 0.3, 0.6)
    tp = T.setup(N, 1, 8, sT, sA, C * sA, np.full((1, N, N), 0.1), [0.5], np.full((1, 4, N, M), C))
    assert len(tp.modes) > 1
    assert np.max(np.abs(T.rhs(tp))) < 1e-12
    assert np.allclose(T.reconstruct(tp, np.zeros(tp.shape)), C, rtol=1e-14)


def test_dense_solve_equals_gmres():
    """Library routine (LU) vs the oracle GMRES on the same alpha-space system (two materials)."""
    cfg = W.small_config(2, N=5, M=8, n_polar=1, n_azim=8)
    tp = T.setup_from_media(cfg, W.make_media(cfg))
    assert len(tp.modes) == 2
    b = T.rhs(tp)
    ad = np.linalg.solve(T.dense_matrix(tp), b.ravel())
    n = b.size                                  # unrestarted: converges in <= n steps
    res = O.gmres(lambda v: T.apply(tp, v), b, restart=n, rtol=1e-11, maxit=n)
    assert res.converged
    assert np.linalg.norm(res.x.ravel() - ad) <= 1e-9 * np.linalg.norm(ad)


def test_refinement_agrees_with_upwind_scheme():
    """TFPS and the psi-space upwind scheme (oracle.rte) discretise the same RTE, so their cell-centre
    solutions approach each other as h -> 0 (transport regime, where the upwind scheme is accurate):
    the difference, compared on the 4 x 4 coarse cells, shrinks under refinement."""
    diffs = []
    for N in (4, 8, 16):
        f = lambda v: np.full((1, N, N), v, np.float64)
        args = (N, 1, 8, f(1.0), f(0.5), f(1.0), f(1.0), [0.3], np.zeros((1, 4, N, 8)))
        tp = T.setup(*args)
        psi_t = T.reconstruct(tp, np.linalg.solve(T.dense_matrix(tp), T.rhs(tp).ravel()))
        pr = O.setup(*args)
        psi_u = np.linalg.solve(O.dense_matrix(pr), O.rhs(pr).ravel()).reshape(pr.shape)
        r = N // 4
        coarse = lambda p: p.reshape(1, 4, r, 4, r, 8).mean(axis=(2, 4))
        diffs.append(np.linalg.norm(coarse(psi_t) - coarse(psi_u)) / np.linalg.norm(coarse(psi_u)))
    assert diffs[1] < 0.75 * diffs[0] and diffs[2] < 0.75 * diffs[1], diffs
