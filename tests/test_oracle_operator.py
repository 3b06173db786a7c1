"""Pins for the oracle's operator and right-hand side.

Closed forms / special cases: manufactured constant solution, pure-absorber
upwind sweep (textbook recursion, coded independently here), N=1 closed form,
linearity, D4 symmetry of config 1, dense LU vs GMRES, and the survey's
regression anchors (tests/golden/anchors_cfg12.json).
"""
import json
import math
import os

import numpy as np
import pytest

import workloads as W
from oracle import rte as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "anchors_cfg12.json")))


def _random_problem(N=8, np_=2, na=8, B=1, seed=0, eps=0.05, sa=0.3, g=0.7, C=None):
    rng = np.random.default_rng(seed)
    sT = np.exp(rng.standard_normal((B, N, N)))
    sA = np.full((B, N, N), sa)
    e = np.full((B, N, N), eps)
    q = sA * (C if C is not None else 1.0)
    gg = np.full(B, g)
    M = np_ * na
    inflow = np.full((B, 4, N, M), C if C is not None else 0.0)
    return O.setup(N, np_, na, sT, sA, q, e, gg, inflow)


@pytest.mark.parametrize("g", [0.0, 0.7, -0.4])
def test_manufactured_constant(g):
    """q = Cσ_a and inflow Ψ ≡ C on every incoming face give exactly ψ ≡ C (any σ_T, ε, g)."""
    C = 2.5
    p = _random_problem(N=8, np_=2, na=8, g=g, C=C)
    psi = np.full(p.shape, C)
    res = O.apply(p, psi) - O.rhs(p)
    assert np.linalg.norm(res) / np.linalg.norm(O.rhs(p)) < 1e-13


def test_linearity():
    p = _random_problem(N=6)
    rng = np.random.default_rng(1)
    x, y = rng.standard_normal(p.shape), rng.standard_normal(p.shape)
    a, b = 0.3, -1.7
    lhs = O.apply(p, a * x + b * y)
    rhs_ = a * O.apply(p, x) + b * O.apply(p, y)
    assert np.allclose(lhs, rhs_, rtol=1e-13, atol=1e-11)


def _sweep(N, qd, sig_t, b):
    """Textbook upwind transport sweep for σ_s = 0: per ordinate, visit cells in upwind order
    and solve (|c|/h + |s|/h + σ_t) ψ = b + |c|/h ψ_up_x + |s|/h ψ_up_y."""
    h = 1.0 / N
    psi = np.zeros((N, N, qd.c.size))
    for m in range(qd.c.size):
        ax, ay = abs(qd.c[m]) / h, abs(qd.s[m]) / h
        iorder = range(N) if qd.c[m] > 0 else range(N - 1, -1, -1)
        jorder = range(N) if qd.s[m] > 0 else range(N - 1, -1, -1)
        di = 1 if qd.c[m] > 0 else -1
        dj = 1 if qd.s[m] > 0 else -1
        for j in jorder:
            for i in iorder:
                upx = psi[j, i - di, m] if 0 <= i - di < N else 0.0
                upy = psi[j - dj, i, m] if 0 <= j - dj < N else 0.0
                psi[j, i, m] = (b[j, i, m] + ax * upx + ay * upy) / (ax + ay + sig_t[j, i])
    return psi


def test_pure_absorber_sweep():
    """σ_s = 0 (σ_T = ε²σ_a): A is a per-ordinate triangular upwind operator; the sweep solves it."""
    N, eps = 7, 0.5
    rng = np.random.default_rng(3)
    sA = rng.uniform(0.5, 2.0, (1, N, N))
    sT = eps * eps * sA
    p = O.setup(N, 2, 8, sT, sA, np.ones((1, N, N)), np.full((1, N, N), eps), [0.6],
                rng.uniform(0, 1, (1, 4, N, 16)))
    assert np.max(np.abs(p.sig_s)) < 1e-15
    b = O.rhs(p)
    psi = _sweep(N, p.qd, p.sig_t[0], b[0])
    assert np.allclose(O.apply(p, psi[None]), b, rtol=1e-13, atol=1e-12)


def test_single_cell_closed_form():
    """N = 1: A = diag(|c|/h + |s|/h + σ_t) − σ_s S (no interior neighbours)."""
    p = _random_problem(N=1, np_=2, na=8, g=0.5)
    M = p.M
    Ad = np.zeros((M, M))
    for k in range(M):
        e = np.zeros(p.shape); e[0, 0, 0, k] = 1
        Ad[:, k] = O.apply(p, e)[0, 0, 0]
    expect = np.diag(np.abs(p.qd.c) + np.abs(p.qd.s) + p.sig_t[0, 0, 0]) - p.sig_s[0, 0, 0] * p.S[0]
    assert np.allclose(Ad, expect, atol=1e-13)


def test_isotropic_apply_rank_one():
    """g = 0 contraction is φ/(4π): A ψ + σ_s φ/(4π) equals the pure transport part."""
    p = _random_problem(N=5, g=0.0)
    p0 = O.Problem(p.N, p.qd, p.sig_t, np.zeros_like(p.sig_s), p.f, p.S, p.inflow)
    psi = np.random.default_rng(5).standard_normal(p.shape)
    phi = psi @ p.qd.w
    assert np.allclose(O.apply(p, psi) + p.sig_s[..., None] * (phi / (4 * math.pi))[..., None],
                       O.apply(p0, psi), rtol=1e-13, atol=1e-12)


def _x_det(p):
    N = p.N
    x = (np.arange(N) + 0.5) / N
    return (1 + 0.5 * np.sin(2 * np.pi * x)[None, :, None] * np.cos(2 * np.pi * x)[:, None, None]
            + 0.25 * p.qd.c - 0.125 * p.qd.s)[None]


@pytest.mark.parametrize("k", [1, 2])
def test_regression_anchors_apply(k):
    a = GOLD[f"cfg{k}"]
    cfg = W.config(k)
    p = O.setup_from_media(cfg, W.make_media(cfg))
    b = O.rhs(p)
    y = O.apply(p, _x_det(p))
    assert abs(np.linalg.norm(b) - a["b_norm"]) < 1e-6 * a["b_norm"]
    assert abs(np.linalg.norm(y) - a["Ax_norm"]) < 1e-7 * a["Ax_norm"]
    assert abs(y.sum() - a["Ax_sum"]) < 1e-8 * abs(a["Ax_sum"])


def _perm(qd, fn):
    """Ordinate permutation m -> m' with (c', s', ζ') = fn(c, s, ζ), found by matching."""
    out = []
    for m in range(qd.c.size):
        c, s = fn(qd.c[m], qd.s[m])
        d = (qd.c - c) ** 2 + (qd.s - s) ** 2 + (qd.zeta - qd.zeta[m]) ** 2
        out.append(int(np.argmin(d)))
        assert d.min() < 1e-24
    return np.array(out)


def test_config1_solution_and_d4_symmetry():
    """Config 1 (uniform medium, zero inflow, symmetric source): GMRES to 1e-12 and the solution
    is invariant under the square's x-, y- and diagonal reflections with the matching ordinate
    permutation; iteration count and solution anchors match the golden file."""
    cfg = W.config(1)
    p = O.setup_from_media(cfg, W.make_media(cfg))
    b = O.rhs(p)
    r = O.gmres(lambda v: O.apply(p, v), b, restart=30, rtol=1e-8, maxit=1000)
    a = GOLD["cfg1"]
    assert r.converged and r.iterations == a["gmres_iters_unprec"]
    x = r.x[0]
    phi = x @ p.qd.w
    N = cfg.N
    assert abs(np.linalg.norm(x) - a["psi_norm"]) < 1e-3
    assert abs(phi[N // 2, N // 2] - a["phi_center"]) < 1e-4
    assert abs(phi[0, 0] - a["phi_corner"]) < 1e-5
    assert abs(x.max() - a["psi_max"]) < 1e-5
    r2 = O.gmres(lambda v: O.apply(p, v), b, restart=30, rtol=1e-12, maxit=3000)
    x = r2.x[0]
    px = _perm(p.qd, lambda c, s: (-c, s))
    py = _perm(p.qd, lambda c, s: (c, -s))
    pd = _perm(p.qd, lambda c, s: (s, c))
    sc = np.abs(x).max()
    assert np.max(np.abs(x[:, ::-1, :][:, :, px] - x)) < 1e-10 * sc
    assert np.max(np.abs(x[::-1, :, :][:, :, py] - x)) < 1e-10 * sc
    assert np.max(np.abs(np.transpose(x, (1, 0, 2))[:, :, pd] - x)) < 1e-10 * sc


def test_dense_lu_agrees_with_gmres():
    """Direct solve on a tiny grid agrees with GMRES at rtol 1e-12."""
    p = _random_problem(N=4, np_=2, na=8, g=0.6, eps=0.3)
    p.f[:] = 1.0
    p.inflow[:, 0] = 1.0
    Ad = O.dense_matrix(p)
    b = O.rhs(p)
    x_lu = np.linalg.solve(Ad, b.ravel())
    r = O.gmres(lambda v: O.apply(p, v), b, restart=30, rtol=1e-12, maxit=2000)
    assert r.converged
    assert np.linalg.norm(r.x.ravel() - x_lu) / np.linalg.norm(x_lu) < 1e-10


def test_rhs_inflow_faces():
    """Ghost terms enter exactly on the inflow face of each incoming ordinate."""
    N = 4
    p = O.setup(N, 1, 4, np.ones((1, N, N)), np.zeros((1, N, N)), np.zeros((1, N, N)),
                np.ones((1, N, N)), [0.0], np.zeros((1, 4, N, 4)))
    for face in range(4):
        p.inflow[:] = 0
        p.inflow[0, face] = 1.0
        b = O.rhs(p)[0]
        nz = np.argwhere(b != 0)
        for j, i, m in nz:
            c, s = p.qd.c[m], p.qd.s[m]
            if face == 0:
                assert i == 0 and c > 0 and abs(b[j, i, m] - abs(c) * N) < 1e-14
            if face == 1:
                assert i == N - 1 and c < 0
            if face == 2:
                assert j == 0 and s > 0 and abs(b[j, i, m] - abs(s) * N) < 1e-14
            if face == 3:
                assert j == N - 1 and s < 0
        assert len(nz) == N * 2   # n_azim=4, n_polar=1: 2 incoming ordinates per face cell
