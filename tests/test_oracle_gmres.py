"""Pins for the oracle's restarted right-preconditioned GMRES.

Library routine (scipy.sparse.linalg.gmres iteration counts, numpy LU), textbook
properties (exact-inverse preconditioner -> 1 step, unrestarted GMRES finishes in
<= n steps, residual monotone inside a cycle), and the zero-weight MgNet identity.
"""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

import workloads as W
from oracle import rte as O


def _small(N=4, np_=2, na=8, g=0.6, eps=0.3, seed=0):
    rng = np.random.default_rng(seed)
    M = np_ * na
    sT = np.exp(rng.standard_normal((1, N, N)))
    p = O.setup(N, np_, na, sT, np.full((1, N, N), 0.4), np.ones((1, N, N)),
                np.full((1, N, N), eps), [g], rng.uniform(0, 1, (1, 4, N, M)))
    return p


def test_exact_inverse_preconditioner_one_step():
    p = _small()
    Ad = O.dense_matrix(p)
    Ainv = np.linalg.inv(Ad)
    b = O.rhs(p)
    r = O.gmres(lambda v: O.apply(p, v), b, P=lambda v: (Ainv @ v.ravel()).reshape(v.shape),
                restart=30, rtol=1e-10, maxit=50)
    assert r.iterations == 1 and r.converged


def test_unrestarted_finishes_within_n():
    p = _small(N=2, np_=1, na=4)
    n = int(np.prod(p.shape))
    b = O.rhs(p)
    r = O.gmres(lambda v: O.apply(p, v), b, restart=n, rtol=1e-12, maxit=n)
    assert r.converged and r.iterations <= n


def test_residual_monotone_within_cycle():
    p = _small(N=6, np_=2, na=8, eps=0.05)
    b = O.rhs(p)
    r = O.gmres(lambda v: O.apply(p, v), b, restart=10, rtol=1e-10, maxit=200)
    h = np.array(r.history)
    for c in range(0, len(h), 10):
        seg = h[c:c + 10]
        assert np.all(np.diff(seg) <= 1e-15)


def _scipy_count(p, b, restart, rtol, maxit):
    n = b.size
    A = spla.LinearOperator((n, n), matvec=lambda v: O.apply(p, v.reshape(p.shape)).ravel(), dtype=np.float64)
    cnt = [0]
    def cb(_):
        cnt[0] += 1
    x, info = spla.gmres(A, b.ravel(), rtol=rtol, atol=0.0, restart=restart, maxiter=maxit,
                         callback=cb, callback_type="pr_norm")
    return cnt[0], info, x


def test_iteration_count_matches_scipy_cfg1():
    """Unpreconditioned GMRES(30), rtol 1e-8 on config 1: our count == scipy's (251)."""
    cfg = W.config(1)
    p = O.setup_from_media(cfg, W.make_media(cfg))
    b = O.rhs(p)
    ours = O.gmres(lambda v: O.apply(p, v), b, restart=30, rtol=1e-8, maxit=1000)
    n_sp, info, x_sp = _scipy_count(p, b, 30, 1e-8, 100)
    assert info == 0
    assert ours.iterations == n_sp == 251
    assert np.linalg.norm(ours.x.ravel() - x_sp) / np.linalg.norm(x_sp) < 1e-7


def test_iteration_count_matches_scipy_small_diffusive():
    p = _small(N=8, np_=2, na=8, eps=0.02, g=0.5, seed=3)
    b = O.rhs(p)
    ours = O.gmres(lambda v: O.apply(p, v), b, restart=30, rtol=1e-8, maxit=3000)
    n_sp, info, _ = _scipy_count(p, b, 30, 1e-8, 200)
    assert info == 0 and ours.converged
    assert abs(ours.iterations - n_sp) <= 1


def test_zero_weight_preconditioner_reproduces_history():
    """P = I + V with V ≡ 0 reproduces the unpreconditioned history exactly."""
    cfg = W.small_config(1, N=8, M=16, L=2, C0=4)
    p = O.setup_from_media(cfg, W.make_media(cfg))
    net = O.make_mgnet(np.zeros(W.mgnet_weight_count(cfg.M, cfg.L, cfg.C0, cfg.nu)), cfg.M, cfg.L, cfg.C0, cfg.nu)
    b = O.rhs(p)
    a = O.gmres(lambda v: O.apply(p, v), b, restart=30, rtol=1e-10, maxit=500)
    c = O.gmres(lambda v: O.apply(p, v), b, P=lambda v: O.vcycle(net, v), restart=30, rtol=1e-10, maxit=500)
    assert a.iterations == c.iterations and a.history == c.history


def test_mgnet_preconditioned_solution_matches_lu():
    """Right preconditioning leaves the solution unchanged: P = I + V(random) vs dense LU."""
    cfg = W.small_config(2, N=8, M=8, n_polar=1, n_azim=8, L=2, C0=4)
    p = O.setup_from_media(cfg, W.make_media(cfg))
    net = O.make_mgnet(W.make_weights(cfg, std=0.05), cfg.M, cfg.L, cfg.C0, cfg.nu)
    b = O.rhs(p)
    x_lu = np.linalg.solve(O.dense_matrix(p), b.ravel())
    r = O.gmres(lambda v: O.apply(p, v), b, P=lambda v: O.vcycle(net, v), restart=30, rtol=1e-11, maxit=5000)
    assert r.converged
    assert np.linalg.norm(r.x.ravel() - x_lu) / np.linalg.norm(x_lu) < 1e-8


def test_arnoldi_columns_consistent_with_gmres():
    """The first cycle's Arnoldi relation A P V_k = V_{k+1} H_k holds (unrotated H)."""
    p = _small(N=4)
    b = O.rhs(p)
    H = O.arnoldi_columns(lambda v: O.apply(p, v), b, None, 5)
    # rebuild V by the same recurrence and check orthonormality + relation
    Ad = O.dense_matrix(p)
    bb = b.ravel()
    V = [bb / np.linalg.norm(bb)]
    for j in range(5):
        w = Ad @ V[j]
        V.append((w - sum(H[i, j] * V[i] for i in range(j + 1))) / H[j + 1, j])
    Vm = np.array(V)
    assert np.allclose(Vm @ Vm.T, np.eye(6), atol=1e-12)
    assert np.allclose(Ad @ Vm[:5].T, Vm.T @ H, atol=1e-10)
