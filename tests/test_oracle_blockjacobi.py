"""Pins for NEXT-2: the paper's polynomial media and the oracle's block-Jacobi
preconditioner, against independent routes: the dense matrix
assembled column by column from apply() (pinned in test_oracle_operator.py), the exact inverse of
a one-cell problem, and the separable product form of the media."""
import numpy as np
import pytest

import workloads as W
from oracle import rte as O


def _problem(media, N, n_polar=1, n_azim=4, g=None):
    B = media.sigma_T.shape[0]
    g = media.g if g is None else np.full(B, g)
    return O.setup(N, n_polar, n_azim, media.sigma_T, media.sigma_a, media.q, media.eps, g, media.inflow)


@pytest.mark.parametrize("regime", ["diffusion", "transport", "centre"])
def test_cell_blocks_are_the_diagonal_blocks_of_the_dense_matrix(regime):
    N, M = 4, 8
    med = W.paper_media(2, N=N, degree=3, regime=regime, M=M, seed=3)
    prob = _problem(med, N, n_polar=1, n_azim=8, g=0.4)
    Ad = O.dense_matrix(prob)
    blocks = O.cell_blocks(prob)
    n_cell = N * N
    for b in range(2):
        for c in range(n_cell):
            k0 = (b * n_cell + c) * M
            np.testing.assert_allclose(blocks[b].reshape(n_cell, M, M)[c], Ad[k0:k0 + M, k0:k0 + M],
                                       rtol=1e-14, atol=1e-12)


def test_block_jacobi_is_the_exact_inverse_on_one_cell():
    """N = 1: A has no inter-cell coupling, so P = A^{-1} and GMRES needs one iteration."""
    med = W.paper_media(3, N=1, degree=2, regime="diffusion", M=8, seed=4)
    prob = _problem(med, 1, n_polar=2, n_azim=4, g=0.3)
    P = O.block_jacobi(prob)
    x = np.random.default_rng(0).standard_normal(prob.shape)
    np.testing.assert_allclose(P(O.apply(prob, x)), x, rtol=1e-10, atol=1e-12)
    b = W.make_paper_rhs(3, N=1, M=8, seed=1).astype(np.float64)
    res = O.gmres(lambda v: O.apply(prob, v), b, P, restart=30, rtol=1e-10, maxit=50)
    assert res.converged and res.iterations == 1


def test_block_jacobi_reduces_diffusion_iterations():
    """The comparison SPEC.md:372 asserts: block Jacobi beats no preconditioner on a diffusive system."""
    N = 16
    med = W.paper_media(1, N=N, degree=2, regime="diffusion", M=4, seed=5)
    prob = _problem(med, N)
    b = W.make_paper_rhs(1, N=N, M=4, seed=2).astype(np.float64)
    A = lambda v: O.apply(prob, v)
    plain = O.gmres(A, b, None, restart=30, rtol=1e-8, maxit=3000)
    bj = O.gmres(A, b, O.block_jacobi(prob), restart=30, rtol=1e-8, maxit=3000)
    assert bj.converged and bj.iterations < plain.iterations


@pytest.mark.parametrize("regime", W.PAPER_REGIMES)
def test_paper_media_form_and_constraints(regime):
    N = 32
    med = W.paper_media(4, N=N, degree=4, regime=regime, seed=6)
    assert (med.sigma_T - med.sigma_a).min() >= 0.2 - 1e-6
    assert med.sigma_a.min() > 0
    X = (np.arange(N) + 0.5) / N
    for b in range(4):
        # sigma_a is an unshifted product p(x) q(y): rank one; sigma_T at most rank two (+ shift)
        assert np.linalg.matrix_rank(med.sigma_a[b].astype(np.float64), tol=1e-4) == 1
        assert np.linalg.matrix_rank(med.sigma_T[b].astype(np.float64), tol=1e-4) <= 2
        e = med.eps[b]
        diff = e < 0.5
        assert np.all((e == 1.0) | ((e >= 0.001 - 1e-9) & (e <= 0.011 + 1e-9)))
        expect = {"diffusion": np.ones((N, N), bool), "transport": np.zeros((N, N), bool),
                  "lr": np.broadcast_to(X[None, :] < 0.5, (N, N)), "rl": np.broadcast_to(X[None, :] >= 0.5, (N, N)),
                  "tb": np.broadcast_to(X[:, None] < 0.5, (N, N)), "bt": np.broadcast_to(X[:, None] >= 0.5, (N, N))}
        centre = (X[None, :] > 0.25) & (X[None, :] < 0.75) & (X[:, None] > 0.25) & (X[:, None] < 0.75)
        expect["centre"], expect["outer"] = centre, ~centre
        assert np.array_equal(diff, expect[regime])
