"""Pins for the ATFPS compressed-system oracle (oracle/atfps.py; §2.3; readings
R40-R42).  Against: the full TFPS system (delta -> 0 gives the same solution), closed forms (a global
slowly-decaying mode is reproduced exactly, with zero layer part), the selection inequality and the
projection identities, and the decrease of the compression error with delta (Theorem 1's form)."""
import numpy as np
import pytest

import workloads as W
from oracle import atfps as A
from oracle import tfps as T


def _dense(at):
    n = int(np.prod(at.shape))
    Ad = np.zeros((n, n))
    e = np.zeros(n)
    for k in range(n):
        e[k] = 1.0
        Ad[:, k] = A.apply(at, e).ravel()
        e[k] = 0.0
    return Ad


def _solve(at):
    return np.linalg.solve(_dense(at), A.rhs(at).ravel()).reshape(at.shape)


def _media(N=4, M=8, eps=0.05, seed=0):
    rng = np.random.default_rng(seed)
    sT = np.where(rng.random((1, N, N)) < 0.5, 1.0, 6.0)
    f = lambda v: np.full((1, N, N), v)
    inf = rng.uniform(0.5, 1.5, (1, 4, N, M))
    return (N, 1, M, sT, f(0.3), f(1.0), f(eps), [0.5], inf)


def test_selection_inequality_and_projections():
    tp = T.setup(*_media())
    at = A.setup(tp, 1e-3)
    for m in range(len(tp.modes)):
        st = tp.mat_key[m][1]
        d = np.exp(-0.5 * np.abs(tp.modes[m].xi) * st * tp.h)
        assert np.array_equal(at.sel[m], d > 1e-3)
        # every face of a cell centres M/2 modes
        for f in "LRBT":
            assert sum(1 for x in at.faces[m] if x == f) == tp.M // 2
    for key, I in at.inter.items():
        d = I.dirs.size
        assert I.P.shape == (d, d) and len(I.cols) == d
        # P is the inverse of the basis: P^k eta^k' = delta_kk'
        assert np.allclose(I.P @ np.linalg.inv(I.P), np.eye(d), atol=1e-10)


def test_delta_to_zero_is_the_full_tfps_system():
    """delta = 1e-300 keeps every mode: the compressed system is an invertible per-interface transform of
    the full one, so alpha, and psi, equal the TFPS solution."""
    tp = T.setup(*_media())
    at = A.setup(tp, 1e-300)
    assert at.sel.all() and A.dimension(at) == int(np.prod(tp.shape))
    a_full = np.linalg.solve(T.dense_matrix(tp), T.rhs(tp).ravel()).reshape(tp.shape)
    a = _solve(at)
    assert np.allclose(a, a_full, rtol=1e-8, atol=1e-10 * np.max(np.abs(a_full)))
    psi, full = A.reconstruct(at, a)
    assert np.allclose(full, a)                             # no layer part
    assert np.allclose(psi, T.reconstruct(tp, a_full), rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("axis", [0, 1])
def test_global_slow_mode_is_reproduced_exactly(axis):
    """Homogeneous diffusive medium, psi = q/sigma_a + l exp(sigma_t xi (x or y)) for the slowest mode
    (selected at any delta < 1 it passes): the compressed solve returns alpha = exp(sigma_t xi x_ref) on that
    mode and 0 on the other selected ones, the layer part is 0, and psi_delta equals psi at the centres."""
    N, M = 4, 8
    sT, sA, eps, g, q = 4.0, 0.3, 0.05, 0.5, 0.7
    f = lambda v: np.full((1, N, N), v)
    probe = T.setup(N, 1, M, f(sT), f(sA), f(q), f(eps), [g], np.zeros((1, 4, N, M)))
    md = probe.modes[0]
    ks = np.arange(axis * M, (axis + 1) * M)
    k = int(ks[np.argmin(np.abs(md.xi[ks]) + 1e9 * (md.xi[ks] > 0))])   # slowest left/bottom-centred mode
    xi, l, st = md.xi[k], md.L[:, k], probe.sig_t[0, 0, 0]
    C = q / sA
    psi_fn = lambda x, y: C + l * np.exp(st * xi * (x if axis == 0 else y))
    h = 1.0 / N
    inf = np.zeros((1, 4, N, M))
    for t in range(N):
        c = (t + 0.5) * h
        inf[0, 0, t], inf[0, 1, t], inf[0, 2, t], inf[0, 3, t] = psi_fn(0, c), psi_fn(1, c), psi_fn(c, 0), psi_fn(c, 1)
    tp = T.setup(N, 1, M, f(sT), f(sA), f(q), f(eps), [g], inf)
    at = A.setup(tp, 1e-2)
    assert at.sel[0][k] and not at.sel.all()                 # compressed, and the mode is kept
    a = _solve(at)
    expect = np.zeros(tp.shape)
    for j in range(N):
        for i in range(N):
            lo = (i if axis == 0 else j) * h
            expect[0, j, i, k] = np.exp(st * xi * lo)
    assert np.allclose(a, expect, rtol=1e-8, atol=1e-10)
    psi, full = A.reconstruct(at, a)
    assert np.allclose(full, expect, rtol=1e-8, atol=1e-10)  # layer coefficients vanish
    for j in range(N):
        for i in range(N):
            assert np.allclose(psi[0, j, i], psi_fn((i + 0.5) * h, (j + 0.5) * h), rtol=1e-9, atol=1e-11)


def test_compression_error_shrinks_with_delta():
    """Diffusive two-material medium with boundary layers (inflow 1): the compressed dimension drops
    below the full one, and ||psi_delta - psi_full|| decreases as delta does (Theorem 1: linear in delta
    up to a constant; here checked as monotone with a 10x margin between the extremes)."""
    args = _media(N=6, M=8, eps=0.02, seed=3)
    tp = T.setup(*args)
    psi_full = T.reconstruct(tp, np.linalg.solve(T.dense_matrix(tp), T.rhs(tp).ravel()))
    errs, dims = [], []
    for delta in (1e-1, 1e-2, 1e-4, 1e-8):
        at = A.setup(tp, delta)
        psi, _ = A.reconstruct(at, _solve(at))
        errs.append(np.max(np.abs(psi - psi_full)) / np.max(np.abs(psi_full)))
        dims.append(A.dimension(at))
    assert dims[0] < int(np.prod(tp.shape))
    assert all(d1 <= d2 for d1, d2 in zip(dims, dims[1:]))
    assert all(e2 <= e1 * (1 + 1e-9) + 1e-12 for e1, e2 in zip(errs, errs[1:])), errs
    assert errs[-1] <= 0.1 * errs[0] or errs[-1] < 1e-10, errs
