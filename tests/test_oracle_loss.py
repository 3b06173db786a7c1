"""Pins of the filtered-loss oracle (oracle/loss.py; NEXT-4, PAPER.md:492-507 eq:loss_delta, readings
R43-R45 of DESIGN.md §3): closed forms of the loss (a constant exact solution gives 0; psi_d = chi^s on a
homogeneous medium gives ||b_bar||), exact recovery of one selected basis function from its collocation
samples (pins the face averaging, the neighbour directions and the point order of the fit), the normal
equations of the least-squares fit, affinity of D, and the gradient against central finite
differences."""
import numpy as np
import pytest

from oracle import atfps as A
from oracle import loss as Lo
from oracle import tfps as T


def _homog(N=4, M=8, sT=4.0, sA=0.3, q=0.7, eps=0.05, g=0.5, inflow=None):
    f = lambda v: np.full((1, N, N), v)
    inf = np.zeros((1, 4, N, M)) if inflow is None else inflow
    return T.setup(N, 1, M, f(sT), f(sA), f(q), f(eps), [g], inf)


def _two_material(N=4, M=8, seed=0, eps=0.05):
    rng = np.random.default_rng(seed)
    sT = np.where(rng.random((1, N, N)) < 0.5, 1.0, 6.0)
    f = lambda v: np.full((1, N, N), v)
    inf = rng.uniform(0.5, 1.5, (1, 4, N, M))
    return T.setup(N, 1, M, sT, f(0.3), f(1.0), f(eps), [0.5], inf)


def test_constant_exact_solution_has_zero_loss():
    """Homogeneous medium with inflow = chi^s = q / sigma_a: psi = chi^s solves the RTE, every collocation
    sample equals chi^s, so D psi = 0, b_bar = 0 and loss_delta = 0 exactly."""
    N, M, sA, q = 4, 8, 0.3, 0.7
    chis = q / sA
    tp = _homog(N, M, sA=sA, q=q, inflow=np.full((1, 4, N, M), chis))
    at = A.setup(tp, 1e-2)
    psi = np.full((1, N, N, M), chis)
    assert np.max(np.abs(Lo.D(at, psi))) < 1e-12
    assert Lo.loss(at, psi)[0] < 1e-12


def test_particular_solution_gives_rhs_norm():
    """Zero inflow: psi_d = chi^s gives alpha = 0 and loss_delta = ||b_bar||_2 (the boundary rows)."""
    tp = _homog()
    at = A.setup(tp, 1e-2)
    psi = np.broadcast_to(tp.chi_s[..., None], (1, tp.N, tp.N, tp.M)).copy()
    assert np.max(np.abs(Lo.D(at, psi))) < 1e-12
    b = A.rhs(at)
    assert abs(Lo.loss(at, psi)[0] - np.linalg.norm(b)) <= 1e-12 * np.linalg.norm(b)
    assert np.linalg.norm(b) > 0.1


@pytest.mark.parametrize("which", ["first", "last"])
def test_single_basis_function_is_recovered(which):
    """Interior cell C, a selected mode k: centre values = chi^k(z_C) + chi^s and each neighbour set so that
    the face average equals chi^k at that face midpoint + chi^s.  D returns e_k at C."""
    tp = _two_material(N=5)
    at = A.setup(tp, 1e-3)
    j, i = 2, 2
    m = tp.mat[0, j, i]
    ks = np.nonzero(at.sel[m])[0]
    k = int(ks[0] if which == "first" else ks[-1])
    E = T.face_matrices(tp, m)
    cs = tp.chi_s[0, j, i]
    rng = np.random.default_rng(3)
    psi = rng.uniform(0.0, 1.0, (1, tp.N, tp.N, tp.M))
    psi[0, j, i] = E["C"][:, k] + cs
    for f, (jn, jn_i) in (("L", (j, i - 1)), ("R", (j, i + 1)), ("B", (j - 1, i)), ("T", (j + 1, i))):
        psi[0, jn, jn_i] = 2.0 * (E[f][:, k] + cs) - psi[0, j, i]
    a = Lo.D(at, psi)[0, j, i]
    expect = np.zeros(2 * tp.M)
    expect[k] = 1.0
    assert np.max(np.abs(a - expect)) < 1e-9


def test_fit_satisfies_normal_equations_and_drops_unselected():
    tp = _two_material()
    at = A.setup(tp, 5e-2)
    assert not at.sel.all()
    rng = np.random.default_rng(1)
    psi = rng.uniform(0.0, 2.0, (1, tp.N, tp.N, tp.M))
    alpha = Lo.D(at, psi)
    Y = Lo.samples(tp, psi)
    for (j, i) in ((0, 0), (1, 2), (3, 3)):
        m = tp.mat[0, j, i]
        G = Lo.fit_matrix(at, m)
        y = (Y[0, j, i] - tp.chi_s[0, j, i]).ravel()
        a = alpha[0, j, i, at.sel[m]]
        assert np.linalg.norm(G.T @ (G @ a - y)) <= 1e-10 * np.linalg.norm(G.T @ y)
        assert np.all(alpha[0, j, i, ~at.sel[m]] == 0.0)


def test_D_is_affine():
    tp = _two_material()
    at = A.setup(tp, 1e-3)
    rng = np.random.default_rng(2)
    p1, p2 = rng.standard_normal((2, 1, tp.N, tp.N, tp.M))
    lhs = Lo.D(at, 0.3 * p1 + 0.7 * p2)
    rhs = 0.3 * Lo.D(at, p1) + 0.7 * Lo.D(at, p2)
    assert np.max(np.abs(lhs - rhs)) <= 1e-10 * max(1.0, np.max(np.abs(lhs)))


def test_gradient_matches_finite_differences():
    tp = _two_material(N=3, M=4)
    at = A.setup(tp, 1e-3)
    rng = np.random.default_rng(4)
    psi = rng.uniform(0.0, 2.0, (1, tp.N, tp.N, tp.M))
    g = Lo.loss_grad(at, psi)
    hstep = 1e-6
    for idx in [(0, 0, 0, 0), (0, 1, 1, 2), (0, 2, 1, 3), (0, 2, 2, 1)]:
        e = np.zeros_like(psi)
        e[idx] = hstep
        fd = (Lo.loss(at, psi + e)[0] - Lo.loss(at, psi - e)[0]) / (2 * hstep)
        assert abs(fd - g[idx]) <= 1e-6 * max(1.0, abs(fd)), (idx, fd, g[idx])
