"""Pins for the oracle's angular discretisation (PAPER.md:29-33 eq:hg, 79-94 §2.1).

Pinned against closed forms (sphere moments, HG integrals via scipy quad), the
discrete conservation invariant and the isotropic limit -- never against the
oracle's own formulas.
"""
import math

import numpy as np
import pytest
from scipy import integrate

from oracle import rte as O

SETS = [(2, 8), (2, 16), (4, 16), (4, 32), (8, 32), (3, 12), (1, 4)]


@pytest.mark.parametrize("np_,na", SETS)
def test_sphere_moments(np_, na):
    """Σw = 4π, Σw c = Σw s = 0, Σw c² = Σw s² = Σw ζ² = 4π/3 (exact for n_polar ≥ 2, n_azim ≥ 4)."""
    q = O.quadrature(np_, na)
    assert q.c.size == np_ * na
    assert abs(q.w.sum() - 4 * math.pi) < 1e-13
    assert abs((q.w * q.c).sum()) < 1e-13 and abs((q.w * q.s).sum()) < 1e-13
    assert abs((q.w * q.c * q.s).sum()) < 1e-13
    if np_ >= 2:
        for v in (q.c, q.s, q.zeta):
            assert abs((q.w * v * v).sum() - 4 * math.pi / 3) < 1e-13
    assert np.all(q.w > 0)
    assert np.allclose(q.c ** 2 + q.s ** 2 + q.zeta ** 2, 1.0, atol=1e-15)


@pytest.mark.parametrize("np_,na", SETS)
def test_polar_rule_exactness(np_, na):
    """The ζ-rule integrates ζ^k on (0,1) exactly for k < 2 n_polar (Gauss-Legendre degree)."""
    q = O.quadrature(np_, na)
    # one azimuth column per polar node: weights a_p = w n_azim / 4π
    nq = na // 4
    zeta_p = q.zeta[0:np_ * nq:nq]
    a_p = q.w[0:np_ * nq:nq] * na / (4 * math.pi)
    for k in range(2 * np_):
        assert abs((a_p * zeta_p ** k).sum() - 1.0 / (k + 1)) < 1e-14


@pytest.mark.parametrize("np_,na", SETS)
def test_sign_closure_and_nonzero(np_, na):
    """Set closed under (c,s) -> (-c,s), (c,-s), (-c,-s); c_m, s_m != 0."""
    q = O.quadrature(np_, na)
    key = {(round(c, 12), round(s, 12), round(z, 12)) for c, s, z in zip(q.c, q.s, q.zeta)}
    for c, s, z in zip(q.c, q.s, q.zeta):
        for sc, ss in ((-1, 1), (1, -1), (-1, -1)):
            assert (round(sc * c, 12), round(ss * s, 12), round(z, 12)) in key
    assert np.all(np.abs(q.c) > 1e-3) and np.all(np.abs(q.s) > 1e-3)


def test_quadrant_major_order():
    """Reading R3: quadrants (+,+), (-,+), (-,-), (+,-), each M/4 consecutive ordinates."""
    q = O.quadrature(4, 16)
    Mq = q.c.size // 4
    signs = [(1, 1), (-1, 1), (-1, -1), (1, -1)]
    for qi, (sc, ss) in enumerate(signs):
        sl = slice(qi * Mq, (qi + 1) * Mq)
        assert np.all(np.sign(q.c[sl]) == sc) and np.all(np.sign(q.s[sl]) == ss)


def test_config1_quadrature_values():
    """M=16 (2x8): ζ ∈ {1/2 ∓ 1/(2√3)} (2-point Gauss on (0,1)) and every weight π/4."""
    q = O.quadrature(2, 8)
    assert np.allclose(sorted(set(np.round(q.zeta, 14))), [0.5 - 0.5 / math.sqrt(3), 0.5 + 0.5 / math.sqrt(3)])
    assert np.allclose(q.w, math.pi / 4, atol=1e-15)


@pytest.mark.parametrize("g", [0.0, 0.5, 0.8, 0.9, -0.6])
def test_hg_closed_form_integrals(g):
    """∫_{S²} HG dΩ = 4π and ∫ HG μ dΩ = 4π g (closed form of eq:hg), by scipy quad."""
    f0 = lambda mu: 2 * math.pi * O.hg(g, np.array(mu))
    f1 = lambda mu: 2 * math.pi * mu * O.hg(g, np.array(mu))
    i0 = integrate.quad(f0, -1, 1, epsabs=1e-13, epsrel=1e-13, limit=200)[0]
    i1 = integrate.quad(f1, -1, 1, epsabs=1e-13, epsrel=1e-13, limit=200)[0]
    assert abs(i0 - 4 * math.pi) < 1e-9
    assert abs(i1 - 4 * math.pi * g) < 1e-9


@pytest.mark.parametrize("np_,na", SETS)
@pytest.mark.parametrize("g", [0.0, 0.5, 0.9, -0.3])
def test_discrete_conservation(np_, na, g):
    """Σ_n K_mn w_n = 1 for every m; S = K W row-stochastic; K ≥ 0."""
    q = O.quadrature(np_, na)
    K, S = O.scattering_matrix(q, g)
    assert np.max(np.abs(K @ q.w - 1.0)) < 1e-14
    assert np.max(np.abs(S.sum(axis=1) - 1.0)) < 1e-14
    assert np.all(K > 0)


def test_isotropic_limit():
    """g = 0: K ≡ 1/(4π) exactly, so (Sψ)_m = φ/(4π) with φ = Σ w ψ (rank one)."""
    q = O.quadrature(4, 16)
    K, S = O.scattering_matrix(q, 0.0)
    assert np.max(np.abs(K - 1 / (4 * math.pi))) < 1e-16
    psi = np.random.default_rng(0).standard_normal(q.c.size)
    assert np.allclose(S @ psi, (q.w @ psi) / (4 * math.pi), atol=1e-15)


def test_kappa_hat_symmetric():
    """κ depends only on u_m·u_n, so the unnormalised κ̂ is symmetric."""
    q = O.quadrature(4, 16)
    kh = O.kappa_hat(q, 0.7)
    assert np.allclose(kh, kh.T, atol=1e-14, rtol=0)


@pytest.mark.parametrize("g", [0.3, 0.5])
def test_raw_rowsums_converge(g):
    """Raw Σ_n κ̂_mn w_n / 4π -> 1 as the quadrature is refined (the 3-D ±ζ reading, Q4)."""
    errs = []
    for np_, na in ((2, 8), (4, 16), (8, 32), (12, 64)):
        q = O.quadrature(np_, na)
        errs.append(np.max(np.abs(O.kappa_hat(q, g) @ q.w / (4 * math.pi) - 1)))
    assert errs[-1] < 1e-3 and errs[-1] < errs[0]


@pytest.mark.parametrize("g", [0.4, 0.7])
def test_first_moment_continuum_limit(g):
    """∫ HG(u·u') (1 + u'_x) dΩ' = 4π (1 + g u_x): the discrete κ̂ contraction converges to it.
    A projected 2-D dot product or a missing ±ζ average fails this."""
    q = O.quadrature(16, 96)
    kh = O.kappa_hat(q, g)
    approx = kh @ (q.w * (1 + q.c))
    exact = 4 * math.pi * (1 + g * q.c)
    assert np.max(np.abs(approx - exact) / exact) < 2e-3
