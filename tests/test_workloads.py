"""Sanity of the seeded input generators (inputs, not results: statistical checks only)."""
import numpy as np

import workloads as W


def test_grf_covariance():
    """Empirical correlation at lag r matches exp(-r²/2ℓ²) (SURVEY §8(d) GRF definition)."""
    rng = np.random.Generator(np.random.PCG64(7))
    ell = 8.0
    acc = {4: [], 8: [], 16: []}
    for _ in range(4):
        G = W.grf(rng, 256, ell, 1.0)
        assert abs(G.mean()) < 1e-12 and abs(G.std() - 1) < 1e-12
        for r in acc:
            acc[r].append(np.mean(G * np.roll(G, r, axis=1)))
    for r, v in acc.items():
        assert abs(np.mean(v) - np.exp(-r * r / (2 * ell * ell))) < 0.06


def test_configs_deterministic_and_shaped():
    for k in (1, 2, 3):
        c = W.config(k)
        a, b = W.make_media(c), W.make_media(c)
        assert np.array_equal(a.sigma_T, b.sigma_T)
        assert a.sigma_T.shape == (c.B, c.N, c.N) and a.inflow.shape == (c.B, 4, c.N, c.M)
        assert a.sigma_T.dtype == np.float32


def test_config4_constraints():
    c = W.small_config(4, N=64, M=16, n_polar=2, n_azim=8)
    m = W.make_media(c)
    assert m.sigma_T.shape[0] == 8
    assert np.all(m.sigma_T - m.sigma_a >= 0.2 - 1e-6)           # PAPER.md:520 shift
    assert np.all(m.eps >= 1e-4 - 1e-9) and np.all(m.eps <= 1.0)
    assert np.all((m.g >= 0) & (m.g <= 0.9))
    assert np.all(m.sigma_T / m.eps >= m.eps * m.sigma_a)         # non-negative scattering (Q11)
    for b in range(8):
        assert len(np.unique(m.sigma_T[b])) <= 32


def test_config2_layout():
    c = W.config(2)
    m = W.make_media(c)
    assert set(np.unique(m.sigma_T)) == {1.0, 10.0}
    assert m.sigma_T[0, 0, 0] == 1.0 and m.sigma_T[0, 0, 8] == 10.0 and m.sigma_T[0, 8, 8] == 1.0
    assert m.q.sum() == 32 * 32                                    # centre quarter
    assert np.all(m.inflow[:, 0] == 1) and np.all(m.inflow[:, 1:] == 0)


def test_weights_distribution():
    c = W.config(2)
    w = W.make_weights(c)
    assert w.size == W.mgnet_weight_count(c.M, c.L, c.C0, c.nu)
    assert abs(w.std() - 0.02) < 1e-3 and abs(w.mean()) < 1e-4
