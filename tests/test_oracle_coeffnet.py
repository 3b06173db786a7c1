"""Pins for the oracle's CoeffNet forward and the modulated MgNet smoother (NEXT-1; PAPER.md:453-465,
482; R31-R33).  Each pin is checked against something other than the oracle's own
formula: a closed form of a hand-built network, or the unmodulated V-cycle (itself pinned in
test_oracle_vcycle.py) with rescaled weights."""
import numpy as np
import pytest

import workloads as W
from oracle import rte as O


def _pack(parts):
    return np.concatenate([np.asarray(p, np.float64).ravel() for p in parts])


def test_coeffnet_weight_count_matches_layout_and_rejects_mismatch():
    cfg = W.small_config(1, N=8, M=16, L=3, C0=4)
    w = W.make_coeffnet_weights(cfg)
    assert w.size == W.coeffnet_weight_count(cfg.L, cfg.C0)
    # the workloads layout and the oracle's unpacking agree name by name
    assert [n for n, _ in W.coeffnet_weight_layout(3, 4)] == [n for n, _ in O.coeffnet_weight_shapes(3, 4)]
    f = np.ones((1, 8, 8))
    with pytest.raises(ValueError):
        O.coeffnet(f, f, f, w[:-1], cfg.L, cfg.C0)


def test_coeffnet_closed_form_pick_channel_network():
    """Trunk convs that pick one input channel at the centre tap, and identity heads, make the maps
    a closed-form ReLU chain of the inputs: with x = (sigma_T, sigma_a, eps),
      h^0_c = ReLU(x_{c mod 3} + beta0_c),   h^1_c[y, x] = ReLU(h^0_{c mod C0}[2y, 2x] + beta1_c),
      a^[l] = h^l + 1,  abar^[l] = 2 h^l - 0.5."""
    rng = np.random.default_rng(7)
    B, N, L, C0 = 2, 8, 2, 4
    sT, sa, ep = (rng.standard_normal((B, N, N)) for _ in range(3))
    parts = []
    betas = []
    for l in range(L):
        C = C0 << l
        Cin = 3 if l == 0 else C0 << (l - 1)
        K = np.zeros((C, Cin, 3, 3))
        for c in range(C):
            K[c, c % Cin, 1, 1] = 1.0
        beta = rng.uniform(-0.5, 0.5, C)
        betas.append(beta)
        parts += [K, beta, np.eye(C), np.ones(C), 2.0 * np.eye(C), -0.5 * np.ones(C)]
    out = O.coeffnet(sT, sa, ep, _pack(parts), L, C0)
    x = np.stack([sT, sa, ep], axis=-1)
    h0 = np.maximum(x[..., [c % 3 for c in range(C0)]] + betas[0], 0.0)
    h1 = np.maximum(h0[:, ::2, ::2, :][..., [c % C0 for c in range(2 * C0)]] + betas[1], 0.0)
    for l, h in enumerate([h0, h1]):
        assert out["a"][l].shape == (B, N >> l, N >> l, C0 << l)
        np.testing.assert_allclose(out["a"][l], h + 1.0, rtol=0, atol=1e-15)
        np.testing.assert_allclose(out["abar"][l], 2.0 * h - 0.5, rtol=0, atol=1e-15)


def test_modulated_vcycle_constant_maps_equal_rescaled_weights():
    """a = ka, abar = kb constant: u + kb B*(f - ka A*u) is the unmodulated smoother with weights
    (ka A, kb B), and the restriction residual f - ka A*u likewise; ka != kb tells a from abar."""
    cfg = W.small_config(2, N=16, M=8, n_polar=1, n_azim=8, L=3, C0=4)
    w = W.make_weights(cfg, std=0.1).astype(np.float64)
    net = O.make_mgnet(w, cfg.M, cfg.L, cfg.C0, cfg.nu)
    ka, kb = 0.7, 1.3
    mod = {"a": [np.full((cfg.B, cfg.N >> l, cfg.N >> l, cfg.C0 << l), ka) for l in range(cfg.L)],
           "abar": [np.full((cfg.B, cfg.N >> l, cfg.N >> l, cfg.C0 << l), kb) for l in range(cfg.L)]}
    scaled = dict(net.W)
    for name in net.W:
        if name.startswith("A"):
            scaled[name] = ka * net.W[name]
        elif name.startswith("Bpre") or name.startswith("Bpost"):
            scaled[name] = kb * net.W[name]
    net2 = O.MgNet(scaled, net.M, net.L, net.C0, net.nu)
    r = W.make_vector(cfg, 1).astype(np.float64)
    np.testing.assert_allclose(O.vcycle(net, r, False, mod=mod), O.vcycle(net2, r, False), rtol=1e-12, atol=1e-13)


def test_modulated_vcycle_unit_maps_and_linearity():
    """Unit maps reproduce the v1 V-cycle exactly; with CoeffNet maps the V-cycle stays linear in r
    (the maps depend on the medium only), as a fixed GMRES preconditioner must be."""
    cfg = W.small_config(3, N=16, M=16, n_polar=2, n_azim=8, L=2, C0=4)
    net = O.make_mgnet(W.make_weights(cfg, std=0.1), cfg.M, cfg.L, cfg.C0, cfg.nu)
    med = W.make_media(cfg)
    ones = {"a": [np.ones((cfg.B, cfg.N >> l, cfg.N >> l, cfg.C0 << l)) for l in range(cfg.L)]}
    ones["abar"] = ones["a"]
    r1, r2 = W.make_vector(cfg, 0).astype(np.float64), W.make_vector(cfg, 1).astype(np.float64)
    assert np.array_equal(O.vcycle(net, r1, True, mod=ones), O.vcycle(net, r1, True))
    mod = O.coeffnet(med.sigma_T, med.sigma_a, med.eps, W.make_coeffnet_weights(cfg, head_std=0.2), cfg.L, cfg.C0)
    lhs = O.vcycle(net, 2.0 * r1 - 3.0 * r2, False, mod=mod)
    rhs = 2.0 * O.vcycle(net, r1, False, mod=mod) - 3.0 * O.vcycle(net, r2, False, mod=mod)
    np.testing.assert_allclose(lhs, rhs, rtol=1e-11, atol=1e-12)
    assert not np.allclose(O.vcycle(net, r1, False, mod=mod), O.vcycle(net, r1, False))
