"""GMRES parity on the fixed-budget configs 3, 4, 5 (SURVEY.md §8(c) "GMRES parity protocol" item 2;
DESIGN.md §6): the full-size MgNet-preconditioned GMRES(30) solve in the benchmarked mode (fp32 basis,
DCGS2, graphs, x0 = 0) against the fp64 oracle's reference run of the same budget.

The budgets (300 / 60 per sample / 30 iterations) end far from rtol, so there is no converged count to
compare; instead the residual history |g_{j+1}|/||b|| over the whole budget and the final iterate x (at
the seeded indices workloads.sample_indices) are compared with the band of the perturbed oracle runs
(the max deviation of a perturbed run from the reference run): K = 4 fp64 runs on perturbed inputs and
one run of the GPU's Gram-Schmidt with fp32 storage (scripts/make_bands_fp32.py; reading R36 v3).  The
asserted bound is max(2x band, a-priori floor) with the floors of reading R36 v4 (maxit * 2^-24 for the
history, the north star's 1e-4 for x); the ratio to the bare band is recorded.  The reference run, the perturbed runs
and the bands are stored in tests/golden/bands_cfg{k}.npz by scripts/make_bands.py, which calls only
oracle/ and workloads/ (the perturbation model is reading R36 in DESIGN.md §3).  Any config-4 sample
whose reference run converges within the budget is held to the north star's +-1 instead.
"""
import os

import numpy as np
import pytest

import workloads as W

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _band(k):
    path = os.path.join(GOLDEN, f"bands_cfg{k}.npz")
    assert os.path.exists(path), f"missing {path} (scripts/make_bands.py {k})"
    return np.load(path)


@pytest.mark.parametrize("k", [3, 4, 5])
def test_fixed_budget_gmres_within_oracle_band(k, margin):
    import paper_2604_23265_b200 as P
    g = _band(k)
    cfg = W.config(k)
    media = W.make_media(cfg)
    p = P.rte_setup(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                    n_polar=cfg.n_polar, n_azim=cfg.n_azim)
    net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, W.make_weights(cfg))
    b = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    P.rte_rhs(p, b)
    P.gmres_prepare(p, net, restart=cfg.restart)
    x = torch.empty(p.shape, dtype=torch.float64, device="cuda")
    reps = P.gmres_solve(p, net, b, x, restart=cfg.restart, maxit=cfg.maxit, rtol=cfg.rtol, x0_zero=True)
    torch.cuda.synchronize()
    idx = W.sample_indices(cfg)
    xs = x.cpu().numpy().reshape(cfg.B, -1)
    samples = sorted({int(key.split("_")[0][1:]) for key in g.files if key.startswith("s") and "_ref_" in key})
    assert samples, "band file has no samples"
    fails = []
    for s in samples:
        rep = reps[s]
        ref_hist = g[f"s{s}_ref_hist"]
        if bool(g[f"s{s}_ref_conv"]):       # converged within the budget: the north star's +-1
            assert margin(abs(rep["iterations"] - int(g[f"s{s}_ref_it"])), 1, f"s{s} iterations") <= 1
            continue
        assert rep["iterations"] == cfg.maxit == int(g[f"s{s}_ref_it"])
        dh = float(np.max(np.abs(rep["history"] - ref_hist) / ref_hist))
        dx = float(np.linalg.norm(xs[s, idx] - g[f"s{s}_ref_xs"]) / np.linalg.norm(g[f"s{s}_ref_xs"]))
        # the band: the largest deviation from the reference among the perturbed runs -- the K input-
        # perturbed fp64 runs and the fp32-storage run of the GPU's own Gram-Schmidt (R36 v3; absent keys
        # = that run is not in the golden file)
        band_h = 2.0 * max(float(g[f"s{s}_band_hist"]), float(g.get(f"s{s}_band_fp32_hist", 0.0)))
        band_x = 2.0 * max(float(g[f"s{s}_band_x"]), float(g.get(f"s{s}_band_fp32_x", 0.0)))
        # R36 v5: the run whose operators each carry a fixed relative error of the north star's single-
        # operator tolerance, as a random field and as a coherent bias (scripts/make_bands_fp32.py --op-tol 1e-5
        # [--coherent]); recorded against the larger of the two separately
        op_h = 2.0 * max(float(g.get(f"s{s}_band_op_hist", 0.0)), float(g.get(f"s{s}_band_opc_hist", 0.0)))
        op_x = 2.0 * max(float(g.get(f"s{s}_band_op_x", 0.0)), float(g.get(f"s{s}_band_opc_x", 0.0)))
        if op_h > 0.0:
            margin(dh, op_h, f"s{s} residual history vs 2x operator-tolerance band (recorded)")
            margin(dx, op_x, f"s{s} iterate x vs 2x operator-tolerance band (recorded)")
        # Recorded, not asserted: neither perturbation model contains the fp32 / 3xTF32 arithmetic *inside*
        # the operators (measured per-application errors 1e-6 ... 8e-6), and at configs 4-5 both bands are
        # tighter than that moves the history (R36 v4: measured ratios in parity_margins.md)
        margin(dh, band_h, f"s{s} residual history vs 2x emulation band (recorded)")
        margin(dx, band_x, f"s{s} iterate x vs 2x emulation band (recorded)")
        # Asserted (R36 v4, a-priori bounds): the history within max(2x band, maxit * u), u = 2^-24 the fp32
        # unit roundoff -- the first-order accumulation bound of an Arnoldi process stored in fp32 over the
        # budget's steps; the iterate within max(2x band, 1e-4), the north star's solution tolerance
        bh = max(band_h, op_h, cfg.maxit * 2.0 ** -24)
        bx = max(band_x, op_x, 1e-4)
        if margin(dh, bh, f"s{s} residual history vs max(2x band, maxit u_fp32)") > bh:
            fails.append((s, "history", dh, bh))
        if margin(dx, bx, f"s{s} iterate x vs max(2x band, 1e-4)") > bx:
            fails.append((s, "x", dx, bx))
        # and the iterate's norm agrees with the reference to the same bound
        dn = abs(np.linalg.norm(xs[s]) / float(g[f"s{s}_ref_xnorm"]) - 1.0)
        if margin(dn, bx, f"s{s} iterate norm vs the x bound") > bx:
            fails.append((s, "xnorm", dn, bx))
    assert not fails, fails
