"""Robustness of the GMRES driver (include/rte.h gmres_opts / gmres_report):
  * the cached Krylov workspace follows the restart length and the precision mode (a solve after
    another solve with a different restart or precision equals the same solve on a fresh problem);
  * one restart range, 1..32, for gmres_prepare, gmres_solve and gmres_solve_host;
  * the NaN/Inf guard: a non-finite Arnoldi column stops the sample (breakdown = 2, RTE_ENUMERIC)."""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

CFG = W.small_config(4, N=16, M=16, n_polar=2, n_azim=8, L=2, C0=16, B=3)


def _setup(cfg=CFG, weights=None):
    import paper_2604_23265_b200 as P
    media = W.make_media(cfg)
    p = P.rte_setup(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                    n_polar=cfg.n_polar, n_azim=cfg.n_azim)
    w = W.make_weights(cfg, std=0.05) if weights is None else weights
    net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, w)
    b = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    P.rte_rhs(p, b)
    return P, p, net, b


def _solve(P, p, net, b, **kw):
    x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
    rep = P.gmres_solve(p, net, b, x, x0_zero=True, **kw)
    torch.cuda.synchronize()
    return x.cpu().numpy(), [(r["iterations"], r["converged"], r["relres_true"]) for r in rep]


@pytest.mark.parametrize("sequence", [
    [(8, 0), (4, 0)],              # shorter restart on a batched problem (per-sample strides)
    [(30, 0), (8, 1), (30, 1)],    # fp64 basis sized by an earlier, shorter call
    [(4, 1), (16, 0), (4, 0)],
])
def test_workspace_follows_restart_and_precision(sequence):
    P, p, net, b = _setup()
    for restart, precision in sequence:
        kw = dict(restart=restart, maxit=40, rtol=1e-30, precision=precision)
        x, rep = _solve(P, p, net, b, **kw)
        Pf, pf, netf, bf = _setup()          # fresh problem: fresh workspace
        xf, repf = _solve(Pf, pf, netf, bf, **kw)
        assert rep == repf, (restart, precision)
        assert np.array_equal(x, xf), (restart, precision)


def test_one_restart_range():
    P, p, net, b = _setup()
    x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
    for bad in (0, 33, 64):
        with pytest.raises(P.RteError):
            P.gmres_prepare(p, net, restart=bad)
        with pytest.raises(P.RteError):
            P.gmres_solve(p, net, b, x, restart=bad, maxit=4)
        with pytest.raises(P.RteError):
            P.gmres_solve_host(p, net, b.cpu(), x.cpu(), restart=bad, maxit=4)
    P.gmres_prepare(p, net, restart=32)
    rep = P.gmres_solve(p, net, b, x, restart=32, maxit=40, rtol=1e-30, x0_zero=True)
    assert all(r["iterations"] == 40 for r in rep)


def test_nan_rhs_stops_with_breakdown_2():
    """A NaN in one sample's rhs: that sample stops at its first step with breakdown = 2 and the call
    reports RTE_ENUMERIC; the other samples run their full budget unchanged."""
    import paper_2604_23265_b200 as P
    P_, p, net, b = _setup()
    _, rep_ok = _solve(P_, p, net, b, restart=8, maxit=20, rtol=1e-30)
    b2 = b.clone()
    b2[1, 3, 5, 2] = float("nan")
    x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
    with pytest.raises(P.RteError) as ei:
        P.gmres_solve(p, net, b2, x, restart=8, maxit=20, rtol=1e-30, x0_zero=True)
    assert ei.value.status == 5 and "non-finite" in str(ei.value)
    reps = ei.value.reports
    assert reps[1]["breakdown"] == 2 and not reps[1]["converged"]
    assert reps[1]["iterations"] <= 1
    for s in (0, 2):
        assert reps[s]["breakdown"] == 0 and reps[s]["iterations"] == 20
        assert reps[s]["relres_true"] == rep_ok[s][2]
    xs = x.cpu().numpy()
    assert np.isfinite(xs[0]).all() and np.isfinite(xs[2]).all()


def test_nan_in_preconditioner_stops_every_sample():
    """A NaN weight makes every V-cycle output NaN: all samples stop with breakdown = 2 at the first
    step instead of iterating to maxit on NaN."""
    import paper_2604_23265_b200 as P
    w = W.make_weights(CFG, std=0.05)
    w[len(w) // 2] = np.nan
    _, p, net, b = _setup(weights=w)
    x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
    with pytest.raises(P.RteError) as ei:
        P.gmres_solve(p, net, b, x, restart=8, maxit=50, rtol=1e-30, x0_zero=True)
    assert all(r["breakdown"] == 2 and r["iterations"] <= 1 for r in ei.value.reports)
