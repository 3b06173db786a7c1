"""The per-Arnoldi-step CUDA graphs of gmres_solve: replaying them is bitwise identical
to launching the kernels, and they are invalidated when the preconditioner changes."""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _setup(cfg):
    import paper_2604_23265_b200 as P
    media = W.make_media(cfg)
    p = P.rte_setup(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                    n_polar=cfg.n_polar, n_azim=cfg.n_azim)
    net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, W.make_weights(cfg, std=0.05))
    b = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    P.rte_rhs(p, b)
    return P, p, net, b, media


def _solve(P, p, net, b, maxit, precond=None):
    x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
    rep = P.gmres_solve(p, net, b, x, restart=8, maxit=maxit, rtol=1e-30, precond=precond, hessenberg=True)
    torch.cuda.synchronize()
    return x.cpu().numpy(), rep


@pytest.mark.parametrize("precond", [1, 0])
def test_graph_replay_is_bitwise_identical(precond):
    """Solve 1 runs every step eagerly (first sight), solve 2 captures and replays, solve 3 replays;
    prepared graphs replay too: all four agree bit for bit (2 restart cycles of 8 steps each)."""
    cfg = W.small_config(5, N=32, M=32, n_polar=2, n_azim=16, L=3, C0=32)
    P, p, net, b, _ = _setup(cfg)
    launches = []
    xs = []
    for _ in range(3):
        P.rte_launch_count(reset=True)
        x, _ = _solve(P, p, net, b, 16, precond)
        launches.append(P.rte_launch_count(reset=True))
        xs.append(x)
    P2, p2, net2, b2, _ = _setup(cfg)
    P2.gmres_prepare(p2, net2, restart=8, precond=precond)
    x4, _ = _solve(P2, p2, net2, b2, 16, precond)
    assert np.array_equal(xs[0], xs[1]) and np.array_equal(xs[0], xs[2]) and np.array_equal(xs[0], x4)
    assert launches[0] == launches[1] == launches[2]  # replayed kernels are counted as launches


def test_graphs_follow_coeffnet_changes():
    """Attaching CoeffNet maps after graphs were captured changes the preconditioner: the solve must
    match a fresh modulated net, not the stale graphs."""
    cfg = W.small_config(5, N=32, M=32, n_polar=2, n_azim=16, L=3, C0=32)
    P, p, net, b, media = _setup(cfg)
    for _ in range(3):
        x_plain, _ = _solve(P, p, net, b, 8)
    cw = W.make_coeffnet_weights(cfg, head_std=0.2)
    P.mgnet_coeffnet(net, media.sigma_T, media.sigma_a, media.eps, cw)
    x_mod, _ = _solve(P, p, net, b, 8)
    x_mod2, _ = _solve(P, p, net, b, 8)
    fresh = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, W.make_weights(cfg, std=0.05))
    P.mgnet_coeffnet(fresh, media.sigma_T, media.sigma_a, media.eps, cw)
    x_fresh, _ = _solve(P, p, fresh, b, 8)
    assert not np.array_equal(x_plain, x_mod)
    assert np.array_equal(x_mod, x_fresh) and np.array_equal(x_mod, x_mod2)
