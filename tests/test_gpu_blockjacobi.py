"""GPU parity of NEXT-2 (the paper's workload and the block-Jacobi preconditioner; PAPER.md:516-533;
DESIGN.md R34-R35) against the fp64 oracle, through the C ABI."""
import numpy as np
import pytest

import workloads as W
from oracle import rte as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _pair(med, N, n_polar=1, n_azim=4, g=0.0):
    import paper_2604_23265_b200 as P
    B = med.sigma_T.shape[0]
    gg = np.full(B, g, np.float32)
    p = P.rte_setup(N, med.sigma_T, med.sigma_a, med.q, med.eps, gg, med.inflow, n_polar=n_polar, n_azim=n_azim)
    op = O.setup(N, n_polar, n_azim, med.sigma_T, med.sigma_a, med.q, med.eps, gg, med.inflow)
    return P, p, op


@pytest.mark.parametrize("regime,N,n_polar,n_azim,g", [("diffusion", 32, 1, 4, 0.0), ("centre", 32, 1, 4, 0.0),
                                                       ("transport", 13, 2, 8, 0.5), ("lr", 8, 2, 16, 0.8)])
def test_block_jacobi_apply_parity(regime, N, n_polar, n_azim, g, margin):
    M = n_polar * n_azim
    med = W.paper_media(3, N=N, degree=3, regime=regime, M=M, seed=11)
    P, p, op = _pair(med, N, n_polar, n_azim, g)
    r = np.random.default_rng(1).standard_normal(op.shape)
    ref = O.block_jacobi(op)(r)
    r64 = torch.from_numpy(r).cuda()
    z64 = torch.empty_like(r64)
    P.rte_blockjacobi_apply(p, r64, z64)
    r32 = r64.float()
    z32 = torch.empty_like(r32)
    P.rte_blockjacobi_apply(p, r32, z32)
    torch.cuda.synchronize()
    assert margin(_rel(z64.cpu().numpy(), ref), 1e-12, "fp64 block-Jacobi rel-L2") <= 1e-12
    assert margin(_rel(z32.cpu().numpy(), ref), 1e-5, "fp32 block-Jacobi rel-L2") <= 1e-5


@pytest.mark.parametrize("regime,precision", [("transport", 1), ("centre", 1), ("diffusion", 1), ("diffusion", 0),
                                              ("transport", 0), ("centre", 0)])
def test_gmres_block_jacobi_iteration_parity(regime, precision, margin):
    """Paper workload (32 x 32, 4 directions): block-Jacobi GMRES reaches rtol in the
    oracle's iteration count +-1 with x to 1e-4, with the fp64 Krylov basis (precision 1) and in the
    fp32-basis mode scripts/paper_workload.py measures (precision 0), including the diffusion regime
    the paper's >= 10x claim is about."""
    N = 32
    med = W.paper_media(2, N=N, degree=2, regime=regime, M=4, seed=12)
    P, p, op = _pair(med, N)
    b = W.make_paper_rhs(2, N=N, M=4, seed=3)
    bd = torch.from_numpy(b).cuda()
    x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
    rep = P.gmres_solve(p, None, bd, x, restart=30, maxit=2000, rtol=1e-8, precond=2, precision=precision)
    torch.cuda.synchronize()
    Pbj = O.block_jacobi(op)
    for s in range(2):
        sub = O.setup(N, 1, 4, med.sigma_T[s:s + 1], med.sigma_a[s:s + 1], med.q[s:s + 1], med.eps[s:s + 1],
                      np.zeros(1), med.inflow[s:s + 1])
        ref = O.gmres(lambda v: O.apply(sub, v), b[s:s + 1].astype(np.float64), O.block_jacobi(sub), restart=30,
                      rtol=1e-8, maxit=2000)
        assert ref.converged and rep[s]["converged"]
        assert margin(abs(rep[s]["iterations"] - ref.iterations), 1, f"iterations[{s}] vs oracle") <= 1, \
            (rep[s]["iterations"], ref.iterations)
        assert margin(_rel(x[s].cpu().numpy(), ref.x[0]), 1e-4, f"x[{s}] rel-L2") <= 1e-4
    assert Pbj is not None


def test_gmres_block_jacobi_one_cell_is_exact():
    """One cell: P = A^{-1}, so GMRES in fp64 (precision=1) converges in one iteration (in the fp32
    mode the fp32-rounded blocks take a few more, measured 3 to 4e-10)."""
    med = W.paper_media(2, N=1, degree=2, regime="diffusion", M=8, seed=13)
    P, p, op = _pair(med, 1, 2, 4, 0.3)
    bd = torch.from_numpy(W.make_paper_rhs(2, N=1, M=8, seed=4)).cuda()
    x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
    rep = P.gmres_solve(p, None, bd, x, restart=30, maxit=10, rtol=1e-10, precond=2, precision=1)
    assert all(r["converged"] and r["iterations"] == 1 for r in rep)


def test_block_jacobi_rejects_oversized_problem():
    import paper_2604_23265_b200 as P
    cfg = W.config(5)
    media = W.make_media(cfg)
    p = P.rte_setup(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                    n_polar=cfg.n_polar, n_azim=cfg.n_azim)
    r = torch.zeros(p.shape, dtype=torch.float32, device="cuda")
    with pytest.raises(P.RteError):
        P.rte_blockjacobi_apply(p, r, torch.empty_like(r))
