"""GPU parity of the filtered loss (NEXT-4; include/rte.h rte_atfps_fit / rte_atfps_loss; PAPER.md:492-507
eq:loss_delta; readings R43-R45) against the fp64 oracle (oracle/loss.py), through the C ABI.

Tolerances: D_delta rel-L2 1e-9 and the loss rel 1e-10 in fp64 (the fit operators come from different
least-squares algorithms on the two sides: an eigen-decomposition of G^T G here -- error ~ cond(G)^2 eps --
numpy's SVD there), D_delta 1e-5 and the loss 1e-4 in fp32 (the residual cancels); the
gradient with respect to psi_d rel-L2 1e-9 (fp64) / 1e-4 (fp32: a difference of two loss-sized
contractions); a GPU-only closed form: the constant exact solution has loss 0.
"""
import numpy as np
import pytest

import workloads as W
from oracle import atfps as A
from oracle import loss as Lo
from oracle import tfps as T

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _media(N=6, M=8, eps=0.02, seed=3, B=1):
    rng = np.random.default_rng(seed)
    sT = np.where(rng.random((B, N, N)) < 0.5, 1.0, 6.0).astype(np.float32)
    f = lambda v: np.full((B, N, N), v, np.float32)
    return W.Media(sigma_T=sT, sigma_a=f(0.3), q=rng.uniform(0.0, 1.0, (B, N, N)).astype(np.float32), eps=f(eps),
                   g=np.full(B, 0.5, np.float32), inflow=rng.uniform(0.5, 1.5, (B, 4, N, M)).astype(np.float32))


def _pair(N, npol, naz, med, delta):
    import paper_2604_23265_b200 as P
    p = P.rte_setup_atfps(N, med.sigma_T, med.sigma_a, med.q, med.eps, med.g, med.inflow, delta=delta,
                          n_polar=npol, n_azim=naz)
    tp = T.setup(N, npol, naz, med.sigma_T, med.sigma_a, med.q, med.eps, med.g, med.inflow)
    return P, p, A.setup(tp, delta)


@pytest.mark.parametrize("N,npol,naz,B,delta", [(6, 1, 8, 1, 1e-2), (5, 1, 4, 2, 1e-3), (7, 2, 8, 1, 1e-1)],
                         ids=["N6-M8", "N5-M4-B2", "N7-M16"])
def test_fit_and_loss_parity(N, npol, naz, B, delta, margin):
    med = _media(N, npol * naz, B=B)
    P, p, at = _pair(N, npol, naz, med, delta)
    rng = np.random.default_rng(N)
    psi = rng.uniform(0.0, 2.0, (B, N, N, npol * naz))
    a_ref = Lo.D(at, psi)
    l_ref = Lo.loss(at, psi)
    a64 = torch.empty(p.shape, dtype=torch.float64, device="cuda")
    P.rte_atfps_fit_f64(p, torch.from_numpy(psi).cuda(), a64)
    a32 = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    P.rte_atfps_fit(p, torch.from_numpy(psi.astype(np.float32)).cuda(), a32)
    l64 = P.rte_atfps_loss_f64(p, torch.from_numpy(psi).cuda())
    l32 = P.rte_atfps_loss(p, torch.from_numpy(psi.astype(np.float32)).cuda())
    torch.cuda.synchronize()
    assert margin(_rel(a64.cpu().numpy(), a_ref), 1e-9, "D_delta fp64 rel-L2") <= 1e-9
    assert margin(_rel(a32.cpu().numpy(), a_ref), 1e-5, "D_delta fp32 rel-L2") <= 1e-5
    assert margin(float(np.max(np.abs(l64 - l_ref) / l_ref)), 1e-10, "loss fp64 rel") <= 1e-10
    # (fp32: the residual b_bar - A_bar alpha cancels; its relative error is eps_32 ||b_bar|| / ||r|| ~ 1e-5)
    assert margin(float(np.max(np.abs(l32 - l_ref) / l_ref)), 1e-4, "loss fp32 rel") <= 1e-4


@pytest.mark.parametrize("N,npol,naz,B,delta", [(4, 1, 4, 1, 1e-3), (3, 1, 8, 2, 1e-2)], ids=["N4-M4", "N3-M8-B2"])
def test_gradient_parity(N, npol, naz, B, delta, margin):
    med = _media(N, npol * naz, B=B)
    P, p, at = _pair(N, npol, naz, med, delta)
    rng = np.random.default_rng(7)
    psi = rng.uniform(0.0, 2.0, (B, N, N, npol * naz))
    g_ref = Lo.loss_grad(at, psi)
    g64 = torch.empty(psi.shape, dtype=torch.float64, device="cuda")
    P.rte_atfps_loss_f64(p, torch.from_numpy(psi).cuda(), grad=g64)
    g32 = torch.empty(psi.shape, dtype=torch.float32, device="cuda")
    P.rte_atfps_loss(p, torch.from_numpy(psi.astype(np.float32)).cuda(), grad=g32)
    torch.cuda.synchronize()
    assert margin(_rel(g64.cpu().numpy(), g_ref), 1e-9, "grad fp64 rel-L2") <= 1e-9
    assert margin(_rel(g32.cpu().numpy(), g_ref), 1e-4, "grad fp32 rel-L2") <= 1e-4


def test_constant_exact_solution_has_zero_loss():
    import paper_2604_23265_b200 as P
    N, M, sA, q = 8, 8, 0.25, 0.75   # (exact in fp32: chi^s = q / sigma_a = 3)
    chis = q / sA
    f = lambda v: np.full((1, N, N), v, np.float32)
    p = P.rte_setup_atfps(N, f(4.0), f(sA), f(q), f(0.0625), np.array([0.5], np.float32),
                          np.full((1, 4, N, M), chis, np.float32), delta=1e-2, n_polar=1, n_azim=M)
    psi = torch.full((1, N, N, M), chis, dtype=torch.float64, device="cuda")
    assert P.rte_atfps_loss_f64(p, psi)[0] < 1e-12


def test_loss_rejects_a_psi_space_problem():
    import paper_2604_23265_b200 as P
    cfg = W.small_config(1, N=4, M=8, n_polar=1, n_azim=8)
    med = W.make_media(cfg)
    p = P.rte_setup(cfg.N, med.sigma_T, med.sigma_a, med.q, med.eps, med.g, med.inflow, n_polar=1, n_azim=8)
    psi = torch.zeros(p.shape, dtype=torch.float32, device="cuda")
    with pytest.raises(P.RteError):
        P.rte_atfps_loss(p, psi)
