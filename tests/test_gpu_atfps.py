"""GPU parity of the ATFPS compressed system (NEXT-3b; include/rte.h rte_setup_atfps)
against the fp64 oracle (oracle/atfps.py), through the C ABI.

Tolerances: kept mask and dimension exact; fp32 apply / rhs / layer reconstruction rel-L2 <= 1e-5; fp64
<= 1e-8 (the interface bases come from different QR / inversion algorithms on the two sides); the
first Arnoldi columns of the compressed system to 1e-5; and a GPU-only closed form: a global slow mode
of a homogeneous medium is reproduced exactly by the compressed solve plus layer reconstruction.
"""
import numpy as np
import pytest

import workloads as W
from oracle import atfps as A
from oracle import rte as O
from oracle import tfps as T

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _small_media(N=6, M=8, eps=0.02, seed=3):
    rng = np.random.default_rng(seed)
    sT = np.where(rng.random((1, N, N)) < 0.5, 1.0, 6.0).astype(np.float32)
    f = lambda v: np.full((1, N, N), v, np.float32)
    return W.Media(sigma_T=sT, sigma_a=f(0.3), q=f(1.0), eps=f(eps), g=np.array([0.5], np.float32),
                   inflow=rng.uniform(0.5, 1.5, (1, 4, N, M)).astype(np.float32))


def _pair(N, n_polar, n_azim, med, delta):
    import paper_2604_23265_b200 as P
    p = P.rte_setup_atfps(N, med.sigma_T, med.sigma_a, med.q, med.eps, med.g, med.inflow, delta=delta,
                          n_polar=n_polar, n_azim=n_azim)
    tp = T.setup(N, n_polar, n_azim, med.sigma_T, med.sigma_a, med.q, med.eps, med.g, med.inflow)
    return P, p, A.setup(tp, delta)


CASES = [(6, 1, 8, None, 1e-1), (6, 1, 8, None, 1e-2), (6, 1, 8, None, 1e-300)]


@pytest.mark.parametrize("N,npol,naz,cfgk,delta", CASES + [pytest.param(64, 2, 16, 2, 1e-4, marks=pytest.mark.slow)],
                         ids=["small-1e-1", "small-1e-2", "small-full", "cfg2-1e-4"])
def test_atfps_apply_rhs_reconstruct(N, npol, naz, cfgk, delta, margin):
    med = W.make_media(W.config(cfgk)) if cfgk else _small_media(N, npol * naz)
    P, p, at = _pair(N, npol, naz, med, delta)
    d, dim, sel = P.rte_atfps_info(p)
    assert d == delta and dim == A.dimension(at) and np.array_equal(sel, at.sel)
    rng = np.random.default_rng(N)
    a = rng.standard_normal(at.shape)
    a32 = a.astype(np.float32)
    y = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    P.rte_apply(p, torch.from_numpy(a32).cuda(), y)
    y64 = torch.empty(p.shape, dtype=torch.float64, device="cuda")
    P.rte_apply_f64(p, torch.from_numpy(a).cuda(), y64)
    b = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    P.rte_rhs(p, b)
    Md = npol * naz
    psi = torch.empty(1, N, N, Md, dtype=torch.float32, device="cuda")
    full = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    P.rte_atfps_reconstruct(p, torch.from_numpy(a32).cuda(), psi, full)
    psi64 = torch.empty(1, N, N, Md, dtype=torch.float64, device="cuda")
    P.rte_atfps_reconstruct_f64(p, torch.from_numpy(a).cuda(), psi64)
    torch.cuda.synchronize()
    assert margin(_rel(y.cpu().numpy(), A.apply(at, a32.astype(np.float64))), 1e-5, "apply fp32") <= 1e-5
    assert margin(_rel(y64.cpu().numpy(), A.apply(at, a)), 1e-8, "apply fp64") <= 1e-8
    assert margin(_rel(b.cpu().numpy(), A.rhs(at)), 1e-5, "rhs") <= 1e-5
    psi_ref, full_ref = A.reconstruct(at, a32.astype(np.float64))
    assert margin(_rel(full.cpu().numpy(), full_ref), 1e-5, "layer coefficients") <= 1e-5
    assert margin(_rel(psi.cpu().numpy(), psi_ref), 1e-5, "psi_delta") <= 1e-5
    assert margin(_rel(psi64.cpu().numpy(), A.reconstruct(at, a)[0]), 1e-8, "psi_delta fp64") <= 1e-8


@pytest.mark.parametrize("precision", [0, 1])
def test_atfps_arnoldi_columns(precision, margin):
    """The first Arnoldi columns (unrotated H) of GMRES on the compressed system equal the oracle's."""
    import paper_2604_23265_b200 as P
    N = 6
    P, p, at = _pair(N, 1, 8, _small_media(N, 8), 1e-2)
    b = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    P.rte_rhs(p, b)
    x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
    steps = 6
    rep = P.gmres_solve(p, None, b, x, restart=30, maxit=steps, rtol=1e-30, hessenberg=True, precond=0,
                        precision=precision)[0]
    H = rep["hessenberg"][:steps + 1, :steps]
    Href = O.arnoldi_columns(lambda v: A.apply(at, v), b.cpu().numpy().astype(np.float64), None, steps)
    for j in range(steps):
        assert margin(_rel(H[:j + 2, j], Href[:j + 2, j]), 1e-5, f"H column {j}") <= 1e-5, j


def test_atfps_gpu_reproduces_a_global_slow_mode(margin):
    """Closed form on the GPU alone: psi = q/sigma_a + l exp(sigma_t xi x) for the slowest x-mode of a
    homogeneous diffusive medium; at delta = 1e-2 (a compressed system) the GPU solve plus layer
    reconstruction returns psi at the cell centres (fp64 basis; the rhs is fp32, hence 1e-5)."""
    import paper_2604_23265_b200 as P
    N, npol, naz = 4, 1, 8
    M = npol * naz
    sT, sA, eps, g, q = 4.0, 0.3, 0.05, 0.5, 0.7
    f = lambda v: np.full((1, N, N), v, np.float32)
    probe = P.rte_setup_tfps(N, f(sT), f(sA), f(q), f(eps), [g], None, n_polar=npol, n_azim=naz)
    xi, L = P.rte_tfps_info(probe)
    ks = np.arange(M)
    k = int(ks[np.argmin(np.abs(xi[0][ks]) + 1e9 * (xi[0][ks] > 0))])
    st = float(np.float32(sT)) / float(np.float32(eps))
    C = float(np.float32(q)) / float(np.float32(sA))
    psi_fn = lambda x, y: C + L[0][:, k] * np.exp(st * xi[0][k] * x)
    h = 1.0 / N
    inf = np.zeros((1, 4, N, M))
    for t in range(N):
        c = (t + 0.5) * h
        inf[0, 0, t], inf[0, 1, t], inf[0, 2, t], inf[0, 3, t] = psi_fn(0, c), psi_fn(1, c), psi_fn(c, 0), psi_fn(c, 1)
    p = P.rte_setup_atfps(N, f(sT), f(sA), f(q), f(eps), [g], inf, delta=1e-2, n_polar=npol, n_azim=naz)
    _, dim, sel = P.rte_atfps_info(p)
    assert sel[0][k] and dim < p.n
    b = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    P.rte_rhs(p, b)
    x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
    rep = P.gmres_solve(p, None, b, x, restart=32, maxit=3000, rtol=1e-10, precision=1, precond=0)[0]
    assert rep["converged"]
    psi = torch.empty(1, N, N, M, dtype=torch.float64, device="cuda")
    P.rte_atfps_reconstruct_f64(p, x, psi)
    torch.cuda.synchronize()
    expect = np.stack([[psi_fn((i + 0.5) * h, (j + 0.5) * h) for i in range(N)] for j in range(N)])[None]
    assert margin(_rel(psi.cpu().numpy(), expect), 1e-5, "psi_delta vs closed form") <= 1e-5
