"""GPU parity of the TFPS alpha-space operator (NEXT-3; include/rte.h rte_setup_tfps)
against the fp64 oracle (oracle/tfps.py), through the C ABI.

Tolerances: fp32 apply rel-L2 <= 1e-5 (the north star's per-operator bound), fp64 apply <= 1e-8 (the
two sides solve the local eigenproblems with different algorithms -- numpy's nonsymmetric eig vs the
library's symmetrised Cholesky + Jacobi -- so the bases agree to 1e-13 at M = 8 and to ~1e-10 at
M = 64, not bit-for-bit), rhs <= 1e-7, reconstruction as the apply.  GMRES on the alpha system: the
first Arnoldi columns to 1e-5 on the two-material config-2 shape (plain and MgNet-preconditioned); a
full solve where restarted GMRES must converge (n = restart = 32: GMRES(32) is exact in <= n steps --
the unpreconditioned TFPS system stagnates restarted GMRES, also in the oracle): fp64 basis +-1 and
alpha to 1e-6; and a GPU-only closed form: a global eigenmode of a homogeneous medium is reproduced
exactly (oracle-independent; tests/test_oracle_tfps.py has the same pin for the oracle).
"""
import numpy as np
import pytest

import workloads as W
from oracle import rte as O
from oracle import tfps as T

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _pair(cfg, media=None):
    import paper_2604_23265_b200 as P
    media = media or W.make_media(cfg)
    p = P.rte_setup_tfps(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                         n_polar=cfg.n_polar, n_azim=cfg.n_azim)
    tp = T.setup_from_media(cfg, media)
    return P, p, tp


CASES = [
    W.config(2),                                                   # two materials, 64^2 x 32 directions
    W.small_config(2, N=5, M=8, n_polar=1, n_azim=8),              # ragged, tiny
    W.small_config(2, N=12, M=16, n_polar=2, n_azim=8, B=2),       # batch (per-sample S)
    W.small_config(2, N=8, M=64, n_polar=4, n_azim=16),            # M = 64: 128 unknowns per cell
]


@pytest.mark.parametrize("cfg", CASES, ids=lambda c: f"N{c.N}-M{c.M}-B{c.B}")
def test_tfps_setup_apply_rhs_reconstruct(cfg, margin):
    P, p, tp = _pair(cfg)
    assert p.M == 2 * cfg.M and p.shape == tp.shape
    xi, L = P.rte_tfps_info(p)
    assert xi.shape[0] == len(tp.modes)
    xo, Lo = T.material_tables(tp)
    assert margin(np.max(np.abs(xi - xo) / np.abs(xo)), 1e-8, "xi") <= 1e-8
    assert margin(np.max(np.abs(L - Lo)), 1e-6, "eigenvectors") <= 1e-6
    rng = np.random.default_rng(cfg.N)
    a = rng.standard_normal(tp.shape)
    a32 = a.astype(np.float32)
    y = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    P.rte_apply(p, torch.from_numpy(a32).cuda(), y)
    y64 = torch.empty(p.shape, dtype=torch.float64, device="cuda")
    P.rte_apply_f64(p, torch.from_numpy(a).cuda(), y64)
    b = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    P.rte_rhs(p, b)
    psi = torch.empty(tp.B, tp.N, tp.N, tp.M, dtype=torch.float32, device="cuda")
    P.rte_tfps_reconstruct(p, torch.from_numpy(a32).cuda(), psi)
    psi64 = torch.empty(tp.B, tp.N, tp.N, tp.M, dtype=torch.float64, device="cuda")
    P.rte_tfps_reconstruct_f64(p, torch.from_numpy(a).cuda(), psi64)
    torch.cuda.synchronize()
    assert margin(_rel(y.cpu().numpy(), T.apply(tp, a32.astype(np.float64))), 1e-5, "apply fp32") <= 1e-5
    assert margin(_rel(y64.cpu().numpy(), T.apply(tp, a)), 1e-8, "apply fp64") <= 1e-8
    assert margin(_rel(b.cpu().numpy(), T.rhs(tp)), 1e-7, "rhs") <= 1e-7
    assert margin(_rel(psi.cpu().numpy(), T.reconstruct(tp, a32.astype(np.float64))), 1e-5, "reconstruct") <= 1e-5
    assert margin(_rel(psi64.cpu().numpy(), T.reconstruct(tp, a)), 1e-8, "reconstruct fp64") <= 1e-8


def test_tfps_rejects_zero_absorption():
    import paper_2604_23265_b200 as P
    N = 4
    z = np.zeros((1, N, N), np.float32)
    with pytest.raises(P.RteError):
        P.rte_setup_tfps(N, z + 1.0, z, z + 1.0, z + 1.0, [0.5], None, n_polar=1, n_azim=8)


@pytest.mark.parametrize("precision", [1, 0])
def test_tfps_gmres_matches_oracle(precision, margin):
    """A system GMRES(32) solves exactly (n = 2 x 2 cells x 8 = 32 unknowns, two materials): fp64 basis
    -> iteration count +-1 and alpha to 1e-6; fp32 basis -> alpha to 1e-4."""
    import paper_2604_23265_b200 as P
    N = 2
    sT = np.array([[[1.0, 10.0], [10.0, 1.0]]], np.float32)
    f = lambda v: np.full((1, N, N), v, np.float32)
    media = W.Media(sigma_T=sT, sigma_a=f(0.1), q=f(1.0), eps=f(0.05), g=np.array([0.5], np.float32),
                    inflow=np.ones((1, 4, N, 4), np.float32))
    cfg = W.small_config(2, N=N, M=4, n_polar=1, n_azim=4)
    P, p, tp = _pair(cfg, media)
    assert len(tp.modes) == 2 and p.n == 32
    b = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    P.rte_rhs(p, b)
    b32 = b.cpu().numpy().astype(np.float64)
    x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
    rtol = 1e-10 if precision else 1e-6
    rep = P.gmres_solve(p, None, b, x, restart=32, maxit=200, rtol=rtol, precision=precision, precond=0)[0]
    ref = O.gmres(lambda v: T.apply(tp, v), b32, restart=32, rtol=rtol, maxit=200)
    assert ref.converged and rep["converged"]
    tol = 1e-6 if precision else 1e-4
    assert margin(_rel(x.cpu().numpy(), ref.x), tol, "alpha rel-L2") <= tol
    if precision:
        assert margin(abs(rep["iterations"] - ref.iterations), 1, "iterations vs oracle") <= 1


@pytest.mark.parametrize("precision", [0, 1])
def test_tfps_arnoldi_columns_config2(precision, margin):
    """Config 2's alpha system (64^2 cells, 32 directions, two materials), unpreconditioned: the first
    Arnoldi columns (unrotated H) equal the oracle's to 1e-5."""
    import paper_2604_23265_b200 as P
    cfg = W.config(2)
    P, p, tp = _pair(cfg)
    b = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    P.rte_rhs(p, b)
    x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
    steps = 6
    rep = P.gmres_solve(p, None, b, x, restart=30, maxit=steps, rtol=1e-30, hessenberg=True, precond=0,
                        precision=precision)[0]
    H = rep["hessenberg"][:steps + 1, :steps]
    Href = O.arnoldi_columns(lambda v: T.apply(tp, v), b.cpu().numpy().astype(np.float64), None, steps)
    for j in range(steps):
        assert margin(_rel(H[:j + 2, j], Href[:j + 2, j]), 1e-5, f"H column {j}") <= 1e-5, j


def test_tfps_mgnet_arnoldi_columns(margin):
    """MgNet on the alpha system (lift from 2 Md channels): the first Arnoldi columns of the
    right-preconditioned process equal the oracle's (TFPS apply + MgNet V-cycle) to 1e-5."""
    import paper_2604_23265_b200 as P
    cfg = W.small_config(2, N=16, M=16, n_polar=2, n_azim=8, L=3, C0=16)
    P, p, tp = _pair(cfg)
    w = W.make_weights(W.small_config(2, N=16, M=2 * cfg.M, n_polar=2, n_azim=16, L=3, C0=16), std=0.05)
    net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, w)
    onet = O.make_mgnet(w, 2 * cfg.M, cfg.L, cfg.C0, cfg.nu)
    b = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    P.rte_rhs(p, b)
    x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
    steps = 4
    rep = P.gmres_solve(p, net, b, x, restart=30, maxit=steps, rtol=1e-30, hessenberg=True)[0]
    H = rep["hessenberg"][:steps + 1, :steps]
    Href = O.arnoldi_columns(lambda v: T.apply(tp, v), b.cpu().numpy().astype(np.float64),
                             lambda v: O.vcycle(onet, v), steps)
    for j in range(steps):
        assert margin(_rel(H[:j + 2, j], Href[:j + 2, j]), 1e-5, f"H column {j}") <= 1e-5, j


def test_tfps_gpu_reproduces_a_global_mode_exactly(margin):
    """Closed form on the GPU alone: a homogeneous medium with inflow and source taken from
    psi = q/sigma_a + l exp(sigma_t xi x) (an exact RTE solution) -- the GPU solve (fp64 basis) returns
    alpha = exp(sigma_t xi x_ref) for that mode in every cell and 0 elsewhere."""
    import paper_2604_23265_b200 as P
    N, npol, naz = 2, 1, 4                                     # n = 32: GMRES(32) is exact
    M = npol * naz
    sT, sA, eps, g, q = 2.0, 0.3, 0.5, 0.4, 0.7
    f = lambda v: np.full((1, N, N), v, np.float32)
    probe = P.rte_setup_tfps(N, f(sT), f(sA), f(q), f(eps), [g], None, n_polar=npol, n_azim=naz)
    xi, L = P.rte_tfps_info(probe)
    k = 1                                                      # an x-mode decaying to the right
    st = float(np.float32(sT)) / float(np.float32(eps))
    h = 1.0 / N
    C = float(np.float32(q)) / float(np.float32(sA))
    psi_fn = lambda x, y: C + L[0][:, k] * np.exp(st * xi[0][k] * x)
    inf = np.zeros((1, 4, N, M))
    for t in range(N):
        c = (t + 0.5) * h
        inf[0, 0, t], inf[0, 1, t], inf[0, 2, t], inf[0, 3, t] = psi_fn(0, c), psi_fn(1, c), psi_fn(c, 0), psi_fn(c, 1)
    p = P.rte_setup_tfps(N, f(sT), f(sA), f(q), f(eps), [g], inf, n_polar=npol, n_azim=naz)
    b = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    P.rte_rhs(p, b)
    x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
    rep = P.gmres_solve(p, None, b, x, restart=32, maxit=200, rtol=1e-10, precision=1, precond=0)[0]
    assert rep["converged"]
    expect = np.zeros(p.shape)
    for i in range(N):
        ref = i * h if xi[0][k] < 0 else (i + 1) * h
        expect[0, :, i, k] = np.exp(st * xi[0][k] * ref)
    # the rhs is fp32 (the inflow rows are rounded), so the solve is exact to fp32 data accuracy
    assert margin(_rel(x.cpu().numpy(), expect), 1e-5, "alpha vs closed form") <= 1e-5
