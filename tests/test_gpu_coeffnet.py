"""GPU parity of NEXT-1 (CoeffNet + modulated MgNet smoother; R31-R33)
against the fp64 oracle, through the C ABI (mgnet_coeffnet, mgnet_modulation, mgnet_vcycle[_f64],
gmres_solve).  Tolerances as for the unmodulated V-cycle: fp32 V-cycle rel-L2 <= 1e-5,
fp64 data flow <= 1e-12, Arnoldi columns <= 1e-5."""
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


CFGS = [
    W.small_config(1, N=8, M=16, L=2, C0=4),                                   # SIMT levels
    W.small_config(2, N=24, M=8, n_polar=1, n_azim=8, L=3, C0=8, B=2),         # batch of 2
    W.small_config(5, N=32, M=32, n_polar=2, n_azim=16, L=3, C0=32),           # tensor-core levels
    W.config(2),
]


def _setup(cfg, head_std=0.2, std=0.05):
    import paper_2604_23265_b200 as P
    media = W.make_media(cfg)
    p = P.rte_setup(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                    n_polar=cfg.n_polar, n_azim=cfg.n_azim)
    w = W.make_weights(cfg, std=std)
    cw = W.make_coeffnet_weights(cfg, head_std=head_std)
    net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, w)
    P.mgnet_coeffnet(net, media.sigma_T, media.sigma_a, media.eps, cw)
    onet = O.make_mgnet(w, cfg.M, cfg.L, cfg.C0, cfg.nu)
    mod = O.coeffnet(media.sigma_T, media.sigma_a, media.eps, cw, cfg.L, cfg.C0)
    return P, p, net, onet, mod, media


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: f"cfg{c.k}-N{c.N}-L{c.L}-C{c.C0}-B{c.B}")
def test_coeffnet_maps_parity(cfg, margin):
    P, p, net, onet, mod, _ = _setup(cfg)
    for l in range(cfg.L):
        assert margin(_rel(P.mgnet_modulation(net, l, 0), mod["a"][l]), 1e-12, f"map a level {l}") <= 1e-12, l
        assert margin(_rel(P.mgnet_modulation(net, l, 1), mod["abar"][l]), 1e-12, f"map abar level {l}") <= 1e-12, l


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: f"cfg{c.k}-N{c.N}-L{c.L}-C{c.C0}-B{c.B}")
def test_modulated_vcycle_parity(cfg, margin):
    P, p, net, onet, mod, _ = _setup(cfg)
    r = W.make_vector(cfg, 2)
    rd = torch.from_numpy(r).cuda()
    z = torch.empty_like(rd)
    P.mgnet_vcycle(net, rd, z, add_identity=True)
    z64 = torch.empty(rd.shape, dtype=torch.float64, device="cuda")
    P.mgnet_vcycle_f64(net, rd.double(), z64, add_identity=False)
    torch.cuda.synchronize()
    ref = O.vcycle(onet, r, add_identity=False, mod=mod)
    assert margin(_rel(z.cpu().numpy().astype(np.float64) - r, ref), 1e-5, "modulated V(r) rel-L2") <= 1e-5
    assert margin(_rel(z64.cpu().numpy(), ref), 1e-12, "fp64 rel-L2") <= 1e-12


def test_removing_maps_restores_the_plain_vcycle():
    cfg = CFGS[2]
    P, p, net, onet, mod, media = _setup(cfg)
    r = torch.from_numpy(W.make_vector(cfg, 1)).cuda()
    zm, z0, z1 = torch.empty_like(r), torch.empty_like(r), torch.empty_like(r)
    P.mgnet_vcycle(net, r, zm)
    P.mgnet_coeffnet(net, None, None, None, None)
    P.mgnet_vcycle(net, r, z0)
    plain = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, W.make_weights(cfg, std=0.05))
    P.mgnet_vcycle(plain, r, z1)
    torch.cuda.synchronize()
    assert torch.equal(z0, z1) and not torch.equal(zm, z0)
    with pytest.raises(P.RteError):
        P.mgnet_modulation(net, 0, 0)


def test_coeffnet_rejects_weight_count_mismatch():
    cfg = CFGS[0]
    P, p, net, onet, mod, media = _setup(cfg)
    with pytest.raises(P.RteError):
        P.mgnet_coeffnet(net, media.sigma_T, media.sigma_a, media.eps, W.make_coeffnet_weights(cfg)[:-1])


@pytest.mark.parametrize("k,steps", [(2, 8), (3, 5)])
def test_gmres_arnoldi_columns_with_coeffnet(k, steps, margin):
    """The modulated preconditioner in GMRES: first Arnoldi columns agree with the oracle's."""
    cfg = W.config(k)
    P, p, net, onet, mod, media = _setup(cfg, head_std=0.02, std=0.02)
    op = O.setup_from_media(cfg, media)
    bd = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    P.rte_rhs(p, bd)
    x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
    rep = P.gmres_solve(p, net, bd, x, restart=cfg.restart, maxit=steps, rtol=1e-30, hessenberg=True)
    H = rep[0]["hessenberg"][:steps + 1, :steps]
    Href = O.arnoldi_columns(lambda v: O.apply(op, v), bd.cpu().numpy().astype(np.float64),
                             lambda v: O.vcycle(onet, v, mod=mod), steps)
    for j in range(steps):
        assert margin(_rel(H[:j + 2, j], Href[:j + 2, j]), 1e-5, f"H column {j}") <= 1e-5, j
