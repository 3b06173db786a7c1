"""NEXT-4 training harness (paper_2604_23265_b200/train.py; readings R43-R45):
the torch MgNet equals the library's V-cycle on the same packed weights (fp32 1e-5, fp64 1e-12), so trained
weights mean the same network on the benchmarked path; rte_set_source gives the right-hand side of a fresh
setup with that source (bit-identical); the loss_delta autograd function hands torch the library's gradient;
training on one (medium, source) pair lowers loss_delta (SPEC.md's overfit smoke test, scaled down)."""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _media(N=16, M=8, B=2, eps=0.05, seed=5):
    rng = np.random.default_rng(seed)
    sT = np.where(rng.random((B, N, N)) < 0.5, 1.0, 6.0).astype(np.float32)
    f = lambda v: np.full((B, N, N), v, np.float32)
    return W.Media(sigma_T=sT, sigma_a=f(0.3), q=f(1.0), eps=f(eps), g=np.full(B, 0.5, np.float32),
                   inflow=np.zeros((B, 4, N, M), np.float32))


@pytest.mark.parametrize("L,C0,N,M", [(3, 16, 16, 8), (2, 32, 16, 32)], ids=["L3-C16", "L2-C32-tc"])
def test_torch_mgnet_equals_library_vcycle(L, C0, N, M, margin):
    import paper_2604_23265_b200 as P
    from paper_2604_23265_b200 import train as TR
    med = _media(N, M)
    p = P.rte_setup(N, med.sigma_T, med.sigma_a, med.q, med.eps, med.g, med.inflow, n_polar=1, n_azim=M)
    rng = np.random.default_rng(1)
    w = rng.normal(0.0, 0.05, TR.weight_count(M, L, C0, 2)).astype(np.float32)
    net = P.mgnet_create(p, L, C0, 2, w)
    r = torch.from_numpy(rng.standard_normal(p.shape).astype(np.float32)).cuda()
    z = torch.empty_like(r)
    P.mgnet_vcycle(net, r, z, add_identity=True)
    tn = TR.MgNet(M, L, C0, 2, w)
    assert np.array_equal(tn.flat(), w)
    torch.backends.cudnn.allow_tf32 = False  # (torch's fp32 convs default to TF32)
    with torch.no_grad():
        zt = tn(r)
        tn64 = TR.MgNet(M, L, C0, 2, w, dtype=torch.float64)
        z64t = tn64(r.double())
    z64 = torch.empty_like(r, dtype=torch.float64)
    P.mgnet_vcycle_f64(net, r.double(), z64, add_identity=True)
    torch.cuda.synchronize()
    rel = lambda a, b: float((a.double() - b.double()).norm() / (b.double() - r.double()).norm())
    assert margin(rel(zt, z64), 1e-5, "torch fp32 MgNet vs library fp64 V-cycle") <= 1e-5
    assert margin(rel(z, z64), 1e-5, "library fp32 vs fp64 V-cycle") <= 1e-5
    assert margin(rel(z64t, z64), 1e-12, "torch fp64 MgNet vs library fp64 V-cycle") <= 1e-12


@pytest.mark.parametrize("kind", ["psi", "atfps"])
def test_set_source_equals_fresh_setup(kind):
    import paper_2604_23265_b200 as P
    N, M = 8, 8
    med = _media(N, M, B=2)
    rng = np.random.default_rng(2)
    q = rng.uniform(0.0, 1.0, (2, N, N)).astype(np.float32)
    inf = rng.uniform(0.0, 1.0, (2, 4, N, M)).astype(np.float32)
    mk = (lambda qq, ii: P.rte_setup(N, med.sigma_T, med.sigma_a, qq, med.eps, med.g, ii, n_polar=1, n_azim=M)) \
        if kind == "psi" else \
        (lambda qq, ii: P.rte_setup_atfps(N, med.sigma_T, med.sigma_a, qq, med.eps, med.g, ii, delta=1e-2,
                                          n_polar=1, n_azim=M))
    p = mk(med.q, med.inflow)
    P.rte_set_source(p, q, inf)
    ref = mk(q, inf)
    b1 = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    b2 = torch.empty_like(b1)
    P.rte_rhs(p, b1)
    P.rte_rhs(ref, b2)
    torch.cuda.synchronize()
    assert torch.equal(b1, b2)


def test_loss_delta_autograd_is_the_library_gradient():
    import paper_2604_23265_b200 as P
    from paper_2604_23265_b200 import train as TR
    N, M = 6, 8
    med = _media(N, M, B=2)
    p2 = P.rte_setup_atfps(N, med.sigma_T, med.sigma_a, med.q, med.eps, med.g, med.inflow, delta=1e-2,
                           n_polar=1, n_azim=M)
    psi = torch.rand((2, N, N, M), device="cuda", requires_grad=True)
    w = torch.tensor([0.25, 2.0], device="cuda")
    (TR.loss_delta(psi, p2) * w).sum().backward()
    g = torch.empty_like(psi.detach())
    P.rte_atfps_loss(p2, psi.detach().contiguous(), g)
    torch.cuda.synchronize()
    expect = g * w.view(-1, 1, 1, 1)
    assert torch.allclose(psi.grad, expect, rtol=0, atol=0)


def test_training_lowers_loss_on_one_pair():
    """One medium, one fixed source: 150 Adam steps (lr 1e-3, cosine) lower loss_delta."""
    from paper_2604_23265_b200 import train as TR
    N, M = 16, 8
    med = _media(N, M, B=1)
    q = np.random.default_rng(3).uniform(0.0, 1.0, (1, 1, N, N)).astype(np.float32)
    out = TR.train(N, 1, M, med, L=3, C0=16, nu=2, delta=1e-2, steps=150, sources=q)
    l0, l1 = out["loss"][0], out["loss"][-1]
    assert l1 < 0.5 * l0, (l0, l1)
    assert out["lr"][-1] < 1e-3 and abs(out["lr"][75] - TR.cosine_lr(75, 150)) < 1e-12
