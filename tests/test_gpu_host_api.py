"""gmres_solve_host (host buffers, copies inside the call) and gmres_opts.x0_zero (include/rte.h):
both are pure plumbing, so their results must be bit-identical to the device-buffer gmres_solve with
x0 = 0 passed explicitly (DESIGN.md §5 "host path")."""
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
    return P, p, net, b


def _dev_solve(P, p, net, b, x0=None, **kw):
    x = torch.zeros(p.shape, dtype=torch.float64, device="cuda") if x0 is None else x0.clone().cuda()
    rep = P.gmres_solve(p, net, b, x, **kw)
    torch.cuda.synchronize()
    return x.cpu().numpy(), rep


def _strip(rep):
    return [{k: (v.tolist() if isinstance(v, np.ndarray) else v) for k, v in r.items()} for r in rep]


@pytest.mark.parametrize("precision", [0, 1])
def test_x0_zero_is_bitwise_identical(precision):
    cfg = W.small_config(5, N=32, M=32, n_polar=2, n_azim=16, L=3, C0=32)
    P, p, net, b = _setup(cfg)
    kw = dict(restart=8, maxit=20, rtol=1e-30, precision=precision)
    x_ref, r_ref = _dev_solve(P, p, net, b, **kw)
    garbage = torch.full(p.shape, np.nan, dtype=torch.float64)  # x0_zero must not read x
    x_z, r_z = _dev_solve(P, p, net, b, x0=garbage, x0_zero=True, **kw)
    assert np.array_equal(x_ref, x_z)
    assert _strip(r_ref) == _strip(r_z)


@pytest.mark.parametrize("x0_zero,pinned", [(True, True), (False, True), (True, False)])
def test_host_solve_matches_device_solve(x0_zero, pinned):
    """Fixed budget (the early copy is always right) with and without x0; numpy (pageable) buffers."""
    cfg = W.small_config(4, N=32, M=16, n_polar=2, n_azim=8, L=3, C0=16, B=2)
    P, p, net, b = _setup(cfg)
    x0 = torch.from_numpy(np.random.default_rng(5).standard_normal(p.shape) * 1e-3)
    kw = dict(restart=8, maxit=20, rtol=1e-30)
    x_ref, r_ref = _dev_solve(P, p, net, b, x0=None if x0_zero else x0, **kw)
    if pinned:
        bh = b.cpu().pin_memory()
        xh = (torch.zeros(p.shape, dtype=torch.float64) if x0_zero else x0.clone()).pin_memory()
        rep = P.gmres_solve_host(p, net, bh, xh, x0_zero=x0_zero, **kw)
        xo = xh.numpy()
    else:
        bh = b.cpu().numpy().copy()
        xo = np.full(p.shape, np.nan)
        rep = P.gmres_solve_host(p, net, bh, xo, x0_zero=x0_zero, **kw)
    assert np.array_equal(xo, x_ref)
    assert _strip(rep) == _strip(r_ref)


def test_host_solve_recopies_when_guess_is_wrong():
    """rtol below what the fp32 basis can certify: the Arnoldi estimate converges (the early copy
    starts), the fp64 true residual does not, and further cycles run -- x_host must still be the
    final x.  Also converging runs stop mid-cycle."""
    cfg = W.small_config(1, N=32, M=16, n_polar=2, n_azim=8, L=3, C0=16)
    P, p, net, b = _setup(cfg)
    for rtol, maxit, nt, m in ((1e-13, 60, net, 8), (1e-4, 600, None, 30)):
        kw = dict(restart=m, maxit=maxit, rtol=rtol)
        x_ref, r_ref = _dev_solve(P, p, nt, b, **kw)
        xh = torch.zeros(p.shape, dtype=torch.float64).pin_memory()
        rep = P.gmres_solve_host(p, nt, b.cpu().pin_memory(), xh, x0_zero=True, **kw)
        assert np.array_equal(xh.numpy(), x_ref)
        assert _strip(rep) == _strip(r_ref)
        if rtol == 1e-13:
            assert r_ref[0]["restarts"] >= 2 and not r_ref[0]["converged"]
        else:
            assert r_ref[0]["converged"] and r_ref[0]["iterations"] < maxit


def test_host_solve_rejects_bad_buffers():
    cfg = W.small_config(1, N=16, M=16, n_polar=2, n_azim=8, L=2, C0=16)
    P, p, net, b = _setup(cfg)
    with pytest.raises(ValueError):
        P.gmres_solve_host(p, net, b, torch.zeros(p.shape, dtype=torch.float64))  # b on the device
    with pytest.raises(ValueError):
        P.gmres_solve_host(p, net, b.cpu(), torch.zeros(p.shape, dtype=torch.float32))  # x dtype
    x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
    with pytest.raises(P.RteError):
        import ctypes as C
        from paper_2604_23265_b200 import _lib
        opts = _lib.gmres_opts(8, 10, 1e-6, 1, 2, 0, 2)  # x0_zero must be 0 or 1
        reps = (_lib.gmres_report * 1)()
        P.check("gmres_solve", P.lib.gmres_solve(p.handle, net.handle, C.c_void_p(b.data_ptr()),
                                                 C.c_void_p(x.data_ptr()), C.byref(opts), reps, None))
