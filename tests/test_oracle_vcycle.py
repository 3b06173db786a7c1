"""Pins for the oracle's MgNet V-cycle (§3.3; readings Q12-Q20).

Each convolution is checked against the library routine (torch.nn.functional in
float64 on CPU); the transposed conv against the adjoint identity; the V-cycle
against closed forms (zero weights, identity taps), linearity, and an
independent NCHW torch composition of the same reading.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import workloads as W
from oracle import rte as O


def _t(x):  # NHWC numpy -> NCHW torch
    return torch.from_numpy(np.ascontiguousarray(np.transpose(x, (0, 3, 1, 2))))


def _n(t):
    return np.transpose(t.numpy(), (0, 2, 3, 1))


@pytest.mark.parametrize("stride,H", [(1, 8), (1, 5), (2, 8), (2, 16)])
def test_conv3x3_matches_torch(stride, H):
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, H, H, 6))
    Wt = rng.standard_normal((10, 6, 3, 3))
    ref = _n(F.conv2d(_t(x), torch.from_numpy(Wt), stride=stride, padding=1))
    assert np.allclose(O.conv3x3(x, Wt, stride), ref, rtol=1e-13, atol=1e-12)


@pytest.mark.parametrize("H", [1, 4, 8])
def test_conv_transpose_matches_torch(H):
    rng = np.random.default_rng(1)
    x = rng.standard_normal((2, H, H, 12))
    Wt = rng.standard_normal((12, 5, 4, 4))      # IOHW
    ref = _n(F.conv_transpose2d(_t(x), torch.from_numpy(Wt), stride=2, padding=1))
    got = O.conv_transpose4x4_s2(x, Wt)
    assert got.shape == (2, 2 * H, 2 * H, 5)
    assert np.allclose(got, ref, rtol=1e-13, atol=1e-12)


def test_transpose_is_adjoint():
    """<C x, y> = <x, Cᵀ y> with C the stride-2 pad-1 4x4 conv (torch conv2d as C)."""
    rng = np.random.default_rng(2)
    Wt = rng.standard_normal((8, 4, 4, 4))       # as conv_transpose: I=8 (coarse), O=4 (fine)
    xf = rng.standard_normal((1, 16, 16, 4))     # fine
    yc = rng.standard_normal((1, 8, 8, 8))       # coarse
    Cx = _n(F.conv2d(_t(xf), torch.from_numpy(Wt), stride=2, padding=1))   # O=8 from I=4
    lhs = np.sum(Cx * yc)
    rhs = np.sum(xf * O.conv_transpose4x4_s2(yc, Wt))
    assert abs(lhs - rhs) < 1e-11 * abs(lhs)


def _net(M=8, L=3, C0=4, nu=2, seed=0, std=0.1):
    n = W.mgnet_weight_count(M, L, C0, nu)
    w = np.random.default_rng(seed).standard_normal(n) * std
    return O.make_mgnet(w, M, L, C0, nu), w


def test_weight_count_mismatch_rejected():
    _, w = _net()
    with pytest.raises(ValueError):
        O.make_mgnet(w[:-1], 8, 3, 4, 2)


def test_zero_weights_identity():
    net, w = _net()
    net0 = O.make_mgnet(np.zeros_like(w), 8, 3, 4, 2)
    r = np.random.default_rng(3).standard_normal((1, 16, 16, 8))
    assert np.array_equal(O.vcycle(net0, r), r)


def test_vcycle_linear():
    net, _ = _net()
    rng = np.random.default_rng(4)
    r1, r2 = rng.standard_normal((2, 1, 16, 16, 8))
    lhs = O.vcycle(net, 2.0 * r1 - 0.5 * r2, add_identity=False)
    rhs = 2.0 * O.vcycle(net, r1, add_identity=False) - 0.5 * O.vcycle(net, r2, add_identity=False)
    assert np.allclose(lhs, rhs, rtol=1e-12, atol=1e-13)


def test_identity_tap_closed_form():
    """L=1, A=0, every B = identity centre tap: 2ν steps give u = 2ν f, so z = r + 2ν Θ Λ r."""
    M, C0, nu = 6, 4, 2
    shapes = W.mgnet_weight_shapes(M, 1, C0, nu)
    rng = np.random.default_rng(5)
    parts = []
    Lam = rng.standard_normal((C0, M, 1, 1)); Th = rng.standard_normal((M, C0, 1, 1))
    for name, shp in shapes:
        if name == "Lambda":
            parts.append(Lam.ravel())
        elif name == "Theta":
            parts.append(Th.ravel())
        elif name.startswith("A"):
            parts.append(np.zeros(shp).ravel())
        else:
            Wb = np.zeros(shp); Wb[np.arange(C0), np.arange(C0), 1, 1] = 1.0
            parts.append(Wb.ravel())
    net = O.make_mgnet(np.concatenate(parts), M, 1, C0, nu)
    r = rng.standard_normal((2, 5, 5, M))
    expect = r + 2 * nu * (r @ Lam[:, :, 0, 0].T) @ Th[:, :, 0, 0].T
    assert np.allclose(O.vcycle(net, r), expect, rtol=1e-13, atol=1e-13)


def _torch_vcycle(Wd, r, L, nu):
    """Independent NCHW composition of the same reading (Q13-Q18) from torch.nn.functional."""
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a))
    x = _t(r)
    f = [F.conv2d(x, T(Wd["Lambda"]))] + [None] * (L - 1)
    u = [None] * L
    conv = lambda a, w, s=1: F.conv2d(a, T(w), stride=s, padding=1)
    for l in range(L):
        u[l] = torch.zeros_like(f[l])
        names = [f"Bpre{l}_{i}" for i in range(nu)] + ([f"Bpost{l}_{i}" for i in range(nu)] if l == L - 1 else [])
        for nm in names:
            u[l] = u[l] + conv(f[l] - conv(u[l], Wd[f"A{l}"]), Wd[nm])
        if l < L - 1:
            f[l + 1] = conv(f[l] - conv(u[l], Wd[f"A{l}"]), Wd[f"R{l}"], 2)
    for l in range(L - 2, -1, -1):
        u[l] = u[l] + F.conv_transpose2d(u[l + 1], T(Wd[f"P{l}"]), stride=2, padding=1)
        for i in range(nu):
            u[l] = u[l] + conv(f[l] - conv(u[l], Wd[f"A{l}"]), Wd[f"Bpost{l}_{i}"])
    return r + _n(F.conv2d(u[0], T(Wd["Theta"])))


@pytest.mark.parametrize("L", [1, 2, 3])
def test_vcycle_matches_torch_composition(L):
    net, _ = _net(M=8, L=L, C0=4, nu=2, std=0.2)
    r = np.random.default_rng(6).standard_normal((2, 16, 16, 8))
    a, b = O.vcycle(net, r), _torch_vcycle(net.W, r, L, 2)
    assert np.max(np.abs(a - b)) < 1e-12 * np.max(np.abs(b))


def test_config_weight_counts():
    """Packed sizes of SURVEY §8(a) a0: 1.2 / 4.8 / 19 / 77 / 307 MiB."""
    mib = {k: W.mgnet_weight_count(c.M, c.L, c.C0, c.nu) * 4 / 2 ** 20 for k, c in W.CONFIGS.items()}
    for k, v in {1: 1.2, 2: 4.8, 3: 19, 4: 77, 5: 307}.items():
        assert abs(mib[k] - v) / v < 0.05, (k, mib[k])


# ---------------------------------------------------------------------------------------------
# Two-level closed form (multi-level branch of vcycle) and the packed weight
# order (reading R20/Q20), pinned together.  Every 3x3 / 4x4 kernel has only its centre tap
# (ky = kx = 1) non-zero, so each conv is a per-pixel channel matrix: the stride-2 restriction
# reads fine pixel (2y, 2x) (pad 1: padded index 2y + 1 = input 2y) and the transposed conv adds
# into fine pixel (2y, 2x) (2y - 1 + 1).  The V-cycle then collapses to per-pixel matrix algebra
# written out below by hand from the algorithm's steps: pre-smooth, restrict the residual of the
# pre-smoothed u, 2 nu coarse steps (pre then post B), prolongate-and-add, post-smooth, head.
# All channel matrices are random and non-symmetric and every B is distinct, so a wrong step order,
# a swapped pre/post set, a restriction of f instead of the residual, an OIHW/IOHW transposition
# or a misplaced block in the packed vector changes the result.
# ---------------------------------------------------------------------------------------------
def _pack_r20(blocks):
    """Pack named tensors in the order DESIGN.md R20 states, written out here independently of
    workloads.mgnet_weight_shapes and oracle.unpack_weights: Lambda; per level l: A^l, pre B x nu,
    post B x nu, then (l < L-1) R^l (OIHW) and P^l (IOHW); Theta."""
    return np.concatenate([blocks[k].ravel() for k in blocks])


def _centre(mat, kh):
    """[O][I] (or [I][O] for IOHW) channel matrix -> kernel with only the centre tap set."""
    Wk = np.zeros(mat.shape + (kh, kh))
    Wk[:, :, 1, 1] = mat
    return Wk


@pytest.mark.parametrize("nu", [1, 2])
def test_two_level_closed_form_and_weight_order(nu):
    M, C0, L = 3, 2, 2
    C1 = 2 * C0
    rng = np.random.default_rng(11 + nu)
    mats = {}
    blocks = {}
    mats["Lambda"] = rng.standard_normal((C0, M))
    blocks["Lambda"] = mats["Lambda"].reshape(C0, M, 1, 1)
    for l, C in ((0, C0), (1, C1)):
        for nm in [f"A{l}"] + [f"Bpre{l}_{i}" for i in range(nu)] + [f"Bpost{l}_{i}" for i in range(nu)]:
            mats[nm] = 0.5 * rng.standard_normal((C, C))
            blocks[nm] = _centre(mats[nm], 3)
        if l == 0:
            mats["R0"] = rng.standard_normal((C1, C0))          # OIHW: out = R0 @ in
            blocks["R0"] = _centre(mats["R0"], 3)
            mats["P0"] = rng.standard_normal((C1, C0))          # IOHW: out = P0.T @ in
            blocks["P0"] = _centre(mats["P0"], 4)
    mats["Theta"] = rng.standard_normal((M, C0))
    blocks["Theta"] = mats["Theta"].reshape(M, C0, 1, 1)
    w = _pack_r20(blocks)
    assert w.size == W.mgnet_weight_count(M, L, C0, nu)
    net = O.make_mgnet(w, M, L, C0, nu)

    H = 6
    r = rng.standard_normal((1, H, H, M))
    expect = np.array(r)
    m = mats
    smooth = lambda u, f, A, Bs: [u := u + B @ (f - A @ u) for B in Bs][-1]
    for y in range(H):
        for x in range(H):
            f0 = m["Lambda"] @ r[0, y, x]
            u0 = smooth(np.zeros(C0), f0, m["A0"], [m[f"Bpre0_{i}"] for i in range(nu)])
            if y % 2 == 0 and x % 2 == 0:                      # fine pixel (2y', 2x') of coarse (y', x')
                f1 = m["R0"] @ (f0 - m["A0"] @ u0)
                u1 = smooth(np.zeros(C1), f1, m["A1"],
                            [m[f"Bpre1_{i}"] for i in range(nu)] + [m[f"Bpost1_{i}"] for i in range(nu)])
                u0 = u0 + m["P0"].T @ u1
            u0 = smooth(u0, f0, m["A0"], [m[f"Bpost0_{i}"] for i in range(nu)])
            expect[0, y, x] += m["Theta"] @ u0
    got = O.vcycle(net, r)
    assert np.allclose(got, expect, rtol=1e-12, atol=1e-12)
    # and the workloads layout the CUDA path is fed with is this same order
    assert [n for n, _ in W.mgnet_weight_shapes(M, L, C0, nu)] == list(blocks)
