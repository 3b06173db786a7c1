"""C-ABI library checks that need no GPU: it loads, exports every function include/rte.h
declares, and its host-side setup (quadrature, HG matrix, argument validation) agrees with
the oracle.  No device computation is called here."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "rte.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(?:rte_status|void|const char\*|int64_t)\s+\**\s*((?:rte|mgnet|gmres)_\w+)\s*\(", src)
    return sorted(set(names))


def test_header_declares_the_north_star_calls():
    names = _header_functions()
    for n in ("rte_setup", "rte_apply", "mgnet_vcycle", "gmres_solve"):
        assert n in names


def test_library_exports_every_header_symbol():
    import paper_2604_23265_b200 as P
    from paper_2604_23265_b200 import _lib
    for n in _header_functions():
        assert hasattr(_lib.lib, n), n
        assert n in _lib.EXPORTED, n
    assert os.path.exists(P.LIB_PATH)


@pytest.mark.parametrize("np_,na", [(2, 8), (2, 16), (4, 16), (4, 32), (8, 32), (3, 12)])
def test_host_quadrature_matches_oracle(np_, na):
    import paper_2604_23265_b200 as P
    from oracle import rte as O
    q = O.quadrature(np_, na)
    c, s, z, w = P.rte_quadrature(np_, na)
    for a, b in ((c, q.c), (s, q.s), (z, q.zeta), (w, q.w)):
        assert np.max(np.abs(a - b)) < 1e-14


@pytest.mark.parametrize("g", [0.0, 0.5, 0.8, 0.9, -0.3])
def test_host_hg_matrix_matches_oracle(g):
    import paper_2604_23265_b200 as P
    from oracle import rte as O
    q = O.quadrature(4, 32)
    S = P.rte_hg_matrix(q.c, q.s, q.zeta, q.w, g)
    assert np.max(np.abs(S - O.scattering_matrix(q, g)[1])) < 1e-14


@pytest.mark.parametrize("bad", ["eps", "g", "neg", "nx"])
def test_setup_rejects_invalid_inputs(bad):
    import paper_2604_23265_b200 as P
    N = 4
    sT, sA, q, e = np.ones((1, N, N)), np.zeros((1, N, N)), np.ones((1, N, N)), np.ones((1, N, N))
    g = [0.5]
    if bad == "eps":
        e = e * 2.0
    elif bad == "g":
        g = [1.0]
    elif bad == "neg":
        sA = np.full((1, N, N), 10.0)   # sigma_T/eps < eps sigma_a
    with pytest.raises(P.RteError) as ei:
        if bad == "nx":
            P.rte_setup(0, sT, sA, q, e, g, n_polar=2, n_azim=8)
        else:
            P.rte_setup(N, sT, sA, q, e, g, n_polar=2, n_azim=8)
    assert ei.value.status == 1  # RTE_EINVAL


def test_rejects_bad_quadrature_request():
    import paper_2604_23265_b200 as P
    with pytest.raises(P.RteError):
        P.rte_quadrature(2, 6)


@pytest.mark.parametrize("L,C0", [(1, 4), (3, 16), (6, 32)])
def test_coeffnet_weight_count_matches_packed_layout(L, C0):
    """mgnet_coeffnet_weight_count (host) equals the documented packed layout (R33)."""
    import paper_2604_23265_b200 as P
    import workloads as W
    assert P.mgnet_coeffnet_weight_count(L, C0) == W.coeffnet_weight_count(L, C0)


def test_host_buffer_validation():
    """gmres_solve_host's marshalling (no GPU): b may be read-only, x must be writeable; dtype,
    contiguity and device are checked before the C call."""
    import torch
    import paper_2604_23265_b200 as P
    b = np.zeros(8, np.float32)
    b.flags.writeable = False
    assert P._host(b, "f32").value == b.ctypes.data
    x = np.zeros(8)
    assert P._host(x, "f64", True).value == x.ctypes.data
    ro = np.zeros(8)
    ro.flags.writeable = False
    for bad, dt, w in ((ro, "f64", True), (np.zeros(8, np.float32), "f64", True), (np.zeros((4, 4))[:, ::2], "f64", True),
                       (torch.zeros(8, dtype=torch.float64), "f32", False), ([0.0] * 8, "f64", True)):
        with pytest.raises(ValueError):
            P._host(bad, dt, w)
    t = torch.zeros(8, dtype=torch.float64)
    assert P._host(t, "f64", True).value == t.data_ptr()
    assert [f[0] for f in P.gmres_opts._fields_][-1] == "x0_zero"


@pytest.mark.parametrize("n_polar,n_azim,g,gamma", [(1, 8, 0.5, 0.99), (2, 16, 0.5, 0.99999), (4, 16, 0.9, 0.5),
                                                   (2, 8, 0.0, 0.0)])
def test_host_tfps_modes_match_oracle(n_polar, n_azim, g, gamma):
    """The library's TFPS eigen solver (symmetrised Cholesky + Jacobi, tfps_setup.cpp) against the oracle's
    numpy.linalg.eig of C^-1 (gamma S - I) (oracle/tfps.py): same xi, same normalised eigenvectors."""
    import paper_2604_23265_b200 as P
    from oracle import rte as O
    from oracle import tfps as T
    qd = O.quadrature(n_polar, n_azim)
    _, S = O.scattering_matrix(qd, g)
    xi, L = P.rte_tfps_modes(qd.c, qd.s, S, gamma)
    md = T.local_modes(qd, S, gamma)
    assert np.allclose(xi, md.xi, rtol=1e-10, atol=1e-12)
    if gamma > 0:   # (gamma = 0: degenerate eigenvalues, eigenvectors defined up to a basis of each eigenspace)
        assert np.allclose(L, md.L, rtol=1e-8, atol=1e-9)
