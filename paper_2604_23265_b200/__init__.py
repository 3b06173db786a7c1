"""B200-native hot path of arXiv 2604.23265 (MgNet-preconditioned GMRES for the steady RTE).

Thin Python binding over the C ABI in ``include/rte.h`` (``librte_b200.so``).  The functions
keep the C names; they only marshal arguments.  Device buffers are torch CUDA tensors and the
stream is torch's current stream.  Every step of the path runs in the library's CUDA kernels;
there is no CPU fallback (importing raises if the library is missing).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import RTE_ENUMERIC, RTE_OK, RteError, check, gmres_opts, gmres_report, lib

__all__ = ["Problem", "MgNet", "rte_setup", "rte_setup_tfps", "rte_setup_atfps", "rte_atfps_info",
           "rte_atfps_reconstruct", "rte_atfps_reconstruct_f64", "rte_atfps_fit", "rte_atfps_fit_f64", "rte_set_source",
           "rte_atfps_loss", "rte_atfps_loss_f64", "rte_tfps_info", "rte_tfps_modes", "rte_tfps_reconstruct",
           "rte_tfps_reconstruct_f64", "rte_rhs", "rte_apply", "rte_apply_f64", "rte_blockjacobi_apply", "mgnet_create",
           "mgnet_vcycle", "mgnet_vcycle_f64", "mgnet_coeffnet", "mgnet_coeffnet_weight_count", "mgnet_modulation", "gmres_prepare", "gmres_solve", "gmres_solve_host", "rte_quadrature", "rte_hg_matrix", "rte_launch_count", "rte_timing_enable", "rte_timing_filter", "rte_timing_reset",
           "rte_timing_get", "RteError", "LIB_PATH"]

LIB_PATH = _lib.LIB_PATH


def _stream(stream=None) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def _fptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _dev(t, dtype_name: str):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.is_contiguous()):
        raise ValueError("expected a contiguous CUDA tensor")
    want = {"f32": torch.float32, "f64": torch.float64}[dtype_name]
    if t.dtype != want:
        raise ValueError(f"expected dtype {want}, got {t.dtype}")
    return C.c_void_p(t.data_ptr())


class Problem:
    """Owner of an ``rte_problem*`` handle (rte_setup / rte_destroy)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        b, n, m, tot = C.c_int(), C.c_int(), C.c_int(), C.c_int64()
        check("rte_problem_info", lib.rte_problem_info(self._h, C.byref(b), C.byref(n), C.byref(m), C.byref(tot)))
        self.batch, self.N, self.M, self.n = b.value, n.value, m.value, tot.value

    @property
    def handle(self):
        return self._h

    @property
    def is_tfps(self) -> bool:
        return lib.rte_tfps_info(self._h, None, None, None, None) == RTE_OK

    @property
    def shape(self):
        return (self.batch, self.N, self.N, self.M)

    def ordinates(self):
        nd = self.M // 2 if self.is_tfps else self.M
        arrs = [np.zeros(nd) for _ in range(4)]
        check("rte_get_ordinates", lib.rte_get_ordinates(self._h, *[_dptr(a) for a in arrs]))
        return tuple(arrs)   # c, s, zeta, w

    def close(self):
        if self._h:
            lib.rte_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def rte_setup(N: int, sigma_T, sigma_a, q, eps, g, inflow=None, *, n_polar: int = 0, n_azim: int = 0,
              ordinates: Optional[Sequence[np.ndarray]] = None, batch: Optional[int] = None,
              _fn: str = "rte_setup", _extra: tuple = ()) -> Problem:
    """rte_setup(grid, ordinates, sigma_T, sigma_a, q, eps, g, inflow) -> Problem (host inputs)."""
    sT, sA, qq, ee = (_f32(a) for a in (sigma_T, sigma_a, q, eps))
    B = batch if batch is not None else (sT.shape[0] if sT.ndim == 3 else 1)
    gg = _f32(np.broadcast_to(np.asarray(g, np.float32), (B,)))
    grid = _lib.rte_grid(B, N, N)
    if ordinates is None:
        ordn = _lib.rte_ordinates(n_polar * n_azim, n_polar, n_azim, None, None, None, None)
        keep = ()
    else:
        keep = tuple(np.ascontiguousarray(np.asarray(a, np.float64)) for a in ordinates)
        ordn = _lib.rte_ordinates(keep[0].size, 0, 0, *[_dptr(a) for a in keep])
    inf = _fptr(_f32(inflow)) if inflow is not None else None
    infa = _f32(inflow) if inflow is not None else None
    h = C.c_void_p()
    check(_fn, getattr(lib, _fn)(C.byref(grid), C.byref(ordn), _fptr(sT), _fptr(sA), _fptr(qq), _fptr(ee),
                                 _fptr(gg), _fptr(infa) if infa is not None else None, *_extra, C.byref(h)))
    del keep, inf
    return Problem(h)


def rte_setup_tfps(N: int, sigma_T, sigma_a, q, eps, g, inflow=None, **kw) -> Problem:
    """rte_setup_tfps: the TFPS alpha-space system of the same problem (NEXT-3, include/rte.h); the
    Problem's vectors hold alpha [batch][N][N][2 Md] (Problem.M = 2 Md)."""
    return rte_setup(N, sigma_T, sigma_a, q, eps, g, inflow, _fn="rte_setup_tfps", **kw)


def rte_setup_atfps(N: int, sigma_T, sigma_a, q, eps, g, inflow=None, *, delta: float, **kw) -> Problem:
    """rte_setup_atfps: the ATFPS compressed system (NEXT-3b, include/rte.h) on the padded [B][N][N][2 Md]
    layout."""
    return rte_setup(N, sigma_T, sigma_a, q, eps, g, inflow, _fn="rte_setup_atfps", _extra=(C.c_double(delta),), **kw)


def rte_atfps_info(p: Problem):
    """(delta, compressed dimension, kept mask [nmat][2 Md] as bool)."""
    d, n = C.c_double(), C.c_int64()
    check("rte_atfps_info", lib.rte_atfps_info(p.handle, C.byref(d), C.byref(n), None))
    nm = rte_tfps_info(p)[0].shape[0]
    sel = np.zeros(nm * p.M, np.uint8)
    check("rte_atfps_info", lib.rte_atfps_info(p.handle, None, None, sel.ctypes.data_as(C.POINTER(C.c_uint8))))
    return d.value, n.value, sel.reshape(nm, p.M).astype(bool)


def rte_atfps_reconstruct(p: Problem, alpha, psi, full=None, stream=None) -> None:
    check("rte_atfps_reconstruct", lib.rte_atfps_reconstruct(p.handle, _dev(alpha, "f32"), _dev(psi, "f32"),
                                                             _dev(full, "f32") if full is not None else None,
                                                             C.c_void_p(_stream(stream))))


def rte_atfps_reconstruct_f64(p: Problem, alpha, psi, full=None, stream=None) -> None:
    check("rte_atfps_reconstruct_f64", lib.rte_atfps_reconstruct_f64(
        p.handle, _dev(alpha, "f64"), _dev(psi, "f64"), _dev(full, "f64") if full is not None else None,
        C.c_void_p(_stream(stream))))


def rte_set_source(p: Problem, q, inflow=None) -> None:
    """Replace the source q [batch][N][N] (and the inflow [batch][4][N][directions] if given); host arrays."""
    qa = _f32(q)
    ia = _f32(inflow) if inflow is not None else None
    check("rte_set_source", lib.rte_set_source(p.handle, _fptr(qa), _fptr(ia) if ia is not None else None))


def rte_atfps_fit(p: Problem, psi, alpha, stream=None) -> None:
    check("rte_atfps_fit", lib.rte_atfps_fit(p.handle, _dev(psi, "f32"), _dev(alpha, "f32"), C.c_void_p(_stream(stream))))


def rte_atfps_fit_f64(p: Problem, psi, alpha, stream=None) -> None:
    check("rte_atfps_fit_f64", lib.rte_atfps_fit_f64(p.handle, _dev(psi, "f64"), _dev(alpha, "f64"),
                                                     C.c_void_p(_stream(stream))))


def rte_atfps_loss(p: Problem, psi, grad=None, stream=None) -> np.ndarray:
    """loss_delta per sample (host float64 [batch]); fills grad (device, psi's layout) if given."""
    out = np.zeros(p.batch, np.float64)
    check("rte_atfps_loss", lib.rte_atfps_loss(p.handle, _dev(psi, "f32"), _dptr(out),
                                               _dev(grad, "f32") if grad is not None else None,
                                               C.c_void_p(_stream(stream))))
    return out


def rte_atfps_loss_f64(p: Problem, psi, grad=None, stream=None) -> np.ndarray:
    out = np.zeros(p.batch, np.float64)
    check("rte_atfps_loss_f64", lib.rte_atfps_loss_f64(p.handle, _dev(psi, "f64"), _dptr(out),
                                                       _dev(grad, "f64") if grad is not None else None,
                                                       C.c_void_p(_stream(stream))))
    return out


def rte_tfps_modes(c, s, S, gamma: float):
    """Host-only: (xi [2M], L [M][2M]) of one TFPS material (include/rte.h rte_tfps_modes)."""
    c, s, S = (np.ascontiguousarray(np.asarray(a, np.float64)) for a in (c, s, S))
    M = c.size
    xi, L = np.zeros(2 * M), np.zeros((M, 2 * M))
    check("rte_tfps_modes", lib.rte_tfps_modes(M, _dptr(c), _dptr(s), _dptr(S), float(gamma), _dptr(xi), _dptr(L)))
    return xi, L


def rte_tfps_info(p: Problem):
    """(xi [nmat][2Md], L [nmat][Md][2Md]) of a TFPS problem's materials (host fp64)."""
    nm, md = C.c_int(), C.c_int()
    check("rte_tfps_info", lib.rte_tfps_info(p.handle, C.byref(nm), C.byref(md), None, None))
    xi = np.zeros((nm.value, 2 * md.value))
    L = np.zeros((nm.value, md.value, 2 * md.value))
    check("rte_tfps_info", lib.rte_tfps_info(p.handle, None, None, _dptr(xi), _dptr(L)))
    return xi, L


def rte_tfps_reconstruct(p: Problem, alpha, psi, stream=None) -> None:
    check("rte_tfps_reconstruct", lib.rte_tfps_reconstruct(p.handle, _dev(alpha, "f32"), _dev(psi, "f32"),
                                                           C.c_void_p(_stream(stream))))


def rte_tfps_reconstruct_f64(p: Problem, alpha, psi, stream=None) -> None:
    check("rte_tfps_reconstruct_f64", lib.rte_tfps_reconstruct_f64(p.handle, _dev(alpha, "f64"), _dev(psi, "f64"),
                                                                   C.c_void_p(_stream(stream))))


def rte_quadrature(n_polar: int, n_azim: int):
    """Host-only: the built-in product quadrature (c, s, zeta, w)."""
    M = n_polar * n_azim
    arrs = [np.zeros(M) for _ in range(4)]
    check("rte_quadrature", lib.rte_quadrature(n_polar, n_azim, *[_dptr(a) for a in arrs]))
    return tuple(arrs)


def rte_hg_matrix(c, s, zeta, w, g: float) -> np.ndarray:
    """Host-only: the row-normalised HG matrix S = K W ([M][M])."""
    arrs = [np.ascontiguousarray(np.asarray(a, np.float64)) for a in (c, s, zeta, w)]
    M = arrs[0].size
    S = np.zeros((M, M))
    check("rte_hg_matrix", lib.rte_hg_matrix(M, *[_dptr(a) for a in arrs], float(g), _dptr(S)))
    return S


def rte_rhs(p: Problem, b, stream=None) -> None:
    check("rte_rhs", lib.rte_rhs(p.handle, _dev(b, "f32"), C.c_void_p(_stream(stream))))


def rte_apply(p: Problem, x, y, stream=None) -> None:
    check("rte_apply", lib.rte_apply(p.handle, _dev(x, "f32"), _dev(y, "f32"), C.c_void_p(_stream(stream))))


def rte_blockjacobi_apply(p: Problem, r, z, stream=None) -> None:
    """z = A_cc^{-1} r per cell (NEXT-2 block Jacobi; float32 or float64 tensors)."""
    if r.dtype == np.float64 or str(getattr(r, "dtype", "")) == "torch.float64":
        check("rte_blockjacobi_apply_f64", lib.rte_blockjacobi_apply_f64(p.handle, _dev(r, "f64"), _dev(z, "f64"),
                                                                        C.c_void_p(_stream(stream))))
    else:
        check("rte_blockjacobi_apply", lib.rte_blockjacobi_apply(p.handle, _dev(r, "f32"), _dev(z, "f32"),
                                                                C.c_void_p(_stream(stream))))


def rte_apply_f64(p: Problem, x, y, stream=None) -> None:
    check("rte_apply_f64", lib.rte_apply_f64(p.handle, _dev(x, "f64"), _dev(y, "f64"), C.c_void_p(_stream(stream))))


class MgNet:
    """Owner of an ``mgnet_net*`` handle (mgnet_create / mgnet_destroy)."""

    def __init__(self, handle, problem: Problem, levels: int, c0: int, nu: int):
        self._h = handle
        self.problem = problem  # keep the problem alive
        self.levels, self.c0, self.nu = levels, c0, nu

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            lib.mgnet_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def mgnet_create(p: Problem, levels: int, c0: int, nu: int, weights) -> MgNet:
    w = _f32(weights).ravel()
    h = C.c_void_p()
    check("mgnet_create", lib.mgnet_create(p.handle, levels, c0, nu, _fptr(w), w.size, C.byref(h)))
    return MgNet(h, p, levels, c0, nu)


def mgnet_coeffnet_weight_count(levels: int, c0: int) -> int:
    return int(lib.mgnet_coeffnet_weight_count(levels, c0))


def mgnet_coeffnet(net: MgNet, sigma_T, sigma_a, eps, weights) -> None:
    """CoeffNet (NEXT-1): compute the modulation maps of every level from the medium and attach them
    to `net` (weights=None removes them).  sigma_T, sigma_a, eps: [batch][N][N] like rte_setup."""
    if weights is None:
        check("mgnet_coeffnet", lib.mgnet_coeffnet(net.handle, None, None, None, None, 0))
        return
    B, N = net.problem.shape[0], net.problem.shape[1]
    f = [_f32(a).reshape(B, N, N) for a in (sigma_T, sigma_a, eps)]
    w = _f32(weights).ravel()
    check("mgnet_coeffnet", lib.mgnet_coeffnet(net.handle, _fptr(f[0]), _fptr(f[1]), _fptr(f[2]), _fptr(w), w.size))


def mgnet_modulation(net: MgNet, level: int, which: int) -> np.ndarray:
    """The fp64 map a^[level] (which=0) or abar^[level] (which=1), [batch][N_l][N_l][C_l]."""
    B, N = net.problem.shape[0], net.problem.shape[1]
    out = np.empty((B, N >> level, N >> level, net.c0 << level), np.float64)
    check("mgnet_modulation", lib.mgnet_modulation(net.handle, level, which, _dptr(out)))
    return out


def mgnet_vcycle(net: MgNet, r, z, add_identity: bool = True, stream=None) -> None:
    check("mgnet_vcycle", lib.mgnet_vcycle(net.handle, _dev(r, "f32"), _dev(z, "f32"), int(add_identity),
                                           C.c_void_p(_stream(stream))))


def mgnet_vcycle_f64(net: MgNet, r, z, add_identity: bool = True, stream=None) -> None:
    check("mgnet_vcycle_f64", lib.mgnet_vcycle_f64(net.handle, _dev(r, "f64"), _dev(z, "f64"), int(add_identity),
                                                   C.c_void_p(_stream(stream))))


def gmres_prepare(p: Problem, net: Optional[MgNet], *, restart: int = 30, precond: Optional[int] = None,
                  reorth: int = 3, precision: int = 0, stream=None) -> None:
    """Capture the per-Arnoldi-step CUDA graphs for gmres_solve with these options (setup; optional)."""
    if precond is None:
        precond = 1 if net is not None else 0
    opts = gmres_opts(restart, 1, 0.0, precond, reorth, precision)
    check("gmres_prepare", lib.gmres_prepare(p.handle, net.handle if net is not None else None, C.byref(opts),
                                             C.c_void_p(_stream(stream))))


def _host(t, dtype_name: str, writeable: bool = False):
    """Host buffer pointer: a contiguous CPU torch tensor (pinned for full-rate copies) or numpy array."""
    import torch
    want_np = {"f32": np.float32, "f64": np.float64}[dtype_name]
    if isinstance(t, torch.Tensor):
        if t.is_cuda or not t.is_contiguous():
            raise ValueError("expected a contiguous CPU tensor")
        if t.dtype != {"f32": torch.float32, "f64": torch.float64}[dtype_name]:
            raise ValueError(f"expected dtype {dtype_name}, got {t.dtype}")
        return C.c_void_p(t.data_ptr())
    if not (isinstance(t, np.ndarray) and t.dtype == want_np and t.flags.c_contiguous
            and (t.flags.writeable or not writeable)):
        raise ValueError(f"expected a contiguous{' writeable' if writeable else ''} {want_np.__name__} array")
    return C.c_void_p(t.ctypes.data)


def _gmres_call(name, fn, p, net, b_ptr, x_ptr, restart, maxit, rtol, precond, reorth, precision, x0_zero,
                history, hessenberg, stream):
    if precond is None:
        precond = 1 if net is not None else 0
    opts = gmres_opts(restart, maxit, rtol, precond, reorth, precision, int(x0_zero))
    B = p.batch
    reps = (gmres_report * B)()
    hist = [np.zeros(max(maxit, 1)) for _ in range(B)]
    hess = [np.zeros((restart + 1) * restart) for _ in range(B)]
    for i in range(B):
        reps[i].history = _dptr(hist[i]) if history else None
        reps[i].hessenberg = _dptr(hess[i]) if hessenberg else None
    status = fn(p.handle, net.handle if net is not None else None, b_ptr, x_ptr, C.byref(opts), reps,
                C.c_void_p(_stream(stream)))
    if status not in (RTE_OK, RTE_ENUMERIC):
        check(name, status)
    out = []
    for i in range(B):
        r = reps[i]
        d = dict(iterations=r.iterations, restarts=r.restarts, converged=bool(r.converged),
                 breakdown=int(r.breakdown), relres_true=r.relres_true, relres_est=r.relres_est)
        if history:
            d["history"] = hist[i][:r.iterations].copy()
        if hessenberg:
            d["hessenberg"] = hess[i].reshape(restart + 1, restart)
        out.append(d)
    if status == RTE_ENUMERIC:  # a NaN/Inf stopped a sample: loud, with the filled reports attached
        err = RteError(name, status)
        err.reports = out
        raise err
    return out


def gmres_solve(p: Problem, net: Optional[MgNet], b, x, *, restart: int = 30, maxit: int = 1000,
                rtol: float = 1e-8, precond: Optional[int] = None, reorth: int = 3, precision: int = 0,
                x0_zero: bool = False, history: bool = True, hessenberg: bool = False, stream=None):
    """Restarted right-preconditioned GMRES; x (float64 CUDA tensor) holds x0 on entry (unless
    x0_zero: then it is set to 0 and A x0 is not applied), x on exit.
    reorth: 3 = DCGS2, delayed re-orthogonalisation (default: CGS2's orthogonality at two basis
    passes per step), 0 = CGS2, 1 = CGS1, 2 = selective re-orthogonalisation (gmres_opts).

    Returns a list of per-sample dicts (iterations, restarts, converged, breakdown, relres_true,
    relres_est, history [, hessenberg])."""
    return _gmres_call("gmres_solve", lib.gmres_solve, p, net, _dev(b, "f32"), _dev(x, "f64"), restart, maxit,
                       rtol, precond, reorth, precision, x0_zero, history, hessenberg, stream)


def gmres_solve_host(p: Problem, net: Optional[MgNet], b, x, *, restart: int = 30, maxit: int = 1000,
                     rtol: float = 1e-8, precond: Optional[int] = None, reorth: int = 3, precision: int = 0,
                     x0_zero: bool = False, history: bool = True, hessenberg: bool = False, stream=None):
    """gmres_solve with HOST buffers (include/rte.h): b float32, x float64 (CPU tensors, pinned for
    full-rate copies, or numpy arrays); the copies in and out happen inside the call."""
    return _gmres_call("gmres_solve_host", lib.gmres_solve_host, p, net, _host(b, "f32"), _host(x, "f64", True), restart,
                       maxit, rtol, precond, reorth, precision, x0_zero, history, hessenberg, stream)


def rte_launch_count(reset: bool = False) -> int:
    return int(lib.rte_launch_count(int(reset)))


def rte_timing_enable(on: bool = True) -> None:
    check("rte_timing_enable", lib.rte_timing_enable(int(on)))


def rte_timing_filter(name: Optional[str] = None) -> None:
    """Time only the launches of class `name` (None = all classes)."""
    check("rte_timing_filter", lib.rte_timing_filter(name.encode() if name else None))


def rte_timing_reset() -> None:
    check("rte_timing_reset", lib.rte_timing_reset())


KINDS = {0: "hbm", 1: "tensor_3xtf32", 2: "fp32_simt", 3: "fp64_simt", 4: "latency"}


def rte_timing_get():
    """Per-kernel-class aggregates since the last reset: list of dicts (name, kind, launches, ms,
    flops, bytes), all algorithmic flops/bytes as tagged by the library."""
    cnt = C.c_int()
    check("rte_timing_get", lib.rte_timing_get(-1, None, 0, None, None, None, None, None, C.byref(cnt)))
    out = []
    for i in range(cnt.value):
        name = C.create_string_buffer(128)
        kind, la = C.c_int(), C.c_int64()
        ms, fl, by = C.c_double(), C.c_double(), C.c_double()
        check("rte_timing_get", lib.rte_timing_get(i, name, 128, C.byref(kind), C.byref(la), C.byref(ms),
                                                   C.byref(fl), C.byref(by), None))
        out.append(dict(name=name.value.decode(), kind=KINDS.get(kind.value, str(kind.value)),
                        launches=la.value, ms=ms.value, flops=fl.value, bytes=by.value))
    return out
