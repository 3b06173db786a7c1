"""ctypes binding of include/rte.h -- argument marshalling only.

Every function named here is the C function of the same name in librte_b200.so; device
buffers are torch CUDA tensors (PyTorch supplies memory and streams, nothing else).  There is
no CPU fallback: if the shared library is missing or fails to load, importing this module
raises ImportError.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RTE_LIB_PATH") or os.path.join(HERE, "librte_b200.so")  # override: perf experiments

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2604_23265_b200.build` "
                      "(there is no CPU fallback)")
lib = C.CDLL(LIB_PATH)

RTE_OK, RTE_EINVAL, RTE_ENOMEM, RTE_ECUDA, RTE_EINTERNAL, RTE_ENUMERIC = range(6)


class rte_grid(C.Structure):
    _fields_ = [("batch", C.c_int), ("nx", C.c_int), ("ny", C.c_int)]


class rte_ordinates(C.Structure):
    _fields_ = [("M", C.c_int), ("n_polar", C.c_int), ("n_azim", C.c_int),
                ("c", C.POINTER(C.c_double)), ("s", C.POINTER(C.c_double)),
                ("zeta", C.POINTER(C.c_double)), ("w", C.POINTER(C.c_double))]


class gmres_opts(C.Structure):
    _fields_ = [("restart", C.c_int), ("maxit", C.c_int), ("rtol", C.c_double),
                ("precond", C.c_int), ("reorth", C.c_int), ("precision", C.c_int), ("x0_zero", C.c_int)]


class gmres_report(C.Structure):
    _fields_ = [("iterations", C.c_int), ("restarts", C.c_int), ("converged", C.c_int),
                ("breakdown", C.c_int), ("relres_true", C.c_double), ("relres_est", C.c_double),
                ("history", C.POINTER(C.c_double)), ("hessenberg", C.POINTER(C.c_double))]


_vp = C.c_void_p
_fp = C.POINTER(C.c_float)
SIGS = {
    "rte_setup": (C.c_int, [C.POINTER(rte_grid), C.POINTER(rte_ordinates), _fp, _fp, _fp, _fp, _fp, _fp,
                            C.POINTER(_vp)]),
    "rte_setup_tfps": (C.c_int, [C.POINTER(rte_grid), C.POINTER(rte_ordinates), _fp, _fp, _fp, _fp, _fp, _fp,
                                 C.POINTER(_vp)]),
    "rte_tfps_modes": (C.c_int, [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                 C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "rte_tfps_info": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_double),
                                C.POINTER(C.c_double)]),
    "rte_tfps_reconstruct": (C.c_int, [_vp, _vp, _vp, _vp]),
    "rte_setup_atfps": (C.c_int, [C.POINTER(rte_grid), C.POINTER(rte_ordinates), _fp, _fp, _fp, _fp, _fp, _fp,
                                  C.c_double, C.POINTER(_vp)]),
    "rte_atfps_info": (C.c_int, [_vp, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_uint8)]),
    "rte_atfps_reconstruct": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "rte_atfps_reconstruct_f64": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "rte_set_source": (C.c_int, [_vp, _fp, _fp]),
    "rte_atfps_fit": (C.c_int, [_vp, _vp, _vp, _vp]),
    "rte_atfps_fit_f64": (C.c_int, [_vp, _vp, _vp, _vp]),
    "rte_atfps_loss": (C.c_int, [_vp, _vp, C.POINTER(C.c_double), _vp, _vp]),
    "rte_atfps_loss_f64": (C.c_int, [_vp, _vp, C.POINTER(C.c_double), _vp, _vp]),
    "rte_tfps_reconstruct_f64": (C.c_int, [_vp, _vp, _vp, _vp]),
    "rte_destroy": (None, [_vp]),
    "rte_problem_info": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                   C.POINTER(C.c_int64)]),
    "rte_get_ordinates": (C.c_int, [_vp, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                    C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "rte_quadrature": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                 C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "rte_hg_matrix": (C.c_int, [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                C.POINTER(C.c_double), C.c_double, C.POINTER(C.c_double)]),
    "rte_rhs": (C.c_int, [_vp, _vp, _vp]),
    "rte_apply": (C.c_int, [_vp, _vp, _vp, _vp]),
    "rte_apply_f64": (C.c_int, [_vp, _vp, _vp, _vp]),
    "mgnet_create": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _fp, C.c_size_t, C.POINTER(_vp)]),
    "mgnet_destroy": (None, [_vp]),
    "mgnet_vcycle": (C.c_int, [_vp, _vp, _vp, C.c_int, _vp]),
    "mgnet_vcycle_f64": (C.c_int, [_vp, _vp, _vp, C.c_int, _vp]),
    "mgnet_coeffnet_weight_count": (C.c_size_t, [C.c_int, C.c_int]),
    "rte_blockjacobi_apply": (C.c_int, [_vp, _vp, _vp, _vp]),
    "rte_blockjacobi_apply_f64": (C.c_int, [_vp, _vp, _vp, _vp]),
    "mgnet_coeffnet": (C.c_int, [_vp, _fp, _fp, _fp, _fp, C.c_size_t]),
    "mgnet_modulation": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "gmres_solve": (C.c_int, [_vp, _vp, _vp, _vp, C.POINTER(gmres_opts), C.POINTER(gmres_report), _vp]),
    "gmres_prepare": (C.c_int, [_vp, _vp, C.POINTER(gmres_opts), _vp]),
    "gmres_solve_host": (C.c_int, [_vp, _vp, _vp, _vp, C.POINTER(gmres_opts), C.POINTER(gmres_report), _vp]),
    "rte_launch_count": (C.c_int64, [C.c_int]),
    "rte_last_error": (C.c_char_p, []),
    "rte_timing_enable": (C.c_int, [C.c_int]),
    "rte_timing_filter": (C.c_int, [C.c_char_p]),
    "rte_debug_counters": (C.c_int, [C.POINTER(C.c_uint64), C.c_int, C.c_int]),
    "rte_timing_reset": (C.c_int, []),
    "rte_timing_get": (C.c_int, [C.c_int, C.c_char_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int64),
                                 C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                 C.POINTER(C.c_int)]),
}
EXPORTED = tuple(SIGS)
for _name, (_res, _args) in SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class RteError(RuntimeError):
    def __init__(self, fn: str, status: int):
        msg = lib.rte_last_error().decode(errors="replace")
        super().__init__(f"{fn} failed with status {status}: {msg}")
        self.status = status


def check(fn: str, status: int) -> None:
    if status != RTE_OK:
        raise RteError(fn, status)
