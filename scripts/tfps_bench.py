"""NEXT-3 measurement: the TFPS alpha-space system of config 2 (64^2 cells x 32 directions, two
materials -> 64 coefficients per cell) on the B200 -- operator applies/s (fp32 and fp64), and GMRES(30)
iterations/s of whole restart cycles, unpreconditioned and with an MgNet (L = 4, C0 = 16) on the
64-channel alpha vectors -- with the kernel's algorithmic flops/bytes per launch (include/rte.h
rte_setup_tfps; csrc/tfps.cu).  Prints one JSON object.

  python scripts/tfps_bench.py [--cycles 3] [--delta 1e-4] > profiles/r02/tfps_cfg2.json
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_23265_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cycles", type=int, default=3)
ap.add_argument("--delta", type=float, default=1e-4, help="ATFPS tolerance of the compressed-system runs")
a = ap.parse_args()
cfg = W.config(2)
media = W.make_media(cfg)
t0 = time.perf_counter()
p = P.rte_setup_tfps(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                     n_polar=cfg.n_polar, n_azim=cfg.n_azim)
setup_ms = (time.perf_counter() - t0) * 1e3
xi, _ = P.rte_tfps_info(p)
out = {"workload": "config 2 TFPS alpha system: 64^2 cells x 32 directions, 64 coefficients per cell",
       "materials": int(xi.shape[0]), "unknowns": p.n, "setup_ms": round(setup_ms, 1)}
x = torch.randn(p.shape, device="cuda")
y = torch.empty_like(x)
x64, y64 = x.double(), torch.empty(p.shape, dtype=torch.float64, device="cuda")


def rate(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return reps / (e0.elapsed_time(e1) * 1e-3)


out["apply_f32_per_s"] = rate(lambda: P.rte_apply(p, x, y))
out["apply_f64_per_s"] = rate(lambda: P.rte_apply_f64(p, x64, y64))
P.rte_timing_enable(True)
P.rte_timing_reset()
P.rte_apply(p, x, y)
torch.cuda.synchronize()
c = [k for k in P.rte_timing_get() if k["name"] == "tfps_apply_f32"][0]
P.rte_timing_enable(False)
out["apply_f32_launch"] = {"ms": c["ms"], "algorithmic_flops": c["flops"], "algorithmic_bytes": c["bytes"],
                           "gflops": c["flops"] / (c["ms"] * 1e-3) / 1e9, "gbs": c["bytes"] / (c["ms"] * 1e-3) / 1e9}
b = torch.empty(p.shape, dtype=torch.float32, device="cuda")
P.rte_rhs(p, b)
cm = W.small_config(2, N=cfg.N, M=2 * cfg.M, n_polar=2, n_azim=32, L=cfg.L, C0=cfg.C0)
net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, W.make_weights(cm))
for name, nt in (("none", None), ("mgnet", net)):
    K = a.cycles * 30
    xs = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
    P.gmres_prepare(p, nt, restart=30, precond=1 if nt else 0)
    P.gmres_solve(p, nt, b, xs, restart=30, maxit=30, rtol=1e-300, x0_zero=True, history=False,
                  precond=1 if nt else 0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rep = P.gmres_solve(p, nt, b, xs, restart=30, maxit=K, rtol=1e-300, x0_zero=True, history=False,
                        precond=1 if nt else 0)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    out[f"gmres_{name}"] = {"iter_per_s": K / (ms * 1e-3), "inner_iterations": K, "ms": ms,
                            "relres_true_after": rep[0]["relres_true"]}
# ATFPS (NEXT-3b): the compressed system of the same problem at delta
pa = P.rte_setup_atfps(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                       delta=a.delta, n_polar=cfg.n_polar, n_azim=cfg.n_azim)
_, dim, _ = P.rte_atfps_info(pa)
out["atfps"] = {"delta": a.delta, "dimension": dim, "padded": pa.n, "compression": dim / pa.n,
                "apply_f32_per_s": rate(lambda: P.rte_apply(pa, x, y))}
ba = torch.empty(pa.shape, dtype=torch.float32, device="cuda")
P.rte_rhs(pa, ba)
neta = P.mgnet_create(pa, cfg.L, cfg.C0, cfg.nu, W.make_weights(cm))
for name, nt in (("none", None), ("mgnet", neta)):
    K = a.cycles * 30
    xs = torch.zeros(pa.shape, dtype=torch.float64, device="cuda")
    P.gmres_prepare(pa, nt, restart=30, precond=1 if nt else 0)
    P.gmres_solve(pa, nt, ba, xs, restart=30, maxit=30, rtol=1e-300, x0_zero=True, history=False,
                  precond=1 if nt else 0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rep = P.gmres_solve(pa, nt, ba, xs, restart=30, maxit=K, rtol=1e-300, x0_zero=True, history=False,
                        precond=1 if nt else 0)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    out["atfps"][f"gmres_{name}"] = {"iter_per_s": K / (ms * 1e-3), "inner_iterations": K, "ms": ms,
                                     "relres_true_after": rep[0]["relres_true"]}
print(json.dumps(out, indent=1))
