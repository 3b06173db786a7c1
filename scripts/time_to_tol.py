"""Time-to-tolerance (BASELINE.json north star: "GMRES iterations/s, time-to-tolerance"): the full
MgNet-preconditioned GMRES(30) solve from x0 = 0 to the config's rtol on the converging configs 1
and 2, on the B200 (device buffers; and end to end through gmres_solve_host) and with the fp64
oracle on the host cores (a baseline, not the target).  Configs 3-5 run their fixed budgets and
report the residual reached ("not reached at budget").  Writes one JSON object to stdout.

  python scripts/time_to_tol.py [--no-oracle] [--configs 1,2,3,4,5] [--reorth 3]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_23265_b200 as P  # noqa: E402
import workloads as W  # noqa: E402


def gpu_solve(cfg, reorth, reps=3):
    media = W.make_media(cfg)
    p = P.rte_setup(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                    n_polar=cfg.n_polar, n_azim=cfg.n_azim)
    net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, W.make_weights(cfg))
    b = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    P.rte_rhs(p, b)
    x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
    P.gmres_prepare(p, net, restart=cfg.restart, reorth=reorth)
    kw = dict(restart=cfg.restart, maxit=cfg.maxit, rtol=cfg.rtol, reorth=reorth, x0_zero=True, history=False)
    P.gmres_solve(p, net, b, x, **kw)  # warm-up (graphs, lazy allocations)
    torch.cuda.synchronize()
    best, rep = None, None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rep = P.gmres_solve(p, net, b, x, **kw)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    bh = b.cpu().pin_memory()
    xh = torch.zeros(p.shape, dtype=torch.float64).pin_memory()
    P.gmres_solve_host(p, net, bh, xh, **kw)
    t0 = time.perf_counter()
    P.gmres_solve_host(p, net, bh, xh, **kw)
    e2e_ms = (time.perf_counter() - t0) * 1e3
    return {"ms": best, "e2e_ms_wall": e2e_ms, "iterations": [r["iterations"] for r in rep],
            "converged": [bool(r["converged"]) for r in rep], "relres_true": [r["relres_true"] for r in rep],
            "iter_per_s": sum(r["iterations"] for r in rep) / len(rep) / (best * 1e-3)}


def oracle_solve(cfg):
    from oracle import rte as O
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    media = W.make_media(cfg)
    op = O.setup_from_media(cfg, media)
    onet = O.make_mgnet(W.make_weights(cfg), cfg.M, cfg.L, cfg.C0, cfg.nu)
    b = O.rhs(op).astype(np.float32).astype(np.float64)
    t0 = time.perf_counter()
    res = O.gmres(lambda v: O.apply(op, v), b, P=lambda v: O.vcycle(onet, v), restart=cfg.restart,
                  rtol=cfg.rtol, maxit=cfg.maxit)
    dt = time.perf_counter() - t0
    return {"s": dt, "iterations": res.iterations, "converged": res.converged, "relres_true": res.relres_true,
            "cores": cores, "host_cpus": os.cpu_count()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("--reorth", type=int, default=3)
    args = ap.parse_args()
    out = {"reorth": args.reorth, "gpu": torch.cuda.get_device_name(0)}
    for k in [int(t) for t in args.configs.split(",")]:
        cfg = W.config(k)
        d = {"budget": cfg.maxit, "rtol": cfg.rtol, "fixed_budget": cfg.fixed_budget, "gpu": gpu_solve(cfg, args.reorth)}
        if not args.no_oracle and k <= 2:
            d["oracle"] = oracle_solve(cfg)
        out[f"cfg{k}"] = d
        print(k, json.dumps(d), file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
