"""NEXT-2 experiment: the paper's test protocol (Fig. 5 context) on the GPU path.

For every regime, 10 seeded test samples (32 x 32 cells, 4 directions, polynomial media of degree
`--degree`, random right-hand sides; R34) are solved by GMRES(30) to rtol 1e-8 with
  none | block Jacobi (R35) | MgNet (synthetic weights) | MgNet + CoeffNet (synthetic weights)
and the iteration counts and solve times are recorded.  The paper's MgNet column used TRAINED
weights, which are not released (training is NEXT-4), so the MgNet rows measure the machinery on
this workload, not the paper's claim.

  python scripts/paper_workload.py [--samples 10] [--degree 2] > profiles/r01_final/paper_workload.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_23265_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--samples", type=int, default=10)
ap.add_argument("--degree", type=int, default=2)
ap.add_argument("--rtol", type=float, default=1e-8)
ap.add_argument("--maxit", type=int, default=3000)
ap.add_argument("--precision", type=int, default=1,
                help="Krylov basis: 1 fp64 (default: the mode whose iteration counts are parity-tested "
                     "+-1 against the oracle, tests/test_gpu_blockjacobi.py), 0 fp32")
args = ap.parse_args()

N, NP, NA, L, C0, NU = 32, 1, 4, 4, 16, 2
M = NP * NA
cfg_like = W.small_config(1, N=N, M=M, n_polar=NP, n_azim=NA, L=L, C0=C0)
weights = W.make_weights(cfg_like, std=0.02, seed=77)
cweights = W.make_coeffnet_weights(cfg_like, seed=78)
out = {"grid": f"{N}x{N}", "directions": M, "precision": args.precision, "mgnet": {"L": L, "C0": C0, "nu": NU}, "rtol": args.rtol,
       "restart": 30, "samples": args.samples, "degree": args.degree, "regimes": {}}
for regime in W.PAPER_REGIMES:
    med = W.paper_media(args.samples, N=N, degree=args.degree, regime=regime, M=M, seed=100)
    b = torch.from_numpy(W.make_paper_rhs(args.samples, N=N, M=M, seed=100)).cuda()
    p = P.rte_setup(N, med.sigma_T, med.sigma_a, med.q, med.eps, med.g, med.inflow, n_polar=NP, n_azim=NA)
    net = P.mgnet_create(p, L, C0, NU, weights)
    netc = P.mgnet_create(p, L, C0, NU, weights)
    P.mgnet_coeffnet(netc, med.sigma_T, med.sigma_a, med.eps, cweights)
    res = {}
    for name, pre, nt in (("none", 0, None), ("block_jacobi", 2, None), ("mgnet", 1, net), ("mgnet_coeffnet", 1, netc)):
        x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
        P.gmres_solve(p, nt, b, x, restart=30, maxit=5, rtol=args.rtol, precond=pre,
                      precision=args.precision)  # warm-up
        x.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = P.gmres_solve(p, nt, b, x, restart=30, maxit=args.maxit, rtol=args.rtol, precond=pre,
                            precision=args.precision)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        its = [r["iterations"] for r in rep]
        res[name] = {"iterations": its, "median": float(np.median(its)), "converged": sum(r["converged"] for r in rep),
                     "ms_per_batch_solve": round(dt * 1e3, 2), "max_relres_true": max(r["relres_true"] for r in rep)}
    out["regimes"][regime] = res
    print(regime, {k: (v["median"], v["converged"]) for k, v in res.items()}, file=sys.stderr)
print(json.dumps(out, indent=1))
