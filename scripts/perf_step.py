"""Per-class device time of one GMRES(30) cycle on a config (experiments): every timing class the
library records, per GMRES iteration.  CFG=5 python scripts/perf_step.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_23265_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

cfg = W.config(int(os.environ.get("CFG", "5")))
K = int(os.environ.get("K", "30"))
media = W.make_media(cfg)
p = P.rte_setup(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                n_polar=cfg.n_polar, n_azim=cfg.n_azim)
net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, W.make_weights(cfg))
b = torch.empty((cfg.B, cfg.N, cfg.N, cfg.M), dtype=torch.float32, device="cuda")
P.rte_rhs(p, b)
x = torch.zeros(b.shape, dtype=torch.float64, device="cuda")
P.gmres_solve(p, net, b, x, restart=30, maxit=K, rtol=1e-300)
torch.cuda.synchronize()
P.rte_timing_enable(True)
P.rte_timing_reset()
x.zero_()
P.gmres_solve(p, net, b, x, restart=30, maxit=K, rtol=1e-300)
torch.cuda.synchronize()
rows = P.rte_timing_get()
tot = sum(r["ms"] for r in rows)
print(f"total {tot / K:.4f} ms per iteration over {K} iterations")
for r in sorted(rows, key=lambda r: -r["ms"]):
    print(f"  {r['name']:34s} {r['launches'] / K:6.1f} launches/it {r['ms'] / K:8.4f} ms/it")
