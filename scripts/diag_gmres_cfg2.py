"""Diagnostic: dump the GPU GMRES residual history for config 2 (unpreconditioned and MgNet) so it
can be compared with the oracle's history off-box (where do the curves separate?)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_23265_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

cfg = W.config(2)
media = W.make_media(cfg)
p = P.rte_setup(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                n_polar=cfg.n_polar, n_azim=cfg.n_azim)
b = torch.empty(p.shape, dtype=torch.float32, device="cuda")
P.rte_rhs(p, b)
out = {}
for precond in (0, 1):
    net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, W.make_weights(cfg)) if precond else None
    for reorth in (0,):
        x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
        rep = P.gmres_solve(p, net, b, x, restart=30, maxit=3000, rtol=1e-6, reorth=reorth)[0]
        print(precond, reorth, rep["iterations"], rep["relres_true"], flush=True)
        out[f"hist_p{precond}_r{reorth}"] = rep["history"]
        out[f"x_p{precond}_r{reorth}"] = x.cpu().numpy()
os.makedirs("gpurun_out", exist_ok=True)
np.savez_compressed("gpurun_out/diag_cfg2.npz", **out)
