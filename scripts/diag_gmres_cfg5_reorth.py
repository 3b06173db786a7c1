"""Does selective re-orthogonalisation change the Arnoldi process on config 5?  Runs one GMRES(30)
cycle with CGS2 and with the selective (DGKS) rule and compares the estimates (experiments)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_23265_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

for k in (5, 3):
    cfg = W.config(k)
    media = W.make_media(cfg)
    p = P.rte_setup(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                    n_polar=cfg.n_polar, n_azim=cfg.n_azim)
    net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, W.make_weights(cfg))
    b = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    P.rte_rhs(p, b)
    out = {}
    for r in (0, 2, 1):
        x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
        rep = P.gmres_solve(p, net, b, x, restart=30, maxit=30 if k == 5 else 90, rtol=1e-300, reorth=r)[0]
        out[r] = np.array(rep["history"])
        print(f"cfg{k} reorth={r}: relres_true={rep['relres_true']:.6e} est_last={rep['relres_est']:.6e}", flush=True)
    print(f"cfg{k} max |est(2)/est(0) - 1| = {np.max(np.abs(out[2] / out[0] - 1)):.3e}, "
          f"|est(1)/est(0) - 1| = {np.max(np.abs(out[1] / out[0] - 1)):.3e}", flush=True)
