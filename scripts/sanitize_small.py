"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): every kernel
family of the hot path at a size that finishes in seconds under instrumentation --
  * tcgen05 GEMMs: the apply (M = 64, N-tile 64) and every MgNet conv class (C0 = 32: the two-CTA-per-SM
    N = 32/64 plans and the one-CTA N = 128 plans, split-K reduction, strided/transposed convs, lift/head);
  * the SIMT apply (M = 16), the fp64 DMMA apply (M = 64) and fp64 V-cycle;
  * the Krylov kernels: GMRES with CGS2, selective and DCGS2 Gram-Schmidt, fp32 and fp64 bases.
  compute-sanitizer --tool racecheck python scripts/sanitize_small.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_23265_b200 as P  # noqa: E402
import workloads as W  # noqa: E402


def run(cfg, reorths=(0, 2, 3), precisions=(0, 1)):
    media = W.make_media(cfg)
    p = P.rte_setup(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                    n_polar=cfg.n_polar, n_azim=cfg.n_azim)
    net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, W.make_weights(cfg, std=0.05))
    b = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    P.rte_rhs(p, b)
    y = torch.empty_like(b)
    P.rte_apply(p, b, y)
    P.mgnet_vcycle(net, b, y, add_identity=True)
    b64 = b.double()
    y64 = torch.empty_like(b64)
    P.rte_apply_f64(p, b64, y64)
    P.mgnet_vcycle_f64(net, b64, y64, add_identity=True)
    for precision in precisions:
        for reorth in reorths:
            x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
            rep = P.gmres_solve(p, net, b, x, restart=6, maxit=8, rtol=1e-30, reorth=reorth, precision=precision,
                                x0_zero=True)
            assert all(r["iterations"] == 8 for r in rep)
    torch.cuda.synchronize()
    print("ok", cfg.N, cfg.M, cfg.L, cfg.C0, flush=True)


run(W.small_config(5, N=32, M=64, n_polar=4, n_azim=16, L=3, C0=32))          # tcgen05 apply + convs
run(W.small_config(4, N=16, M=16, n_polar=2, n_azim=8, L=2, C0=16, B=2), precisions=(0,))  # SIMT paths, batch
print("sanitize_small done")
