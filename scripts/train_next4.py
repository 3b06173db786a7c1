"""NEXT-4 measurement: train MgNet on the filtered loss loss_delta (paper_2604_23265_b200/train.py) and
compare GMRES(30) iteration counts to rtol 1e-8 with the trained weights against no preconditioner, block
Jacobi and the untrained network, on held-out media and sources (the protocol of PAPER.md:529-541 at a
desk scale; readings R43-R46).

Media (R46): 32 x 32 cells, 4 directions (the paper's discretisation), piecewise-constant
two-material media (sigma_T in {1, 6} on random 8 x 8 blocks -- the TFPS/ATFPS loss groups cells by
material, so the paper's polynomial media, where every cell is its own material, are out of reach of
this implementation), sigma_a = 0.3, the diffusion regime eps = 0.01 (c + 0.1), c ~ U[0, 1] per sample
(PAPER.md:521), g = 0.5, zero inflow; sources q ~ U[0, 1] per cell.  Everything runs on the GPU.

  python scripts/train_next4.py [--steps 400] [--out profiles/r02/train_next4.json]
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
from paper_2604_23265_b200 import train as TR  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=400)
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--test", type=int, default=10)
ap.add_argument("--delta", type=float, default=1e-4)
ap.add_argument("--out", default=None)
a = ap.parse_args()
N, NPOL, NAZ = 32, 1, 4
M = NPOL * NAZ
L, C0, NU = 4, 16, 2


def media(B, seed):
    rng = np.random.default_rng(seed)
    blk = rng.random((B, N // 8, N // 8)) < 0.5
    sT = np.where(np.kron(blk, np.ones((8, 8))) > 0, 6.0, 1.0).astype(np.float32)
    f = lambda v: np.full((B, N, N), v, np.float32)
    eps = (0.01 * (rng.uniform(0.0, 1.0, B) + 0.1)).astype(np.float32)
    return W.Media(sigma_T=sT, sigma_a=f(0.3), q=f(1.0), eps=np.broadcast_to(eps[:, None, None], (B, N, N)).copy(),
                   g=np.full(B, 0.5, np.float32), inflow=np.zeros((B, 4, N, M), np.float32))


t0 = time.time()
train_media = media(a.batch, 11)
val_q = [np.random.default_rng(100 + k).uniform(0, 1, (a.batch, N, N)).astype(np.float32) for k in range(4)]
out = TR.train(N, NPOL, NAZ, train_media, L=L, C0=C0, nu=NU, delta=a.delta, steps=a.steps, seed=0,
               eval_every=max(1, a.steps // 10), val_sources=val_q)
t_train = time.time() - t0
w_trained = out["weights"]
w_init = np.random.default_rng(0).normal(0.0, 0.02, TR.weight_count(M, L, C0, NU)).astype(np.float32)

# held-out test: new media and sources, the psi-space discrete-ordinates system (the hot path's operator)
tm = media(a.test, 23)
q = np.random.default_rng(24).uniform(0, 1, (a.test, N, N)).astype(np.float32)
p = P.rte_setup(N, tm.sigma_T, tm.sigma_a, q, tm.eps, tm.g, tm.inflow, n_polar=NPOL, n_azim=NAZ)
p2 = P.rte_setup_atfps(N, tm.sigma_T, tm.sigma_a, q, tm.eps, tm.g, tm.inflow, delta=a.delta, n_polar=NPOL,
                       n_azim=NAZ)
b = torch.empty(p.shape, dtype=torch.float32, device="cuda")
P.rte_rhs(p, b)
res = {}
for name, kw in (("none", dict(precond=0)), ("block_jacobi", dict(precond=2)),
                 ("mgnet_untrained", dict(w=w_init)), ("mgnet_trained", dict(w=w_trained))):
    net = None
    if "w" in kw:
        net = P.mgnet_create(p, L, C0, NU, kw["w"])
        z = torch.empty_like(b)
        P.mgnet_vcycle(net, b, z, add_identity=True)
        with torch.no_grad():
            ld = TR.loss_delta(z, p2)
        res[name + "_test_loss_delta"] = [float(v) for v in ld.cpu().numpy()]
    x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
    reps = P.gmres_solve(p, net, b, x, restart=30, maxit=3000, rtol=1e-8, x0_zero=True,
                         **({"precond": kw["precond"]} if "precond" in kw else {}))
    res[name] = [int(r["iterations"]) for r in reps]
    res[name + "_converged"] = [bool(r["converged"]) for r in reps]
    if name == "block_jacobi":
        # the loss floor: loss_delta of the converged upwind (psi-space) solution itself -- the gap between
        # the two discretisations (upwind DO vs ATFPS) that no network output can close
        with torch.no_grad():
            res["upwind_solution_test_loss_delta"] = [float(v) for v in
                                                      TR.loss_delta(x.float().contiguous(), p2).cpu().numpy()]
summary = {k: float(np.median(v)) for k, v in res.items() if not k.endswith(("_converged", "_loss_delta"))}
summary.update({k: float(np.median(v)) for k, v in res.items() if k.endswith("_loss_delta")})
report = {
    "what": "NEXT-4: MgNet trained on loss_delta (library-evaluated), GMRES(30) iterations to rtol 1e-8 on "
            "held-out media/sources (psi-space operator), median over test samples",
    "grid": f"{N}x{N}, {M} directions, L={L} C0={C0} nu={NU}, delta={a.delta}",
    "train": {"steps": a.steps, "batch": a.batch, "seconds": round(t_train, 1), "loss_first": out["loss"][0],
              "loss_last": out["loss"][-1], "val": out["val"], "lr_last": out["lr"][-1]},
    "median_iterations": summary,
    "per_sample": res,
}
s = json.dumps(report, indent=1)
print(s)
if a.out:
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    open(a.out, "w").write(s)
