"""Round-2 diagnostics on the B200 (writes gpurun_out/diag_r2_*.npz / .json):
  1. per-operator parity margins: rte_apply and V(r) rel-L2 vs the fp64 oracle, configs 1-5, on the
     seeded random vector and on b (a smooth, physically shaped vector);
  2. GMRES (fp32 basis, the benchmarked mode) on configs 1-2: iteration counts, histories, x;
  3. fixed-budget GMRES on configs 3, 4, 5: residual histories and x (config 3 whole, configs 4-5 at
     seeded sample indices) for the off-box band comparison (scripts/make_bands.py)."""
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
from oracle import rte as O  # noqa: E402

OUT = os.path.join(ROOT, "gpurun_out")
os.makedirs(OUT, exist_ok=True)
which = sys.argv[1:] or ["ops", "conv", "budget"]


def rel(a, b):
    a = np.asarray(a, np.float64).ravel(); b = np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def setup(cfg):
    media = W.make_media(cfg)
    p = P.rte_setup(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                    n_polar=cfg.n_polar, n_azim=cfg.n_azim)
    return media, p


res = {}
if "ops" in which:
    for k in (1, 2, 3, 4, 5):
        t0 = time.time()
        cfg = W.config(k)
        media, p = setup(cfg)
        op = O.setup_from_media(cfg, media)
        w = W.make_weights(cfg)
        net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, w)
        onet = O.make_mgnet(w, cfg.M, cfg.L, cfg.C0, cfg.nu)
        bd = torch.empty(p.shape, dtype=torch.float32, device="cuda")
        P.rte_rhs(p, bd)
        nb = 1 if k != 4 else 2
        vecs = {"random": W.make_vector(cfg), "b": bd.cpu().numpy()}
        r = {}
        for name, v in vecs.items():
            vd = torch.from_numpy(np.ascontiguousarray(v)).cuda()
            y = torch.empty_like(vd)
            P.rte_apply(p, vd, y)
            z = torch.empty_like(vd)
            P.mgnet_vcycle(net, vd, z, add_identity=False)
            torch.cuda.synchronize()
            v64 = v[:nb].astype(np.float64)
            r[f"apply_{name}"] = rel(y[:nb].cpu().numpy(), O.apply(O.Problem(op.N, op.qd, op.sig_t[:nb], op.sig_s[:nb], op.f[:nb], op.S[:nb], op.inflow[:nb]), v64))
            r[f"vcycle_{name}"] = rel(z[:nb].cpu().numpy(), O.vcycle(onet, v64, add_identity=False))
        r["seconds"] = time.time() - t0
        res[f"cfg{k}"] = r
        print(k, r, flush=True)
    json.dump(res, open(os.path.join(OUT, "diag_r2_ops.json"), "w"), indent=1)

if "conv" in which:
    out = {}
    for k in (1, 2):
        cfg = W.config(k)
        media, p = setup(cfg)
        bd = torch.empty(p.shape, dtype=torch.float32, device="cuda")
        P.rte_rhs(p, bd)
        w = W.make_weights(cfg)
        net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, w)
        for precond in (0, 1):
            for reorth in (3, 0, 2):
                x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
                rep = P.gmres_solve(p, net if precond else None, bd, x, restart=30, maxit=cfg.maxit, rtol=cfg.rtol,
                                    reorth=reorth)[0]
                tag = f"cfg{k}_p{precond}_r{reorth}"
                print(tag, rep["iterations"], rep["relres_true"], flush=True)
                out[tag + "_it"] = rep["iterations"]
                out[tag + "_hist"] = rep["history"]
                out[tag + "_x"] = x.cpu().numpy()
    np.savez_compressed(os.path.join(OUT, "diag_r2_conv.npz"), **out)

if "conv2" in which:  # config 2 only, every mode
    out = {}
    cfg = W.config(2)
    media, p = setup(cfg)
    bd = torch.empty(p.shape, dtype=torch.float32, device="cuda")
    P.rte_rhs(p, bd)
    net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, W.make_weights(cfg))
    for precond in (0, 1):
        for reorth in (3, 0):
            x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
            rep = P.gmres_solve(p, net if precond else None, bd, x, restart=30, maxit=cfg.maxit, rtol=cfg.rtol,
                                reorth=reorth)[0]
            tag = f"cfg2_p{precond}_r{reorth}"
            print(tag, rep["iterations"], rep["relres_true"], flush=True)
            out[tag + "_it"] = rep["iterations"]
            out[tag + "_hist"] = rep["history"]
            out[tag + "_x"] = x.cpu().numpy()
    np.savez_compressed(os.path.join(OUT, "diag_r2_conv2.npz"), **out)

if "budget" in which:
    out = {}
    for k in (3, 4, 5):
        cfg = W.config(k)
        media, p = setup(cfg)
        bd = torch.empty(p.shape, dtype=torch.float32, device="cuda")
        P.rte_rhs(p, bd)
        w = W.make_weights(cfg)
        net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, w)
        x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
        reps = P.gmres_solve(p, net, bd, x, restart=30, maxit=cfg.maxit, rtol=cfg.rtol, hessenberg=True,
                             reorth=int(os.environ.get("DIAG_REORTH", "2")))
        for s, rep in enumerate(reps):
            out[f"cfg{k}_s{s}_hist"] = rep["history"]
            out[f"cfg{k}_s{s}_H"] = rep["hessenberg"]
            out[f"cfg{k}_s{s}_it"] = rep["iterations"]
        xs = x.cpu().numpy()
        out[f"cfg{k}_xnorm"] = np.linalg.norm(xs.reshape(cfg.B, -1), axis=1)
        if k == 3:
            out[f"cfg{k}_x"] = xs
        else:
            idx = W.sample_indices(cfg)
            out[f"cfg{k}_xs"] = xs.reshape(cfg.B, -1)[:, idx]
        print(k, [r["iterations"] for r in reps], [r["relres_true"] for r in reps], flush=True)
    np.savez_compressed(os.path.join(OUT, "diag_r2_budget.npz"), **out)
