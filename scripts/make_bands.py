"""Perturbed-oracle bands for the GMRES parity protocol (SURVEY.md §8(c) "GMRES parity protocol";
DESIGN.md §6, reading R36).  Calls only oracle/ and workloads/ -- never the CUDA path.

For a config it runs the fp64 oracle GMRES (x0 = 0, restart 30, the config's rtol and budget, MgNet
preconditioner with the config's seeded weights) on the fp32-rounded rhs -- the reference run --
and K = 4 perturbed runs.  Run k solves a fixed nearby problem, with its own seeded N(0, 1) noise xi
per element (model "input", the default):
  * the rhs            b_k = b (1 + 6e-8 xi)
  * the medium          sigma_T, sigma_a, eps (1 + d xi) per cell, g (1 + d xi) per sample
  * the MgNet weights   w (1 + d xi)
with d = --delta (1e-6): an operator that differs from the reference one by a consistent relative
error of the order of an fp32 implementation's per-operator error -- the way fp32 rounding of
coefficients and fixed-order accumulations perturb the GPU's operator, the same at every application.
(Model "iid" perturbs every operator output independently at every call instead; measured on configs
4-5 it averages out in the residual history -- bands of 4e-10..7e-8 -- and does not represent a
systematic rounding error; kept for the record.)  The band of a quantity is the max deviation of the
4 perturbed runs from the reference run; the GPU must lie within 2x that band (tests/test_gpu_bands.py).

Stored per config (tests/golden/bands_cfg{k}.npz): the reference histories and iteration counts
per sample, the reference x at workloads.sample_indices(cfg), the perturbed runs' histories and
counts, and the band values.

  python scripts/make_bands.py 3 4 5 [--runs 4] [--samples 0,1,...] [--delta 1e-6] [--model input]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from oracle import rte as O  # noqa: E402

D_B = 6e-8
D_OP = 2e-6   # default per-op relative perturbation of A and V (--delta)
TMP = os.environ.get("BANDS_TMP", "/tmp/bands")


def noisy(fn, delta, rng):
    def g(v):
        y = fn(v)
        return y * (1.0 + delta * rng.standard_normal(y.shape))
    return g


def run(cfg, s, b32, op_s, onet, k, delta, model="input", media=None, weights=None):
    """Reference run (k < 0) or perturbed run k of sample s."""
    A = lambda v: O.apply(op_s, v)
    V = lambda v: O.vcycle(onet, v, add_identity=False)
    b = b32
    if k >= 0 and model == "iid":
        rng = np.random.Generator(np.random.PCG64([5000 + cfg.k, s, k]))
        b = b32 * (1.0 + D_B * rng.standard_normal(b32.shape))
        A = noisy(A, delta, rng)
        V = noisy(V, delta, rng)
    elif k >= 0:
        rng = np.random.Generator(np.random.PCG64([5100 + cfg.k, s, k]))
        b = b32 * (1.0 + D_B * rng.standard_normal(b32.shape))
        pert = lambda a: np.asarray(a, np.float64) * (1.0 + delta * rng.standard_normal(np.shape(a)))
        sl = slice(s, s + 1)
        opk = O.setup(cfg.N, cfg.n_polar, cfg.n_azim, pert(media.sigma_T[sl]), pert(media.sigma_a[sl]),
                      media.q[sl], pert(media.eps[sl]), pert(media.g[sl]), media.inflow[sl])
        onk = O.make_mgnet(pert(weights), cfg.M, cfg.L, cfg.C0, cfg.nu)
        A = lambda v: O.apply(opk, v)
        V = lambda v: O.vcycle(onk, v, add_identity=False)
    P = lambda v: v + V(v)
    return O.gmres(A, b, P=P, restart=cfg.restart, rtol=cfg.rtol, maxit=cfg.maxit)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", type=int, nargs="+")
    ap.add_argument("--runs", type=int, default=4)
    ap.add_argument("--samples", type=str, default=None)
    ap.add_argument("--delta", type=float, default=D_OP)
    ap.add_argument("--model", choices=["input", "iid"], default="input")
    args = ap.parse_args()
    os.makedirs(TMP, exist_ok=True)
    for k in args.configs:
        cfg = W.config(k)
        media = W.make_media(cfg)
        op = O.setup_from_media(cfg, media)
        weights = W.make_weights(cfg)
        onet = O.make_mgnet(weights, cfg.M, cfg.L, cfg.C0, cfg.nu)
        b32_all = O.rhs(op).astype(np.float32).astype(np.float64)   # the GPU solves the fp32 b
        idx = W.sample_indices(cfg)
        samples = range(cfg.B) if args.samples is None else [int(t) for t in args.samples.split(",")]
        for s in samples:
            op_s = O.Problem(op.N, op.qd, op.sig_t[s:s + 1], op.sig_s[s:s + 1], op.f[s:s + 1], op.S[s:s + 1],
                             op.inflow[s:s + 1])
            b32 = b32_all[s:s + 1]
            for r in [-1] + list(range(args.runs)):
                path = _path(k, s, r, args.delta, args.model)
                if os.path.exists(path):
                    continue
                t0 = time.time()
                res = run(cfg, s, b32, op_s, onet, r, args.delta, args.model, media, weights)
                x = res.x.ravel()
                np.savez(path, hist=np.array(res.history), it=res.iterations, conv=res.converged,
                         relres=res.relres_true, xs=x[idx], xnorm=np.linalg.norm(x))
                print(f"cfg{k} s{s} run{r}: {res.iterations} it, conv {res.converged}, relres {res.relres_true:.3e}, "
                      f"{time.time() - t0:.0f} s", flush=True)
        if args.runs > 0:
            assemble(cfg, samples, args.runs, args.delta, args.model)


def _path(k, s, r, delta, model="input"):
    if r < 0:
        return os.path.join(TMP, f"cfg{k}_s{s}_r{r}.npz")
    tag = "" if model == "iid" else "_in"
    return os.path.join(TMP, f"cfg{k}_s{s}_r{r}_d{delta:.0e}{tag}.npz")


def assemble(cfg, samples, runs, delta, model="input"):
    out = {"d_b": D_B, "delta": delta, "model": model, "runs": runs}
    idx = W.sample_indices(cfg)
    sub = lambda xs: xs if xs.size == idx.size else xs.ravel()[idx]   # (older files kept all of x)
    for s in samples:
        ref = np.load(_path(cfg.k, s, -1, delta, model))
        for key in ("hist", "it", "conv", "relres", "xnorm"):
            out[f"s{s}_ref_{key}"] = ref[key]
        out[f"s{s}_ref_xs"] = sub(ref["xs"])
        dh, dx, dit = [], [], []
        for r in range(runs):
            d = np.load(_path(cfg.k, s, r, delta, model))
            n = min(len(d["hist"]), len(ref["hist"]))
            dh.append(float(np.max(np.abs(d["hist"][:n] - ref["hist"][:n]) / ref["hist"][:n])))
            dx.append(float(np.linalg.norm(sub(d["xs"]) - sub(ref["xs"])) / np.linalg.norm(sub(ref["xs"]))))
            dit.append(int(abs(int(d["it"]) - int(ref["it"]))))
            out[f"s{s}_run{r}_it"] = d["it"]
            out[f"s{s}_run{r}_hist"] = d["hist"]
        out[f"s{s}_band_hist"] = max(dh)
        out[f"s{s}_band_x"] = max(dx)
        out[f"s{s}_band_it"] = max(dit)
        print(f"cfg{cfg.k} s{s}: ref it {int(ref['it'])} conv {bool(ref['conv'])}; band hist {max(dh):.3e} "
              f"x {max(dx):.3e} it {max(dit)} (runs: {[int(np.load(_path(cfg.k, s, r, delta, model))['it']) for r in range(runs)]})",
              flush=True)
    os.makedirs(os.path.join(ROOT, "tests", "golden"), exist_ok=True)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", f"bands_cfg{cfg.k}.npz"), **out)


if __name__ == "__main__":
    main()
