"""Perturbed-oracle bands for the GMRES parity protocol (SURVEY.md §8(c) "GMRES parity protocol";
DESIGN.md §6).  Calls only oracle/ and workloads/ -- never the CUDA path.

For a config it runs the fp64 oracle GMRES (x0 = 0, restart 30, the config's rtol and budget, MgNet
preconditioner with the config's seeded weights) on the fp32-rounded rhs -- the reference run --
and K = 4 perturbed runs.  Run k perturbs, with its own seeded noise xi ~ N(0, 1) per element,
  * the rhs:                b_k = b (1 + 6e-8 xi)              (the fp32 rounding
                                                               of b)
  * every operator output:  A_k(v) = A(v) (1 + d_A xi)         (an fp32 apply's per-op error)
  * every V-cycle output:   P_k(v) = v + V(v) (1 + d_V xi)     (the correction V(v) = z - v carries
                                                               the fp32 V-cycle's error, R27)
d = d_A = d_V (--delta) is the per-op relative error of an fp32 implementation of the operators
(reading R36).  The band of a quantity is the max deviation of the 4 perturbed runs
from the reference run; the GPU must lie within 2x that band (tests/test_gpu_bands.py).

Stored per config (tests/golden/bands_cfg{k}.npz): the reference histories and iteration counts
per sample, the reference x at workloads.sample_indices(cfg) (all of x for small configs), the
perturbed runs' histories / counts / sampled x, and the band values.

  python scripts/make_bands.py 2 3 4 5   [--runs 4] [--samples 0,1,...]
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


def run(cfg, s, b32, op_s, onet, k, delta):
    """Reference run (k < 0) or perturbed run k of sample s."""
    A = lambda v: O.apply(op_s, v)
    V = lambda v: O.vcycle(onet, v, add_identity=False)
    b = b32
    if k >= 0:
        rng = np.random.Generator(np.random.PCG64([5000 + cfg.k, s, k]))
        b = b32 * (1.0 + D_B * rng.standard_normal(b32.shape))
        A = noisy(A, delta, rng)
        V = noisy(V, delta, rng)
    P = lambda v: v + V(v)
    return O.gmres(A, b, P=P, restart=cfg.restart, rtol=cfg.rtol, maxit=cfg.maxit)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", type=int, nargs="+")
    ap.add_argument("--runs", type=int, default=4)
    ap.add_argument("--samples", type=str, default=None)
    ap.add_argument("--delta", type=float, default=D_OP)
    args = ap.parse_args()
    os.makedirs(TMP, exist_ok=True)
    for k in args.configs:
        cfg = W.config(k)
        media = W.make_media(cfg)
        op = O.setup_from_media(cfg, media)
        onet = O.make_mgnet(W.make_weights(cfg), cfg.M, cfg.L, cfg.C0, cfg.nu)
        b32_all = O.rhs(op).astype(np.float32).astype(np.float64)   # the GPU solves the fp32 b
        idx = W.sample_indices(cfg)
        samples = range(cfg.B) if args.samples is None else [int(t) for t in args.samples.split(",")]
        for s in samples:
            op_s = O.Problem(op.N, op.qd, op.sig_t[s:s + 1], op.sig_s[s:s + 1], op.f[s:s + 1], op.S[s:s + 1],
                             op.inflow[s:s + 1])
            b32 = b32_all[s:s + 1]
            for r in [-1] + list(range(args.runs)):
                path = _path(k, s, r, args.delta)
                if os.path.exists(path):
                    continue
                t0 = time.time()
                res = run(cfg, s, b32, op_s, onet, r, args.delta)
                x = res.x.ravel()
                np.savez(path, hist=np.array(res.history), it=res.iterations, conv=res.converged,
                         relres=res.relres_true, xs=x[idx], xnorm=np.linalg.norm(x))
                print(f"cfg{k} s{s} run{r}: {res.iterations} it, conv {res.converged}, relres {res.relres_true:.3e}, "
                      f"{time.time() - t0:.0f} s", flush=True)
        if args.runs > 0:
            assemble(cfg, samples, args.runs, args.delta)


def _path(k, s, r, delta):
    return os.path.join(TMP, f"cfg{k}_s{s}_r{r}.npz" if r < 0 else f"cfg{k}_s{s}_r{r}_d{delta:.0e}.npz")


def assemble(cfg, samples, runs, delta):
    out = {"d_b": D_B, "d_op": delta, "runs": runs}
    idx = W.sample_indices(cfg)
    sub = lambda xs: xs if xs.size == idx.size else xs.ravel()[idx]   # (older files kept all of x)
    for s in samples:
        ref = np.load(_path(cfg.k, s, -1, delta))
        for key in ("hist", "it", "conv", "relres", "xnorm"):
            out[f"s{s}_ref_{key}"] = ref[key]
        out[f"s{s}_ref_xs"] = sub(ref["xs"])
        dh, dx, dit = [], [], []
        for r in range(runs):
            d = np.load(_path(cfg.k, s, r, delta))
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
              f"x {max(dx):.3e} it {max(dit)} (runs: {[int(np.load(_path(cfg.k, s, r, delta))['it']) for r in range(runs)]})",
              flush=True)
    os.makedirs(os.path.join(ROOT, "tests", "golden"), exist_ok=True)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", f"bands_cfg{cfg.k}.npz"), **out)


if __name__ == "__main__":
    main()
