"""fp32-storage runs for the GMRES parity bands (reading R36 v3; oracle-only, never the CUDA
path): the benchmarked path's own Gram-Schmidt (DCGS2, the formulas of krylov.cu as restated in
scripts/emulate_fp32_gmres.py) on the ORACLE's operator and MgNet preconditioner, with the Krylov basis,
the preconditioner output z = P q and the operator output w = A z stored in float32, dots in float64 and
updates in float32 with float32 coefficients -- the storage precision of the GPU path -- right-
preconditioned, x0 = 0, the config's restart and fixed budget.  Its deviation from the fp64 MGS reference
run (tests/golden/bands_cfg{k}.npz) is added to the band file as s{s}_band_fp32_hist / s{s}_band_fp32_x.

  python scripts/make_bands_fp32.py 3 4 5 [--samples 0,3]

--op-tol E (reading R36 v5): the same fp32-storage run on operators that each carry a fixed relative
error of the north star's single-operator tolerance E = 1e-5 -- z = q + (1 + E xi_V) (.) V(q) and
w = (1 + E xi_A) (.) A z with xi_V, xi_A ~ N(0,1) per unknown, drawn once per (config, sample) from a
seeded generator and kept for the whole solve (a fixed nearby linear operator, not per-call noise: that
averages out of the history, R36) -- i.e. an implementation whose every V-cycle and apply is within 1e-5
rel-L2 of the oracle's, which is all the north star asks of one.  Stored as s{s}_band_op_hist / _x.
--coherent: the coherent error of that size instead, z = q + (1 - E) V(q) (s{s}_band_opc_hist / _x).
"""
from __future__ import annotations

import argparse
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from oracle import rte as O  # noqa: E402

f32 = np.float32


def d64(a, c):
    return float(np.dot(a.astype(np.float64), c.astype(np.float64)))


def gmres_dcgs2_fp32(A, P, b, restart, maxit, rtol):
    """Right-preconditioned GMRES(restart) with DCGS2 on fp32 storage; returns (history, x)."""
    n = b.size
    x = np.zeros(n)
    bn = np.linalg.norm(b)
    hist = []
    total = 0
    r = b.copy()
    while True:
        beta = np.linalg.norm(r)
        if beta <= rtol * bn or total >= maxit:
            return np.array(hist), x
        V = np.zeros((restart + 1, n), f32)
        al = np.zeros(restart + 1)
        H = np.zeros((restart + 1, restart))
        V[0] = r.astype(f32)
        al[0] = 1 / beta
        cs = np.zeros(restart)
        sn = np.zeros(restart)
        g = np.zeros(restart + 1)
        g[0] = beta
        a_prev = None
        k = 0
        for j in range(restart):
            w = A(P((al[j] * V[j].astype(np.float64)).astype(f32)))
            at = al[j]
            z = np.array([al[i] * d64(V[i], w) for i in range(j + 1)])
            s = a_prev[:j] * at if j > 0 else np.zeros(0)
            r_ = math.sqrt(max(1 - float(np.sum(s * s)), 1e-300))
            if j > 0:
                hl = H[j, j - 1]
                H[:j, j - 1] += hl * s
                H[j, j - 1] = hl * r_
            c = np.array([sum(H[i, kk] * s[kk] for kk in range(j)) for i in range(j + 1)])
            sz = float(np.dot(s, z[:j])) if j > 0 else 0.0
            h = np.zeros(j + 1)
            h[:j] = (z[:j] - c[:j]) / r_
            h[j] = ((z[j] - sz) / r_ - c[j]) / r_
            d = c + r_ * h
            cA = (s * al[:j] / at).astype(f32)
            cB = np.zeros(j + 1)
            cB[:j] = (d[:j] - d[j] * s / r_) * al[:j]
            cB[j] = d[j] * at / r_
            cB = cB.astype(f32)
            vj = V[j].copy()
            wn = (w - cB[j] * vj).astype(f32)
            for i in range(j):
                vj = (vj - cA[i] * V[i]).astype(f32)
                wn = (wn - cB[i] * V[i]).astype(f32)
            V[j] = vj
            al[j] = at / r_
            a_prev = np.array([al[i] * d64(V[i], wn) for i in range(j + 1)])
            n2 = d64(wn, wn)
            V[j + 1] = wn
            al[j + 1] = 1 / math.sqrt(n2)
            col = h
            hj1 = math.sqrt(n2) / r_
            H[:j + 1, j] = h
            H[j + 1, j] = hj1
            cc = col.copy()
            for i in range(j):
                t = cs[i] * cc[i] + sn[i] * cc[i + 1]
                cc[i + 1] = -sn[i] * cc[i] + cs[i] * cc[i + 1]
                cc[i] = t
            den = math.hypot(cc[j], hj1)
            cs[j] = cc[j] / den
            sn[j] = hj1 / den
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            k = j + 1
            hist.append(abs(g[j + 1]) / bn)
            if abs(g[j + 1]) <= rtol * bn or total >= maxit:
                break
        at = al[k]
        s = a_prev[:k] * at
        r_ = math.sqrt(max(1 - float(np.sum(s * s)), 1e-300))
        hl = H[k, k - 1]
        H[:k, k - 1] += hl * s
        H[k, k - 1] = hl * r_
        e = np.zeros(k + 1)
        e[0] = beta
        y = np.linalg.lstsq(H[:k + 1, :k], e, rcond=None)[0]
        Q = V[:k].astype(np.float64) * al[:k, None]
        x = x + P(Q.T @ y).astype(np.float64)
        r = b - O_apply64(x)  # the fp64 restart residual (krylov.cu: apply_f64)
        if total >= maxit:
            return np.array(hist), x


def main():
    global O_apply64
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", type=int, nargs="+")
    ap.add_argument("--samples", type=str, default=None)
    ap.add_argument("--op-tol", type=float, default=0.0)
    ap.add_argument("--coherent", action="store_true")
    a = ap.parse_args()
    for k in a.configs:
        cfg = W.config(k)
        media = W.make_media(cfg)
        op = O.setup_from_media(cfg, media)
        onet = O.make_mgnet(W.make_weights(cfg), cfg.M, cfg.L, cfg.C0, cfg.nu)
        b32_all = O.rhs(op).astype(np.float32).astype(np.float64)
        idx = W.sample_indices(cfg)
        path = os.path.join(ROOT, "tests", "golden", f"bands_cfg{k}.npz")
        g = dict(np.load(path))
        samples = sorted({int(key.split("_")[0][1:]) for key in g if key.startswith("s") and "_ref_" in key})
        if a.samples:
            samples = [s for s in samples if s in {int(t) for t in a.samples.split(",")}]
        for s in samples:
            op_s = O.Problem(op.N, op.qd, op.sig_t[s:s + 1], op.sig_s[s:s + 1], op.f[s:s + 1], op.S[s:s + 1],
                             op.inflow[s:s + 1])
            shape = (1, cfg.N, cfg.N, cfg.M)
            A = lambda v: O.apply(op_s, np.asarray(v, np.float64).reshape(shape)).ravel().astype(f32)
            P = lambda v: (np.asarray(v, np.float64) + O.vcycle(onet, np.asarray(v, np.float64).reshape(shape),
                                                                 add_identity=False).ravel()).astype(f32)
            O_apply64 = lambda x: O.apply(op_s, x.reshape(shape)).ravel()
            tag = "fp32"
            if a.op_tol > 0.0:
                tag = "op"
                rng = np.random.Generator(np.random.PCG64([5000 + k, s]))
                dV = (1.0 + a.op_tol * rng.standard_normal(int(np.prod(shape)))).astype(np.float64)
                dA = (1.0 + a.op_tol * rng.standard_normal(int(np.prod(shape)))).astype(np.float64)
                if a.coherent:
                    # the coherent error of the same size: V(q) scaled by (1 - E) everywhere -- the shape of a
                    # rounding *bias* (the tensor core's fp32 accumulation truncates, DESIGN.md §6 numerics 1),
                    # which, unlike a random field, does not average out of the Arnoldi inner products.  (The
                    # same scaling of A leaves the residual history unchanged: the Krylov space is the same.)
                    tag = "opc"
                    dV = 1.0 - a.op_tol
                    dA = 1.0
                A = lambda v, dA=dA: (dA * O.apply(op_s, np.asarray(v, np.float64).reshape(shape)).ravel()).astype(f32)
                P = lambda v, dV=dV: (np.asarray(v, np.float64) + dV * O.vcycle(
                    onet, np.asarray(v, np.float64).reshape(shape), add_identity=False).ravel()).astype(f32)
            b = b32_all[s:s + 1].ravel()
            t0 = time.time()
            hist, x = gmres_dcgs2_fp32(A, P, b, cfg.restart, cfg.maxit, cfg.rtol)
            ref = g[f"s{s}_ref_hist"]
            n = min(len(hist), len(ref))
            dh = float(np.max(np.abs(hist[:n] - ref[:n]) / ref[:n]))
            xs = x[idx]
            dx = float(np.linalg.norm(xs - g[f"s{s}_ref_xs"]) / np.linalg.norm(g[f"s{s}_ref_xs"]))
            g[f"s{s}_{tag}_hist"] = hist
            g[f"s{s}_{tag}_xs"] = xs
            g[f"s{s}_band_{tag}_hist"] = dh
            g[f"s{s}_band_{tag}_x"] = dx
            if tag in ("op", "opc"):
                g["op_tol"] = a.op_tol
            print(f"cfg{k} s{s}: fp32-storage DCGS2 run{' + operators at ' + str(a.op_tol) + ' (' + tag + ')' if tag != 'fp32' else ''}, "
                  f"{len(hist)} it, history dev {dh:.3e}, x dev {dx:.3e}, {time.time() - t0:.0f} s", flush=True)
        np.savez_compressed(path, **g)


O_apply64 = None

if __name__ == "__main__":
    main()
