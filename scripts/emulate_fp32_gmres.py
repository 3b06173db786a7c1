"""fp32-storage emulation of the GPU path's GMRES on the ORACLE's operator (oracle-only; no CUDA):
restarted GMRES(30) with the Krylov basis and every operator output stored in float32, dots in float64,
updates in float32 with float32 coefficients -- CGS2 (reorth 0) and DCGS2 (reorth 3, the same
formulas as krylov.cu's dcgs_coef_kernel / dcgs_update_kernel / dcgs_backsolve_kernel) -- against the
fp64 MGS oracle (1290 iterations), on config 2 unpreconditioned.  It measures how far fp32 storage
alone moves the iteration count of this diffusive solve.

  python scripts/emulate_fp32_gmres.py dcgs2 cgs2  > profiles/r02/emulate_fp32_gmres.json
"""
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle.rte as O, workloads as W
cfg = W.config(2); media = W.make_media(cfg); op = O.setup_from_media(cfg, media)
b = O.rhs(op).astype(np.float32).astype(np.float64).ravel()
f32 = np.float32
d64 = lambda a, c: float(np.dot(a.astype(np.float64), c.astype(np.float64)))


def A(v):
    return O.apply(op, v.reshape(op.shape)).ravel().astype(f32)


def gmres(mode, restart=30, rtol=1e-6, maxit=3000):
    n = b.size; x = np.zeros(n); bn = np.linalg.norm(b); total = 0
    while True:
        r = b - O.apply(op, x.reshape(op.shape)).ravel(); beta = np.linalg.norm(r)
        if beta <= rtol * bn or total >= maxit:
            return total, beta / bn
        V = np.zeros((restart + 1, n), f32); al = np.zeros(restart + 1); H = np.zeros((restart + 1, restart))
        V[0] = r.astype(f32); al[0] = 1 / beta
        cs = np.zeros(restart); sn = np.zeros(restart); g = np.zeros(restart + 1); g[0] = beta
        a_prev = None; k = 0
        for j in range(restart):
            w = A((al[j] * V[j].astype(np.float64)).astype(f32))
            if mode == 'cgs2':
                h1 = np.array([al[i] * d64(V[i], w) for i in range(j + 1)])
                c = (h1 * al[:j + 1]).astype(f32); v = w.copy()
                for i in range(j + 1): v = (v - c[i] * V[i]).astype(f32)
                h2 = np.array([al[i] * d64(V[i], v) for i in range(j + 1)])
                c = (h2 * al[:j + 1]).astype(f32)
                for i in range(j + 1): v = (v - c[i] * V[i]).astype(f32)
                col = h1 + h2; hj1 = math.sqrt(d64(v, v)); V[j + 1] = v; al[j + 1] = 1 / hj1
                H[:j + 1, j] = col; H[j + 1, j] = hj1
            else:
                at = al[j]
                z = np.array([al[i] * d64(V[i], w) for i in range(j + 1)])
                s = a_prev[:j] * at if j > 0 else np.zeros(0)
                r_ = math.sqrt(max(1 - float(np.sum(s * s)), 1e-300))
                if j > 0:
                    hl = H[j, j - 1]; H[:j, j - 1] += hl * s; H[j, j - 1] = hl * r_
                c = np.array([sum(H[i, kk] * s[kk] for kk in range(j)) for i in range(j + 1)])
                sz = float(np.dot(s, z[:j])) if j > 0 else 0.0
                h = np.zeros(j + 1); h[:j] = (z[:j] - c[:j]) / r_; h[j] = ((z[j] - sz) / r_ - c[j]) / r_
                d = c + r_ * h
                cA = (s * al[:j] / at).astype(f32); cB = np.zeros(j + 1)
                cB[:j] = (d[:j] - d[j] * s / r_) * al[:j]; cB[j] = d[j] * at / r_; cB = cB.astype(f32)
                vj = V[j].copy(); wn = (w - cB[j] * vj).astype(f32)
                for i in range(j):
                    vj = (vj - cA[i] * V[i]).astype(f32); wn = (wn - cB[i] * V[i]).astype(f32)
                V[j] = vj; al[j] = at / r_
                a_prev = np.array([al[i] * d64(V[i], wn) for i in range(j + 1)])
                n2 = d64(wn, wn)
                V[j + 1] = wn; al[j + 1] = 1 / math.sqrt(n2); col = h; hj1 = math.sqrt(n2) / r_
                H[:j + 1, j] = h; H[j + 1, j] = hj1
            cc = col.copy()
            for i in range(j):
                t = cs[i] * cc[i] + sn[i] * cc[i + 1]; cc[i + 1] = -sn[i] * cc[i] + cs[i] * cc[i + 1]; cc[i] = t
            den = math.hypot(cc[j], hj1); cs[j] = cc[j] / den; sn[j] = hj1 / den
            g[j + 1] = -sn[j] * g[j]; g[j] = cs[j] * g[j]; total += 1; k = j + 1
            if abs(g[j + 1]) <= rtol * bn or total >= maxit:
                break
        if mode == 'dcgs2':
            at = al[k]; s = a_prev[:k] * at; r_ = math.sqrt(max(1 - float(np.sum(s * s)), 1e-300))
            hl = H[k, k - 1]; H[:k, k - 1] += hl * s; H[k, k - 1] = hl * r_
        e = np.zeros(k + 1); e[0] = beta
        y = np.linalg.lstsq(H[:k + 1, :k], e, rcond=None)[0]
        Q = V[:k].astype(np.float64) * al[:k, None]
        x = x + Q.T @ y


out = {"config": 2, "preconditioner": "none", "oracle_fp64_mgs_iterations": 1290}
for mode in sys.argv[1:]:
    it, rel = gmres(mode)
    out[mode] = {"iterations": it, "relres_true": float(rel)}
    print(mode, it, rel, file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))
