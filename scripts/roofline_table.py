"""Per-class roofline table of one GMRES(30) cycle on config 5 (for DESIGN.md / profiles/): every
timing class's device time per iteration and its achieved throughput against its own bound, from the
library's algorithmic flops/bytes and MEASURED_PEAKS.json.

  python scripts/roofline_table.py > profiles/r01_final/roofline_table.md
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_23265_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
hbm = peaks["hbm_gbs"]
bf16 = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
smax = peaks.get("sm_max_mhz", 1965.0)
PEAK = {"hbm": (hbm, "GB/s"), "tensor_3xtf32": (bf16 * 1.1 / 2.25 / 3.0, "TFLOP/s"),
        "fp32_simt": (148 * 128 * 2 * smax * 1e6 / 1e12, "TFLOP/s"), "fp64_simt": (37.2, "TFLOP/s")}

cfg = W.config(int(os.environ.get("CFG", "5")))
K = 30
media = W.make_media(cfg)
p = P.rte_setup(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                n_polar=cfg.n_polar, n_azim=cfg.n_azim)
net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, W.make_weights(cfg))
b = torch.empty(p.shape, dtype=torch.float32, device="cuda")
P.rte_rhs(p, b)
x = torch.zeros(p.shape, dtype=torch.float64, device="cuda")
P.gmres_solve(p, net, b, x, restart=30, maxit=K, rtol=1e-300, history=False)
torch.cuda.synchronize()
P.rte_timing_enable(True)
P.rte_timing_reset()
x.zero_()
P.gmres_solve(p, net, b, x, restart=30, maxit=K, rtol=1e-300, history=False)
torch.cuda.synchronize()
rows = P.rte_timing_get()
P.rte_timing_enable(False)
tot = sum(r["ms"] for r in rows)
print(f"# Per-class rooflines, config {cfg.k}, one GMRES({K}) cycle (profiled: every launch event-timed)\n")
print("| class | bound | launches/it | ms/it | share | achieved | peak | fraction |")
print("|---|---|---|---|---|---|---|---|")
for r in sorted(rows, key=lambda r: -r["ms"]):
    kind = r["kind"]
    ms_l = r["ms"] / max(r["launches"], 1)
    if kind == "hbm" and r["bytes"] > 0:
        ach = r["bytes"] / r["launches"] / (ms_l * 1e-3) / 1e9
    elif kind in ("tensor_3xtf32", "fp32_simt", "fp64_simt") and r["flops"] > 0:
        ach = r["flops"] / r["launches"] / (ms_l * 1e-3) / 1e12
    else:
        ach = None
    pk, unit = PEAK.get(kind, (None, ""))
    frac = f"{ach / pk:.2f}" if (ach is not None and pk) else "—"
    achs = f"{ach:.0f} {unit}" if ach is not None else "—"
    pks = f"{pk:.0f} {unit}" if pk else "—"
    print(f"| {r['name']} | {kind} | {r['launches'] / K:.1f} | {r['ms'] / K:.4f} | {r['ms'] / tot:.3f} | {achs} | {pks} | {frac} |")
