"""Per-class roofline table of one GMRES(30) cycle on config 5 (for DESIGN.md / profiles/): every
timing class's device time per iteration and its achieved throughput against its binding bound
(the larger of algorithmic bytes / HBM and algorithmic flops / compute peak), from the library's
algorithmic flops/bytes and MEASURED_PEAKS.json.

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
# the binding roofline of a class is the larger of its two lower bounds, algorithmic bytes / HBM and
# algorithmic flops / its compute peak (a tensor-core GEMM with a short K can be HBM-bound)
for r in sorted(rows, key=lambda r: -r["ms"]):
    kind = r["kind"]
    n = max(r["launches"], 1)
    t = r["ms"] / n * 1e-3  # s per launch
    pk_c, unit_c = PEAK.get(kind, (None, "")) if kind != "hbm" else (None, "")
    t_mem = r["bytes"] / n / (hbm * 1e9) if r["bytes"] > 0 else 0.0
    t_cmp = r["flops"] / n / (pk_c * 1e12) if (pk_c and r["flops"] > 0) else 0.0
    if t_mem == 0.0 and t_cmp == 0.0:
        bound, achs, pks, frac = kind, "—", PEAK.get(kind, (None, ""))[0], "—"
        pks = f"{pks:.0f} {PEAK[kind][1]}" if pks else "—"
    elif t_mem >= t_cmp:
        bound = "hbm"
        achs, pks = f"{r['bytes'] / n / t / 1e9:.0f} GB/s", f"{hbm:.0f} GB/s"
        frac = f"{t_mem / t:.2f}"
    else:
        bound = kind
        achs, pks = f"{r['flops'] / n / t / 1e12:.0f} {unit_c}", f"{pk_c:.0f} {unit_c}"
        frac = f"{t_cmp / t:.2f}"
    print(f"| {r['name']} | {bound} | {r['launches'] / K:.1f} | {r['ms'] / K:.4f} | {r['ms'] / tot:.3f} | {achs} | {pks} | {frac} |")
