"""Per-kernel-class device times of one rte_apply and one mgnet_vcycle on a config (default 5).
Perf experiments only (RTE_TC_DBG switches make results wrong on purpose)."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_23265_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
cfg = W.config(a.config)
media = W.make_media(cfg)
p = P.rte_setup(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                n_polar=cfg.n_polar, n_azim=cfg.n_azim)
net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, W.make_weights(cfg))
x = torch.from_numpy(W.make_vector(cfg)).cuda()
y = torch.empty_like(x)
z = torch.empty_like(x)
for _ in range(2):
    P.rte_apply(p, x, y)
    P.mgnet_vcycle(net, x, z, True)
torch.cuda.synchronize()
P.rte_timing_enable(True)
P.rte_timing_reset()
for _ in range(a.reps):
    P.rte_apply(p, x, y)
    P.mgnet_vcycle(net, x, z, True)
torch.cuda.synchronize()
cls = P.rte_timing_get()
P.rte_timing_enable(False)
out = {c["name"]: round(c["ms"] / a.reps, 4) for c in sorted(cls, key=lambda c: -c["ms"])}
out["_total_ms"] = round(sum(c["ms"] for c in cls) / a.reps, 4)
# wall time of the same work without per-launch events (the gap to _total_ms = kernel boundaries)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    P.rte_apply(p, x, y)
    P.mgnet_vcycle(net, x, z, True)
e1.record()
torch.cuda.synchronize()
out["_wall_ms"] = round(e0.elapsed_time(e1) / a.reps, 4)
P.rte_launch_count(reset=True)
P.rte_apply(p, x, y)
P.mgnet_vcycle(net, x, z, True)
out["_launches"] = P.rte_launch_count(reset=True)
out["_dbg"] = os.environ.get("RTE_TC_DBG", "0")
print(json.dumps(out))
