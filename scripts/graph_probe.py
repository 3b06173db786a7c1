"""Experiment: how much do kernel-boundary gaps cost?  Times one apply + one V-cycle eagerly and as
a replayed CUDA graph (captured through torch on the current stream).  CFG=5 python scripts/graph_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_23265_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

cfg = W.config(int(os.environ.get("CFG", "5")))
media = W.make_media(cfg)
p = P.rte_setup(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                n_polar=cfg.n_polar, n_azim=cfg.n_azim)
net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, W.make_weights(cfg))
x = torch.from_numpy(W.make_vector(cfg)).cuda()
y, z = torch.empty_like(x), torch.empty_like(x)


def work():
    P.rte_apply(p, x, y)
    P.mgnet_vcycle(net, x, z, True)


for _ in range(3):
    work()
torch.cuda.synchronize()
reps = 10
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    work()
e1.record()
torch.cuda.synchronize()
eager = e0.elapsed_time(e1) / reps
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    work()
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
with torch.cuda.graph(g):
    work()
z_eager = z.clone()
g.replay()
torch.cuda.synchronize()
same = torch.equal(z, z_eager)
e0.record()
for _ in range(reps):
    g.replay()
e1.record()
torch.cuda.synchronize()
graph = e0.elapsed_time(e1) / reps
print(f"eager {eager:.4f} ms  graph {graph:.4f} ms  gain {100 * (eager - graph) / eager:.1f}%  bitwise-equal {same}")
