"""Run-to-run bitwise determinism of the V-cycle (REPS repeats against the first; experiments)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_23265_b200 as P  # noqa: E402
import workloads as W  # noqa: E402
k = int(sys.argv[1])
cfg = W.config(k)
media = W.make_media(cfg)
p = P.rte_setup(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                n_polar=cfg.n_polar, n_azim=cfg.n_azim)
net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, W.make_weights(cfg))
r = torch.from_numpy(W.make_vector(cfg, 2)).cuda()
z0 = torch.empty_like(r)
P.mgnet_vcycle(net, r, z0, add_identity=False)
bad, mx = 0, 0.0
for rep in range(int(os.environ.get("REPS", "12"))):
    z = torch.empty_like(r)
    P.mgnet_vcycle(net, r, z, add_identity=False)
    torch.cuda.synchronize()
    d = float((z - z0).abs().max())
    mx = max(mx, d)
    bad += d > 0
print("cfg", k, "nondeterministic repeats", bad, "max", mx, flush=True)
