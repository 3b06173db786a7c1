import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2604_23265_b200 as P, workloads as W
cfg = W.config(5); media = W.make_media(cfg)
p = P.rte_setup(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow, n_polar=cfg.n_polar, n_azim=cfg.n_azim)
net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, W.make_weights(cfg))
b = torch.empty((1, cfg.N, cfg.N, cfg.M), dtype=torch.float32, device="cuda"); P.rte_rhs(p, b)
x = torch.zeros(b.shape, dtype=torch.float64, device="cuda")
P.gmres_solve(p, net, b, x, restart=30, maxit=5, rtol=1e-300, history=False)
for on in (False, True, False, True):
    P.rte_timing_enable(on); P.rte_timing_reset(); x.zero_(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); P.gmres_solve(p, net, b, x, restart=30, maxit=30, rtol=1e-300, history=False); e1.record()
    torch.cuda.synchronize(); print("timing", on, "ms/it", e0.elapsed_time(e1) / 30)
P.rte_timing_enable(False)
