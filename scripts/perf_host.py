"""Host enqueue time vs device time of rte_apply and mgnet_vcycle (per-launch timing OFF):
if the host takes longer to enqueue a V-cycle than the GPU takes to run it, the path is
launch-bound (experiments)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_23265_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = W.config(k)
media = W.make_media(cfg)
p = P.rte_setup(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                n_polar=cfg.n_polar, n_azim=cfg.n_azim)
net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, W.make_weights(cfg))
x = torch.from_numpy(W.make_vector(cfg)).cuda()
z = torch.empty_like(x)
y = torch.empty_like(x)
for name, fn in (("vcycle", lambda: P.mgnet_vcycle(net, x, z, True)), ("apply", lambda: P.rte_apply(p, x, y))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    reps = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        fn()
    t_host = (time.perf_counter() - t0) / reps * 1e3
    e1.record()
    torch.cuda.synchronize()
    t_dev = e0.elapsed_time(e1) / reps
    P.rte_launch_count(True)
    fn()
    torch.cuda.synchronize()
    print(f"cfg{k} {name}: host enqueue {t_host:.3f} ms/call, device {t_dev:.3f} ms/call, "
          f"launches/call {P.rte_launch_count(True)}", flush=True)
