"""Per-role cycle breakdown of the tensor-core GEMM over one V-cycle (experiments: needs a library
built with -DRTE_TC_PROF=1 -- var_libs/librte_prof.so, selected with RTE_LIB_PATH -- and RTE_TC_DBG
with bit 6; see csrc/tc_gemm.cuh g_tc_prof)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_23265_b200 as P  # noqa: E402
from paper_2604_23265_b200 import _lib  # noqa: E402
import workloads as W  # noqa: E402

cfg = W.config(int(os.environ.get("CFG", "5")))
media = W.make_media(cfg)
p = P.rte_setup(cfg.N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                n_polar=cfg.n_polar, n_azim=cfg.n_azim)
net = P.mgnet_create(p, cfg.L, cfg.C0, cfg.nu, W.make_weights(cfg))
x = torch.from_numpy(W.make_vector(cfg)).cuda()
z = torch.empty_like(x)
P.mgnet_vcycle(net, x, z, True)
torch.cuda.synchronize()
buf = (C.c_uint64 * 24)()
_lib.lib.rte_debug_counters(buf, 24, 1)
P.mgnet_vcycle(net, x, z, True)
P.rte_apply(p, x, z)  # (the filter bits in RTE_TC_DBG select which kernels are counted)
torch.cuda.synchronize()
_lib.lib.rte_debug_counters(buf, 24, 1)
v = list(buf)
kb = max(v[13], 1)
names = ["prod_total", "prod_wait", "mma_total", "mma_wait_in", "mma_wait_acc", "mma_issue", "conv_total",
         "conv_wait", "conv_work", "prom_total", "prom_wait", "prom_tmem", "epilogue", "kblocks", "conv_kbloop", "mma_kbloop", "epi_stage", "epi_rows", "epi_bar2", "prod_waitA", "prod_issueA", "prod_issueB", "mma_wait_bfull", "conv_wait_afull"]
print(f"dbg={os.environ.get('RTE_TC_DBG')} kblocks={v[13]} (cycles per K block, summed over CTAs):")
for i, nm in [(i, n) for i, n in enumerate(names) if i != 13]:
    print(f"  {nm:14s} {v[i] / kb:10.1f}")
