"""Training harness of the filtered MgNet solver (NEXT-4; PAPER.md:492-507 eq:loss / eq:loss_delta, the
training setup PAPER.md:529-530; readings R43-R45 in DESIGN.md §3).

* ``MgNet`` is the V-cycle of csrc/mgnet.cu (``mgnet_vcycle`` with the pass-through, z = r + Theta u^0) as a
  torch module with the packed weight order R20, so that ``MgNet.flat()`` feeds ``mgnet_create`` directly.
  The network's forward and backward during TRAINING use torch's conv2d / conv_transpose2d (cuDNN): this
  harness is not on the benchmarked path, which runs the trained weights through our kernels
  (``mgnet_vcycle`` / ``gmres_solve``).  CoeffNet modulation (NEXT-1) is not trained here.
* ``loss_delta`` is the paper's filtered loss evaluated by the library: ``rte_atfps_loss`` runs D_delta,
  the compressed operator A_bar_delta, b_bar_delta and the gradient with respect to the network output
  psi_d in our CUDA kernels (csrc/loss.cu, csrc/tfps.cu); the autograd function hands that gradient to
  torch for the weight gradients.
* ``train``: the network input is the psi-space right-hand side b (``rte_rhs`` of the discrete-ordinates
  problem of the same medium and source), the output psi_d = MgNet(b) (R44); random right-hand sides are
  random sources q ~ U[0, 1] per cell drawn per step and installed with ``rte_set_source`` in both problems;
  Adam with the initial learning rate 1e-3 and cosine annealing (Adam is R45's reading of the
  unnamed optimiser); the objective is the batch mean of loss_delta.
"""
from __future__ import annotations

import math
from typing import Dict, List, Optional

import numpy as np
import torch
import torch.nn.functional as F

from . import (Problem, rte_atfps_loss, rte_rhs, rte_set_source, rte_setup, rte_setup_atfps)


def weight_count(M: int, L: int, C0: int, nu: int) -> int:
    """Floats in the packed weight vector (R20), as mgnet_create checks it."""
    n = 2 * C0 * M
    for level in range(L):
        C = C0 << level
        n += (1 + 2 * nu) * C * C * 9
        if level < L - 1:
            n += 2 * C * C * 9 + 2 * C * C * 16
    return n


class MgNet(torch.nn.Module):
    """Linear MgNet V-cycle in NCHW torch layout; inputs/outputs [B][N][N][M] like the
    library's vectors.  Parameter order = R20: Lambda [C0][M][1][1]; per level A, nu pre-smoothers B,
    nu post-smoothers B (each [C][C][3][3]), then (not on the coarsest level) R [2C][C][3][3] (stride-2 conv)
    and P [2C][C][4][4] (stride-2 transposed conv, IOHW); Theta [M][C0][1][1]."""

    def __init__(self, M: int, L: int, C0: int, nu: int, weights: Optional[np.ndarray] = None,
                 device: str = "cuda", dtype=torch.float32):
        super().__init__()
        self.M, self.L, self.C0, self.nu = M, L, C0, nu
        shapes = [(C0, M, 1, 1)]
        for level in range(L):
            C = C0 << level
            shapes += [(C, C, 3, 3)] * (1 + 2 * nu)
            if level < L - 1:
                shapes += [(2 * C, C, 3, 3), (2 * C, C, 4, 4)]
        shapes.append((M, C0, 1, 1))
        n = sum(int(np.prod(s)) for s in shapes)
        if weights is None:
            weights = np.zeros(n, np.float32)
        weights = np.asarray(weights, np.float32).ravel()
        if weights.size != n:
            raise ValueError(f"MgNet: expected {n} weights, got {weights.size}")
        self.params = torch.nn.ParameterList()
        off = 0
        for s in shapes:
            k = int(np.prod(s))
            t = torch.tensor(weights[off:off + k].reshape(s), dtype=dtype, device=device)
            self.params.append(torch.nn.Parameter(t))
            off += k

    def _unpacked(self):
        it = iter(self.params)
        lift = next(it)
        levels = []
        for level in range(self.L):
            A = next(it)
            pre = [next(it) for _ in range(self.nu)]
            post = [next(it) for _ in range(self.nu)]
            R = P = None
            if level < self.L - 1:
                R, P = next(it), next(it)
            levels.append((A, pre, post, R, P))
        head = next(it)
        return lift, levels, head

    def forward(self, r: torch.Tensor) -> torch.Tensor:
        lift, levels, head = self._unpacked()
        x = r.permute(0, 3, 1, 2)
        L = self.L
        f: List[torch.Tensor] = [F.conv2d(x, lift)] + [None] * (L - 1)
        u: List[torch.Tensor] = [None] * L
        for level in range(L):
            A, pre, post, R, _ = levels[level]
            steps = pre + (post if level == L - 1 else [])
            uu = torch.zeros_like(f[level])
            for i, Bw in enumerate(steps):
                if i == 0:
                    uu = F.conv2d(f[level], Bw, padding=1)                    # u = B * f  (u = 0 before)
                else:
                    uu = uu + F.conv2d(f[level] - F.conv2d(uu, A, padding=1), Bw, padding=1)
            u[level] = uu
            if level < L - 1:
                t = f[level] - F.conv2d(uu, A, padding=1) if steps else f[level]
                f[level + 1] = F.conv2d(t, R, stride=2, padding=1)            # restriction
        for level in range(L - 2, -1, -1):
            A, _, post, _, P = levels[level]
            u[level] = u[level] + F.conv_transpose2d(u[level + 1], P, stride=2, padding=1)  # prolongation
            for Bw in post:
                u[level] = u[level] + F.conv2d(f[level] - F.conv2d(u[level], A, padding=1), Bw, padding=1)
        z = x + F.conv2d(u[0], head)
        return z.permute(0, 2, 3, 1).contiguous()

    def flat(self) -> np.ndarray:
        """The packed weight vector (R20) for mgnet_create."""
        return np.concatenate([p.detach().cpu().numpy().astype(np.float32).ravel() for p in self.params])


class _LossDelta(torch.autograd.Function):
    """loss_delta per sample from the library; backward = the library's gradient scaled per sample."""

    @staticmethod
    def forward(ctx, psi: torch.Tensor, prob: Problem):
        psi_c = psi.detach().contiguous()
        grad = torch.empty_like(psi_c)
        loss = rte_atfps_loss(prob, psi_c, grad)
        ctx.save_for_backward(grad)
        return torch.from_numpy(loss).to(device=psi.device, dtype=psi.dtype)

    @staticmethod
    def backward(ctx, gout: torch.Tensor):
        (grad,) = ctx.saved_tensors
        return grad * gout.view(-1, 1, 1, 1), None


def loss_delta(psi: torch.Tensor, prob: Problem) -> torch.Tensor:
    """eq:loss_delta of the network output psi [B][N][N][M] on the ATFPS problem `prob` (per sample)."""
    return _LossDelta.apply(psi, prob)


def train(N: int, n_polar: int, n_azim: int, media, *, L: int, C0: int, nu: int, delta: float, steps: int,
          lr: float = 1e-3, seed: int = 0, init_std: float = 0.02, eval_every: int = 0,
          val_sources: Optional[np.ndarray] = None, weights: Optional[np.ndarray] = None,
          sources: Optional[np.ndarray] = None) -> Dict:
    """Train MgNet on loss_delta over the batch of media `media` (a workloads.Media with B samples; sources
    redrawn every step, or cycled through `sources` [k][B][N][N] if given).  Returns the trained weights
    (R20) and the loss curves."""
    M = n_polar * n_azim
    torch.backends.cudnn.allow_tf32 = False  # train the fp32 function the library evaluates (no TF32 convs)
    p0 = rte_setup(N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow,
                   n_polar=n_polar, n_azim=n_azim)
    p2 = rte_setup_atfps(N, media.sigma_T, media.sigma_a, media.q, media.eps, media.g, media.inflow, delta=delta,
                         n_polar=n_polar, n_azim=n_azim)
    B = p0.batch
    rng = np.random.default_rng(seed)
    if weights is None:
        weights = rng.normal(0.0, init_std, weight_count(M, L, C0, nu)).astype(np.float32)
    net = MgNet(M, L, C0, nu, weights)
    opt = torch.optim.Adam(net.parameters(), lr=lr)
    sched = torch.optim.lr_scheduler.CosineAnnealingLR(opt, T_max=max(1, steps))
    b = torch.empty(p0.shape, dtype=torch.float32, device="cuda")

    def evaluate(qs):
        vals = []
        with torch.no_grad():
            for q in qs:
                rte_set_source(p0, q)
                rte_set_source(p2, q)
                rte_rhs(p0, b)
                vals.append(float(loss_delta(net(b), p2).mean()))
        return float(np.mean(vals))

    hist, val_hist, lrs = [], [], []
    for step in range(steps):
        q = (rng.uniform(0.0, 1.0, (B, N, N)).astype(np.float32) if sources is None
             else np.asarray(sources[step % len(sources)], np.float32))
        rte_set_source(p0, q)
        rte_set_source(p2, q)
        rte_rhs(p0, b)
        opt.zero_grad(set_to_none=True)
        loss = loss_delta(net(b), p2).mean()
        loss.backward()
        opt.step()
        lrs.append(float(opt.param_groups[0]["lr"]))
        sched.step()
        hist.append(float(loss.detach()))
        if eval_every and val_sources is not None and (step % eval_every == 0 or step == steps - 1):
            val_hist.append((step, evaluate(val_sources)))
    return {"weights": net.flat(), "loss": hist, "val": val_hist, "lr": lrs, "net": net, "problems": (p0, p2)}


def cosine_lr(step: int, steps: int, lr0: float = 1e-3) -> float:
    """The learning rate of CosineAnnealingLR(T_max = steps, eta_min = 0) at `step` (for tests)."""
    return 0.5 * lr0 * (1.0 + math.cos(math.pi * step / steps))
