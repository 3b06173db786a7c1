"""Seeded synthetic inputs for the five BASELINE.json configs.

This module is the ONLY code shared by the oracle (``oracle/``) and the CUDA path
(``paper_2604_23265_b200``).  It produces *inputs* only -- media fields, inflow
data, MgNet weights and random test vectors -- and holds none of the method's
arithmetic (no quadrature, no kernel, no operator, no V-cycle, no Krylov step).

Recipes follow SURVEY.md §8(d) (config table, GRF definition, Voronoi rule) and
the paper's media constraint "shift sigma_T such that sigma_T - sigma_a >= 0.2"
(§4.1).  Seeds: media 1000+k, weights 2000+k, vectors 3000+k
(numpy PCG64).  All arrays are float32 (the C-ABI's input precision); the oracle
reads them as float64.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

__all__ = [
    "Config", "CONFIGS", "config", "Media", "make_media", "mgnet_weight_shapes",
    "mgnet_weight_count", "make_weights", "make_vector", "grf", "small_config", "sample_indices",
]


@dataclasses.dataclass(frozen=True)
class Config:
    """One workload (BASELINE.json ``configs[k-1]``)."""
    k: int                 # 1-based config id
    N: int                 # cells per side (nx == ny == N), h = 1/N
    M: int                 # total number of ordinates (= 4 * paper's M)
    n_polar: int           # product quadrature: n_polar Gauss-Legendre zeta nodes
    n_azim: int            # ... times n_azim offset-uniform azimuths (M = n_polar*n_azim)
    B: int                 # batch of independent media
    L: int                 # MgNet levels
    C0: int                # MgNet channels at level 0 (C_l = C0 * 2^l)
    nu: int                # smoothing steps pre / post
    restart: int
    rtol: float
    maxit: int             # iteration cap (full solve) or fixed budget (cfgs 3-5)
    fixed_budget: bool     # True where GMRES does not converge with random weights

    @property
    def unknowns(self) -> int:
        return self.B * self.N * self.N * self.M


CONFIGS = {
    1: Config(1, 32, 16, 2, 8, 1, 3, 16, 2, 30, 1e-8, 1000, False),
    2: Config(2, 64, 32, 2, 16, 1, 4, 16, 2, 30, 1e-6, 3000, False),
    3: Config(3, 128, 64, 4, 16, 1, 4, 32, 2, 30, 1e-6, 300, True),
    4: Config(4, 256, 128, 4, 32, 8, 5, 32, 2, 30, 1e-6, 60, True),
    5: Config(5, 512, 256, 8, 32, 1, 6, 32, 2, 30, 1e-6, 30, True),
}


def config(k: int) -> Config:
    return CONFIGS[k]


def small_config(k: int, N: int, M: Optional[int] = None, n_polar: Optional[int] = None,
                 n_azim: Optional[int] = None, L: Optional[int] = None,
                 C0: Optional[int] = None, B: Optional[int] = None) -> Config:
    """A reduced copy of config k (same media recipe, smaller grid/angles/net)."""
    c = CONFIGS[k]
    np_ = n_polar if n_polar is not None else c.n_polar
    na = n_azim if n_azim is not None else c.n_azim
    if M is not None and (n_polar is None and n_azim is None):
        # keep the polar count, shrink azimuths
        na = M // np_
    return dataclasses.replace(
        c, N=N, M=np_ * na, n_polar=np_, n_azim=na,
        L=L if L is not None else c.L, C0=C0 if C0 is not None else c.C0,
        B=B if B is not None else c.B)


@dataclasses.dataclass
class Media:
    """Cell-valued media (all float32, shape [B][N][N] = [batch][y=j][x=i])."""
    sigma_T: np.ndarray
    sigma_a: np.ndarray
    q: np.ndarray
    eps: np.ndarray
    g: np.ndarray          # [B]
    inflow: np.ndarray     # [B][4 faces: L(x=0), R(x=1), B(y=0), T(y=1)][N][M]


def grf(rng: np.random.Generator, N: int, ell: float, log_std: float) -> np.ndarray:
    """Periodic Gaussian random field on the N x N cell grid (SURVEY.md §8(d) "GRF G").

    White noise W, G_hat(k) = W_hat(k) exp(-|k|^2 ell^2 / 4) with k in rad/cell
    (covariance proportional to exp(-r^2 / 2 ell^2)); standardised to sample
    mean 0 / std 1, then scaled by ``log_std``.
    """
    W = rng.standard_normal((N, N))
    k = 2.0 * np.pi * np.fft.fftfreq(N)            # rad / cell
    k2 = k[:, None] ** 2 + k[None, :] ** 2
    G = np.real(np.fft.ifft2(np.fft.fft2(W) * np.exp(-k2 * ell * ell / 4.0)))
    G = (G - G.mean()) / G.std()
    return G * log_std


def _cell_centres(N: int):
    c = (np.arange(N) + 0.5) / N
    return c[None, :], c[:, None]      # x (varies along i / axis 1), y (along j / axis 0)


def make_media(cfg: Config) -> Media:
    """Seeded media for config ``cfg.k`` at the grid size ``cfg.N`` (seed 1000+k)."""
    N, M, B = cfg.N, cfg.M, cfg.B
    rng = np.random.Generator(np.random.PCG64(1000 + cfg.k))
    shape = (B, N, N)
    sT = np.ones(shape); sa = np.zeros(shape); q = np.ones(shape); eps = np.ones(shape)
    g = np.zeros(B); inflow = np.zeros((B, 4, N, M))
    X, Y = _cell_centres(N)
    jj, ii = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    if cfg.k == 1:
        pass                                                   # eps=1, sT=1, sa=0, q=1, g=0
    elif cfg.k == 2:
        eps[:] = 1e-2
        blk = max(1, 8 * N // 64)                              # 8x8-cell blocks at N=64
        sT[:] = np.where(((ii // blk) + (jj // blk)) % 2 == 0, 1.0, 10.0)
        sa[:] = 0.1
        inside = (X > 0.25) & (X < 0.75) & (Y > 0.25) & (Y < 0.75)
        q[:] = np.where(inside, 1.0, 0.0)
        g[:] = 0.5
        inflow[:, 0, :, :] = 1.0                               # Psi = 1 on x = 0 (c_m > 0 read)
    elif cfg.k == 3:
        eps[:] = 1e-3
        ell = 8.0 * N / 128
        sT[0] = np.exp(grf(rng, N, ell, 1.0))
        nb = max(1, N // 16)                                   # 16x16-cell blocks (8x8 blocks at N=128)
        blocks = rng.uniform(0.0, 0.5, size=(nb, nb))
        bs = N // nb
        sa[0] = blocks[jj // bs, ii // bs]
        g[:] = 0.9
    elif cfg.k == 4:
        for b in range(B):
            eps[b] = 10.0 ** rng.uniform(-4.0, 0.0)
            seeds = rng.uniform(0.0, 1.0, size=(32, 2))        # (x, y)
            d2 = (X[None] - seeds[:, 0, None, None]) ** 2 + (Y[None] - seeds[:, 1, None, None]) ** 2
            region = np.argmin(d2, axis=0)                     # ties -> lowest index
            sT_r = rng.uniform(0.5, 20.0, size=32)
            sa_r = rng.uniform(0.0, 1.0, size=32)
            sT[b] = sT_r[region]
            sa[b] = sa_r[region]
            gap = (sT[b] - sa[b]).min()
            if gap < 0.2:                                      # PAPER.md:520 shift
                sT[b] += 0.2 - gap
            g[b] = rng.uniform(0.0, 0.9)
    elif cfg.k == 5:
        eps[:] = 1e-4
        ell = 16.0 * N / 512
        sT[0] = np.exp(grf(rng, N, ell, 1.5))
        sa[:] = 0.05
        g[:] = 0.8
        inflow[:, 2, :, :] = 1.0                               # Psi = 1 on y = 0 (s_m > 0 read)
    else:
        raise ValueError(cfg.k)
    f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    return Media(f32(sT), f32(sa), f32(q), f32(eps), f32(g), f32(inflow))


def mgnet_weight_shapes(M: int, L: int, C0: int, nu: int):
    """Packed MgNet weight order, PyTorch layouts.

    Returns a list of (name, shape).  Lambda [C0][M][1][1]; for l in 0..L-1:
    A^l [C_l][C_l][3][3], pre B^{l,1..nu}, post B'^{l,1..nu}; if l < L-1:
    R^l [C_{l+1}][C_l][3][3] (OIHW) and P^l [C_{l+1}][C_l][4][4]
    (conv_transpose IOHW); finally Theta [M][C0][1][1].
    """
    out = [("Lambda", (C0, M, 1, 1))]
    for l in range(L):
        C = C0 << l
        out.append((f"A{l}", (C, C, 3, 3)))
        for i in range(nu):
            out.append((f"Bpre{l}_{i}", (C, C, 3, 3)))
        for i in range(nu):
            out.append((f"Bpost{l}_{i}", (C, C, 3, 3)))
        if l < L - 1:
            out.append((f"R{l}", (2 * C, C, 3, 3)))
            out.append((f"P{l}", (2 * C, C, 4, 4)))
    out.append(("Theta", (M, C0, 1, 1)))
    return out


def mgnet_weight_count(M: int, L: int, C0: int, nu: int) -> int:
    return int(sum(math.prod(s) for _, s in mgnet_weight_shapes(M, L, C0, nu)))


def make_weights(cfg: Config, std: float = 0.02, seed: Optional[int] = None) -> np.ndarray:
    """Packed float32 MgNet weights, i.i.d. N(0, std^2) drawn in fp64 (seed 2000+k), cast RN."""
    n = mgnet_weight_count(cfg.M, cfg.L, cfg.C0, cfg.nu)
    rng = np.random.Generator(np.random.PCG64(2000 + cfg.k if seed is None else seed))
    return (rng.standard_normal(n) * std).astype(np.float32)


def coeffnet_weight_layout(L: int, C0: int):
    """(name, shape) of the packed CoeffNet weights in order (R33; layout only): per level
    l, trunk conv K_l [C_l][C_in][3][3] (C_in = 3 at l = 0, else C_{l-1}), its bias [C_l], the
    a-head [C_l][C_l] and bias [C_l], the abar-head [C_l][C_l] and bias [C_l]; C_l = C0 2^l."""
    out = []
    for l in range(L):
        C = C0 << l
        Cin = 3 if l == 0 else (C0 << (l - 1))
        out += [(f"K{l}", (C, Cin, 3, 3)), (f"beta{l}", (C,)), (f"Ga{l}", (C, C)), (f"ga{l}", (C,)),
                (f"Gb{l}", (C, C)), (f"gb{l}", (C,))]
    return out


def coeffnet_weight_count(L: int, C0: int) -> int:
    return int(sum(math.prod(s) for _, s in coeffnet_weight_layout(L, C0)))


def make_coeffnet_weights(cfg: Config, head_std: float = 0.002, seed: Optional[int] = None) -> np.ndarray:
    """Packed float32 CoeffNet weights (seed 4000+k), drawn in fp64 and cast RN: trunk convs
    N(0, 2/fan_in) (He), trunk biases 0, head weights N(0, head_std^2 / C_l), head biases 1 -- a
    near-identity modulation (config 5: maps within ~1 +- 0.4; the paper's trained weights are
    not released)."""
    rng = np.random.Generator(np.random.PCG64(4000 + cfg.k if seed is None else seed))
    parts = []
    for name, shp in coeffnet_weight_layout(cfg.L, cfg.C0):
        n = math.prod(shp)
        if name.startswith("K"):
            fan_in = shp[1] * 9
            parts.append(rng.standard_normal(n) * math.sqrt(2.0 / fan_in))
        elif name.startswith("beta"):
            parts.append(np.zeros(n))
        elif name.startswith("G"):
            parts.append(rng.standard_normal(n) * head_std / math.sqrt(shp[0]))
        else:
            parts.append(np.ones(n))
    return np.concatenate(parts).astype(np.float32)


PAPER_REGIMES = ("diffusion", "transport", "lr", "rl", "tb", "bt", "centre", "outer")


def paper_media(n_samples: int, N: int = 32, degree: int = 2, regime: str = "diffusion", M: int = 4,
                seed: int = 0) -> Media:
    """The paper's test media (§4.1; NEXT-2): per sample,
      sigma = (2 + sum_{k<=n} c_{x,k} (x - 1/2)^k) (2 + sum_{k<=n} c_{y,k} (y - 1/2)^k),
      c ~ U[-1, 1], drawn independently for sigma_T and sigma_a, evaluated at cell centres
      (R34); sigma_T is shifted so that sigma_T - sigma_a >= 0.2 everywhere.
    eps regimes: "diffusion" eps = 0.01 (c + 0.1), c ~ U[0, 1] per sample; "transport" eps = 1;
    the six sharp-interface layouts mix the two in space: "lr"/"rl" (left/right half diffusive),
    "tb"/"bt" (bottom/top half diffusive), "centre" ([1/4, 3/4]^2 diffusive, transport outside)
    and "outer" (vice versa).  q = 0, g = 0, no inflow: the paper pairs the media with random
    right-hand sides, so the GMRES experiments draw b directly (make_paper_rhs)."""
    if regime not in PAPER_REGIMES:
        raise ValueError(f"regime must be one of {PAPER_REGIMES}")
    rng = np.random.Generator(np.random.PCG64([5000, seed]))
    X, Y = _cell_centres(N)

    def poly():
        cx = rng.uniform(-1.0, 1.0, degree + 1)
        cy = rng.uniform(-1.0, 1.0, degree + 1)
        px = 2.0 + sum(cx[k] * (X - 0.5) ** k for k in range(degree + 1))
        py = 2.0 + sum(cy[k] * (Y - 0.5) ** k for k in range(degree + 1))
        return px * py
    sT = np.zeros((n_samples, N, N)); sa = np.zeros_like(sT); eps = np.ones_like(sT)
    for b in range(n_samples):
        t, a = poly(), poly()
        gap = (t - a).min()
        if gap < 0.2:
            t = t + (0.2 - gap)
        sT[b], sa[b] = t, a
        e_diff = 0.01 * (rng.uniform(0.0, 1.0) + 0.1)
        diff = {"diffusion": np.ones((N, N), bool), "transport": np.zeros((N, N), bool),
                "lr": np.broadcast_to(X < 0.5, (N, N)), "rl": np.broadcast_to(X >= 0.5, (N, N)),
                "tb": np.broadcast_to(Y < 0.5, (N, N)), "bt": np.broadcast_to(Y >= 0.5, (N, N)),
                "centre": (X > 0.25) & (X < 0.75) & (Y > 0.25) & (Y < 0.75)}
        diff["outer"] = ~diff["centre"]
        eps[b] = np.where(diff[regime], e_diff, 1.0)
    f32 = lambda a: np.asarray(a, np.float32)
    return Media(f32(sT), f32(sa), f32(np.zeros_like(sT)), f32(eps), np.zeros(n_samples, np.float32),
                 np.zeros((n_samples, 4, N, M), np.float32))


def make_paper_rhs(n_samples: int, N: int = 32, M: int = 4, seed: int = 0) -> np.ndarray:
    """Random right-hand sides for the paper workload: b ~ U[0, 1] i.i.d. per unknown (float32)."""
    rng = np.random.Generator(np.random.PCG64([6000, seed]))
    return rng.uniform(0.0, 1.0, (n_samples, N, N, M)).astype(np.float32)


def make_vector(cfg: Config, which: int = 0) -> np.ndarray:
    """Parity vector x ~ N(0,1) i.i.d. per unknown, float32 [B][N][N][M] (seed 3000+k)."""
    rng = np.random.Generator(np.random.PCG64([3000 + cfg.k, which]))
    return rng.standard_normal((cfg.B, cfg.N, cfg.N, cfg.M)).astype(np.float32)


def sample_indices(cfg: Config, count: int = 16384) -> np.ndarray:
    """Seeded, sorted, distinct indices into one sample's flattened unknowns (seed 4000+k): where the
    fixed-budget parity tests compare the iterate x of configs too large to store whole."""
    n = cfg.N * cfg.N * cfg.M
    rng = np.random.Generator(np.random.PCG64([4000 + cfg.k]))
    return np.sort(rng.choice(n, size=min(count, n), replace=False))
