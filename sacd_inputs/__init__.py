"""Seeded synthetic inputs for SaCD (arXiv 2003.03572) -- shared by the oracle tests,
the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no MTTKRP, Gram, gradient, importance,
selection or objective).  It only defines:

* the counter-based generator `rand(seed, tag, ctr)`:
      mix64(z)  = SplitMix64 finaliser
      rand(seed, tag, ctr) = mix64(mix64(seed ^ tag) + (ctr + 1) * 0x9E3779B97F4A7C15)   (mod 2^64)
      unit24(x) = (x >> 40) * 2^-24      unit53(x) = (x >> 11) * 2^-53
  Tags: INIT=1 (factor init; implemented independently by the CUDA path and by oracle/),
  COORD=2, VALUE=3, PLANT=4, NOISE=5, SPLIT=6 (held-out split).
* the five BASELINE.json workloads c1..c5 (SURVEY.md section 8(d) "Synthetic inputs"):
  coordinates are "the first nnz distinct (q,p,s) in draw order", draw j using
  ctr = 3j + mode; values are keyed by the linear key q*P*S + p*S + s.

The paper's own synthetic workloads are random tensors (section 6.4:
mode lengths 2^6..2^14, densities 1e-3..1e-7, ranks 10..125); its real datasets
(Delicious, LastFM, Movielens, Gowalla; Table 3) are not available and
are stood in for by c3 (user x location x time counts) and c4 (user x item x tag binary).

Everything is computed with torch integer ops (int64 two's-complement wrap-around for
the mod-2^64 arithmetic), so the same function gives bit-identical tensors on CPU and on
CUDA.  Floating-point tables (Zipf / Poisson CDFs) are always built on the CPU in fp64.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

TAG_INIT, TAG_COORD, TAG_VALUE, TAG_PLANT, TAG_NOISE, TAG_SPLIT = 1, 2, 3, 4, 5, 6
SEED_BASE = 2003035720

_M64 = (1 << 64)


def _s64(c: int) -> int:
    """uint64 constant -> the int64 with the same bit pattern."""
    c &= _M64 - 1
    return c - _M64 if c >= (1 << 63) else c


_C1 = _s64(0xBF58476D1CE4E5B9)
_C2 = _s64(0x94D049BB133111EB)
_GOLD = _s64(0x9E3779B97F4A7C15)


def _lsr(x: torch.Tensor, k: int) -> torch.Tensor:
    """Logical shift right of int64 viewed as uint64."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def mix64_t(z: torch.Tensor) -> torch.Tensor:
    z = (z ^ _lsr(z, 30)) * _C1
    z = (z ^ _lsr(z, 27)) * _C2
    return z ^ _lsr(z, 31)


def mix64_int(z: int) -> int:
    z &= _M64 - 1
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (_M64 - 1)
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (_M64 - 1)
    return z ^ (z >> 31)


def rand_t(seed: int, tag: int, ctr: torch.Tensor) -> torch.Tensor:
    """rand(seed, tag, ctr) for an int64 tensor of counters; returns int64 bit patterns."""
    base = _s64(mix64_int((seed ^ tag) & (_M64 - 1)))
    return mix64_t(base + (ctr + 1) * _GOLD)


def rand_int(seed: int, tag: int, ctr: int) -> int:
    """Scalar reference of rand(); uint64 result."""
    return mix64_int((mix64_int(seed ^ tag) + (ctr + 1) * 0x9E3779B97F4A7C15) & (_M64 - 1))


def unit24_t(x: torch.Tensor) -> torch.Tensor:
    return _lsr(x, 40).to(torch.float64) * (2.0 ** -24)


def unit53_t(x: torch.Tensor) -> torch.Tensor:
    return _lsr(x, 11).to(torch.float64) * (2.0 ** -53)


# ----------------------------------------------------------------------------- tables
def zipf_cdf(n: int, s: float) -> np.ndarray:
    """fp64 CDF of the Zipf(s) law on ranks 1..n, built on the CPU (deterministic)."""
    w = np.arange(1, n + 1, dtype=np.float64) ** (-s)
    c = np.cumsum(w)
    return c / c[-1]


def poisson_cdf(lam: float, kmax: int = 64) -> np.ndarray:
    p = np.empty(kmax, dtype=np.float64)
    p[0] = math.exp(-lam)
    for k in range(1, kmax):
        p[k] = p[k - 1] * lam / k
    return np.cumsum(p)


# ----------------------------------------------------------------------------- configs
@dataclass(frozen=True)
class Config:
    cid: int
    name: str
    dims: tuple
    nnz: int
    rank: int
    iters: int
    index_dist: tuple          # per mode: ("uniform",) or ("zipf", s)
    values: str                # "unit", "rating", "poisson2", "ones", "planted"
    draw_factor: float = 1.02  # first guess of draws / nnz (grown until enough)
    ranks: tuple = field(default=())  # c5 rank sweep

    @property
    def seed(self) -> int:
        return SEED_BASE + self.cid


CONFIGS = {
    "c1": Config(1, "c1", (100, 100, 100), 10_000, 5, 10, (("uniform",),) * 3, "unit"),
    "c2": Config(2, "c2", (10_000, 10_000, 10_000), 1_000_000, 16, 50, (("uniform",),) * 3, "rating"),
    "c3": Config(3, "c3", (100_000, 50_000, 1_000), 10_000_000, 32, 50,
                 (("zipf", 1.1), ("zipf", 1.1), ("uniform",)), "poisson2", draw_factor=1.35),
    "c4": Config(4, "c4", (1_000_000, 500_000, 10_000), 100_000_000, 64, 20,
                 (("zipf", 1.2),) * 3, "ones", draw_factor=2.95),
    "c5": Config(5, "c5", (20_000, 20_000, 20_000), 20_000_000, 8, 20, (("uniform",),) * 3, "planted",
                 ranks=(8, 16, 32, 64, 128, 256)),
}


def custom_config(dims, nnz, rank, *, index_dist=None, values="unit", cid=100, iters=10) -> Config:
    """A small uniform config for tests (same recipe as c1)."""
    return Config(cid, f"custom{cid}", tuple(int(d) for d in dims), int(nnz), int(rank), iters,
                  index_dist or (("uniform",),) * 3, values)


def _draw_indices(cfg: Config, j0: int, j1: int, device) -> torch.Tensor:
    """coords for draws j0..j1-1 as an int64 [n,3] tensor."""
    j = torch.arange(j0, j1, dtype=torch.int64, device=device)
    cols = []
    for m in range(3):
        u = unit53_t(rand_t(cfg.seed, TAG_COORD, 3 * j + m))
        dist = cfg.index_dist[m]
        n = cfg.dims[m]
        if dist[0] == "uniform":
            idx = torch.floor(u * n).to(torch.int64)
        else:
            cdf = torch.from_numpy(zipf_cdf(n, dist[1])).to(device)
            idx = torch.searchsorted(cdf, u, right=True)
        cols.append(torch.clamp(idx, max=n - 1))
    return torch.stack(cols, dim=1)


def make_coords(cfg: Config, device="cpu") -> torch.Tensor:
    """The first cfg.nnz distinct coordinates in draw order, returned sorted by (q,p,s)
    as an int64 [nnz,3] tensor on `device`."""
    Q, P, S = cfg.dims
    assert Q * P * S < (1 << 62)
    nnz = cfg.nnz
    if nnz == 0:
        return torch.zeros((0, 3), dtype=torch.int64, device=device)
    assert nnz <= Q * P * S
    D = max(int(nnz * cfg.draw_factor) + 64, nnz)
    while True:
        c = _draw_indices(cfg, 0, D, device)
        key = (c[:, 0] * P + c[:, 1]) * S + c[:, 2]
        del c
        uniq, inv = torch.unique(key, sorted=True, return_inverse=True)
        if uniq.numel() < nnz:
            D = int(D * 1.3) + 1024
            del key, uniq, inv
            continue
        first = torch.full((uniq.numel(),), D, dtype=torch.int64, device=device)
        first.scatter_reduce_(0, inv, torch.arange(D, dtype=torch.int64, device=device), reduce="amin")
        del inv
        sel = torch.sort(first).values[:nnz]
        del first, uniq
        keys = torch.sort(key[sel]).values
        del key, sel
        q = keys // (P * S)
        rem = keys - q * (P * S)
        p = rem // S
        s = rem - p * S
        return torch.stack([q, p, s], dim=1)


def make_values(cfg: Config, coords: torch.Tensor) -> torch.Tensor:
    """fp32 values keyed by the linear key (independent of draw order)."""
    Q, P, S = cfg.dims
    dev = coords.device
    key = (coords[:, 0] * P + coords[:, 1]) * S + coords[:, 2]
    if cfg.values == "unit":            # 1 - unit24 in (0,1]
        v = 1.0 - unit24_t(rand_t(cfg.seed, TAG_VALUE, key))
    elif cfg.values == "rating":        # integers 1..5
        v = 1.0 + torch.floor(5.0 * unit53_t(rand_t(cfg.seed, TAG_VALUE, key)))
    elif cfg.values == "poisson2":      # Poisson(2) + 1 by inverse CDF
        cdf = torch.from_numpy(poisson_cdf(2.0)).to(dev)
        k = torch.searchsorted(cdf, unit53_t(rand_t(cfg.seed, TAG_VALUE, key)), right=True)
        v = (k + 1).to(torch.float64)
    elif cfg.values == "ones":
        v = torch.ones(key.shape, dtype=torch.float64, device=dev)
    elif cfg.values == "planted":
        return _planted_values(cfg, coords.cpu()).to(dev)
    else:
        raise ValueError(cfg.values)
    return v.to(torch.float32)


def planted_factors(cfg: Config, rank_true: int = 10):
    """Planted nonnegative factors (uniform [0,1) from the PLANT stream), fp64 CPU."""
    out, off = [], 0
    for n in cfg.dims:
        ctr = torch.arange(n * rank_true, dtype=torch.int64) + off
        out.append(unit24_t(rand_t(cfg.seed, TAG_PLANT, ctr)).reshape(n, rank_true))
        off += n * rank_true
    return out


def _planted_values(cfg: Config, coords: torch.Tensor, rank_true: int = 10) -> torch.Tensor:
    """c5: fl32(sum_r a_qr b_pr c_sr (fp64, r ascending) + |0.01 N(0,1)|), Box-Muller on NOISE.
    Always evaluated on the CPU so libm rounding is identical for every caller."""
    Q, P, S = cfg.dims
    a, b, c = planted_factors(cfg, rank_true)
    q, p, s = coords[:, 0], coords[:, 1], coords[:, 2]
    acc = torch.zeros(coords.shape[0], dtype=torch.float64)
    for r in range(rank_true):
        acc = acc + (a[q, r] * b[p, r]) * c[s, r]
    key = (q * P + p) * S + s
    u1 = unit53_t(rand_t(cfg.seed, TAG_NOISE, 2 * key))
    u2 = unit53_t(rand_t(cfg.seed, TAG_NOISE, 2 * key + 1))
    nrm = torch.sqrt(-2.0 * torch.log1p(-u1)) * torch.cos(2.0 * math.pi * u2)
    return (acc + torch.abs(0.01 * nrm)).to(torch.float32)


def make_tensor(cfg: Config, device="cpu"):
    """(coords uint32-valued int32 [nnz,3] contiguous, vals fp32 [nnz]) on `device`.
    Coordinates are sorted by (q,p,s).  int32 storage holds indices < 2^31."""
    c = make_coords(cfg, device)
    v = make_values(cfg, c)
    return c.to(torch.int32).contiguous(), v.contiguous()


def tiny_tensor(dims, density, seed, *, values="unit", device="cpu"):
    """Small random tensor for oracle pins: each cell kept iff unit53 < density."""
    Q, P, S = dims
    key = torch.arange(Q * P * S, dtype=torch.int64, device=device)
    keep = unit53_t(rand_t(seed, TAG_COORD, key)) < density
    key = key[keep]
    q = key // (P * S)
    p = (key - q * P * S) // S
    s = key - q * P * S - p * S
    c = torch.stack([q, p, s], 1)
    if values == "unit":
        v = (1.0 - unit24_t(rand_t(seed, TAG_VALUE, key))).to(torch.float32)
    else:
        raise ValueError(values)
    return c.to(torch.int32).contiguous(), v.contiguous()


def split_train_test(coords: torch.Tensor, vals: torch.Tensor, dims, seed: int, test_frac: float = 0.2):
    """Seeded held-out split (the paper's 80/20 protocol): an entry is a test
    entry iff unit53(rand(seed, SPLIT, linear key)) < test_frac.  Keyed by the coordinate,
    so the split does not depend on entry order.  Use the tensor's own seed: rand() streams
    collide when seed ^ tag collide (reading C12), e.g. seed 3 / COORD=2 and seed 7 / SPLIT=6.
    Returns (train_c, train_v, test_c, test_v)."""
    c = coords.long()
    key = (c[:, 0] * dims[1] + c[:, 1]) * dims[2] + c[:, 2]
    test = unit53_t(rand_t(seed, TAG_SPLIT, key)) < test_frac
    return coords[~test], vals[~test], coords[test], vals[test]
