"""Seeded synthetic inputs for BASELINE.json's configs (test/bench infrastructure).

BASELINE.json names no dataset: every config is synthetic, described by its
shapes and value distributions.  These generators follow those descriptions;
seeds are fixed per config and recorded in every bench line.  ``scale`` shrinks
N (and optionally K) for parity tests the CPU oracle can finish in seconds.

configs[0] c0: fp64 N=1e4 K=50 M=5 P=10, labels U[1,P]; all 16 flag combos
configs[1] c1: fp64 N=1e6 K=500 M=10 P=100 near-equal folds (random_partitioning)
configs[2] c2: fp64 N=1e5 K=2000 M=1 P=50 Dirichlet(2) fold sizes, 10% columns sigma=1e-3
configs[3] c3: fp32 N=4e6 K=1024 M=16 P=20 random labels, X = mu + sigma * t5
configs[4] c4: fp64 N=1e7 K=256 M=32 P=5 contiguous row blocks
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SEEDS = {0: 20240123, 1: 20240124, 2: 20240125, 3: 20240126, 4: 20240127}
SHAPES = {0: (10_000, 50, 5, 10), 1: (1_000_000, 500, 10, 100), 2: (100_000, 2000, 1, 50),
          3: (4_000_000, 1024, 16, 20), 4: (10_000_000, 256, 32, 5)}
CONFIGS = {0: list(range(16)), 1: [15], 2: [12, 10], 3: [0, 1, 2, 3, 4, 5, 6, 7, 8, 10, 12, 14], 4: [15]}
DTYPES = {0: np.float64, 1: np.float64, 2: np.float64, 3: np.float32, 4: np.float64}
DESCRIPTIONS = {0: "all 16 flag combinations, labels U[1,P]",
                1: "center+scale X and Y, near-equal folds via random_partitioning",
                2: "Dirichlet(2) fold sizes, 10% of columns sigma=1e-3; center X,Y then center+scale X",
                3: "fp32 inputs, X = mu + sigma*t5, 12 distinct flag combinations, tcgen05 3xTF32",
                4: "contiguous fold blocks, center+scale X and Y"}


@dataclass
class Workload:
    cid: int
    x: np.ndarray
    y: np.ndarray
    labels: np.ndarray  # int32, 1-based
    p: int
    cfgs: list
    seed: int

    @property
    def n(self):
        return self.x.shape[0]

    @property
    def k(self):
        return self.x.shape[1]

    @property
    def m(self):
        return self.y.shape[1]

    @property
    def flops(self) -> float:
        """Algorithmic flops of one all-fold pass: 2·N·K(K+M) (BASELINE.json metric)."""
        return 2.0 * self.n * self.k * (self.k + self.m)


_M64 = (1 << 64) - 1


def mt19937_64(seed: int, count: int) -> np.ndarray:
    """The first `count` draws of std::mt19937_64(seed), vectorised in numpy (the C++
    standard's engine: n = 312, m = 156; checked against its specified 10000th value
    and against the engine library's and the oracle's streams in tests/test_host_logic.py).
    Plain numpy so that both bench arms draw identical labels without loading any .so."""
    n, m = 312, 156
    mt = np.zeros(n, dtype=np.uint64)
    mt[0] = seed & _M64
    for i in range(1, n):
        prev = int(mt[i - 1])
        mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & _M64
    um, lm = np.uint64(0xFFFFFFFF80000000), np.uint64(0x7FFFFFFF)
    a, zero, one = np.uint64(0xB5026F5AA96619E9), np.uint64(0), np.uint64(1)
    out = np.empty(-(-count // n) * n, dtype=np.uint64)
    for b in range(out.size // n):
        # twist: words [0, m) read old words only, [m, n-1) read the new [0, m-1), the last wraps to new 0
        y = (mt[:m] & um) | (mt[1:m + 1] & lm)
        mt[:m] = mt[m:] ^ (y >> one) ^ np.where(y & one, a, zero)
        y = (mt[m:n - 1] & um) | (mt[m + 1:] & lm)
        mt[m:n - 1] = mt[:m - 1] ^ (y >> one) ^ np.where(y & one, a, zero)
        y = (mt[n - 1] & um) | (mt[0] & lm)
        mt[n - 1] = mt[m - 1] ^ (y >> one) ^ (a if y & one else zero)
        x = mt.copy()
        x ^= (x >> np.uint64(29)) & np.uint64(0x5555555555555555)
        x ^= (x << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        x ^= (x << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        x ^= x >> np.uint64(43)
        out[b * n:(b + 1) * n] = x
    return out[:count]


def random_partitioning(n: int, p: int, seed: int) -> np.ndarray:
    """random_partitioning (random.hpp:38-50) with std::mt19937_64(seed): labels
    1 + (i mod p), then Fisher-Yates from the last row down (one draw per swap)."""
    labels = (1 + np.arange(n, dtype=np.int64) % p).astype(np.int32)
    if n < 2:
        return labels
    draws = mt19937_64(seed, n - 1)
    i = np.arange(n - 1, 0, -1, dtype=np.uint64)
    js = (draws % (i + np.uint64(1))).astype(np.int64).tolist()
    lab = labels.tolist()
    for ii, j in zip(range(n - 1, 0, -1), js):
        lab[ii], lab[j] = lab[j], lab[ii]
    return np.asarray(lab, dtype=np.int32)


def _labels(cid: int, n: int, p: int, rng: np.random.Generator, seed: int) -> np.ndarray:
    if cid == 1:
        # "row i in fold i mod P after a seeded shuffle": the reference's own
        # random_partitioning (random.hpp:38-50) with std::mt19937_64(seed).
        return random_partitioning(n, p, seed)
    if cid == 2:
        w = rng.gamma(2.0, size=p)
        w /= w.sum()
        raw = w * n
        sizes = np.floor(raw).astype(np.int64)
        sizes = np.maximum(sizes, 1)
        rem = n - sizes.sum()
        order = np.argsort(-(raw - np.floor(raw)))
        i = 0
        while rem != 0:
            j = order[i % p]
            if rem > 0:
                sizes[j] += 1
                rem -= 1
            elif sizes[j] > 1:
                sizes[j] -= 1
                rem += 1
            i += 1
        labels = np.repeat(np.arange(1, p + 1, dtype=np.int32), sizes)
        return rng.permutation(labels).astype(np.int32)
    if cid == 4:
        return (1 + (np.arange(n, dtype=np.int64) * p) // n).astype(np.int32)  # contiguous blocks
    lab = rng.integers(1, p + 1, n).astype(np.int32)
    lab[:p] = np.arange(1, p + 1, dtype=np.int32)[rng.permutation(p)]  # every fold non-empty
    return lab


def make(cid: int, scale: float = 1.0, k: int | None = None, m: int | None = None, seed: int | None = None) -> Workload:
    n0, k0, m0, p = SHAPES[cid]
    n = max(int(round(n0 * scale)), 4 * p)
    k = k0 if k is None else k
    m = m0 if m is None else m
    seed = SEEDS[cid] if seed is None else seed
    rng = np.random.default_rng(seed)
    if cid == 3:
        mu = rng.uniform(-10, 10, k)
        sigma = np.exp(rng.uniform(np.log(0.1), np.log(10), k))
        x = mu + sigma * rng.standard_t(5, size=(n, k))
    else:
        mu = rng.uniform(-5, 5, k)
        sigma = rng.uniform(0.5, 2, k)
        if cid == 2:
            sigma[rng.permutation(k)[: max(1, k // 10)]] = 1e-3
        x = mu + sigma * rng.standard_normal((n, k))
    b = rng.standard_normal((k, m))
    y = x @ b + 0.1 * rng.standard_normal((n, m)) + rng.uniform(-3, 3, m)
    dt = DTYPES[cid]
    return Workload(cid, np.ascontiguousarray(x, dt), np.ascontiguousarray(y, dt), _labels(cid, n, p, rng, seed), p,
                    list(CONFIGS[cid]), seed)


def make_device(cid: int, device, seed: int | None = None):
    """Full-size config generated on the GPU with torch (plumbing, not product):
    returns (x, y, labels) as CUDA tensors plus p and the configs."""
    import torch

    n, k, m, p = SHAPES[cid]
    seed = SEEDS[cid] if seed is None else seed
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    f64 = torch.float64
    if cid == 3:
        mu = torch.empty(k, device=device, dtype=f64).uniform_(-10, 10, generator=g)
        sigma = torch.exp(torch.empty(k, device=device, dtype=f64).uniform_(np.log(0.1), np.log(10), generator=g))
        z = torch.randn(n, k, device=device, dtype=torch.float32, generator=g)
        chi = torch.zeros(n, 1, device=device, dtype=torch.float32)
        for _ in range(5):
            chi += torch.randn(n, 1, device=device, dtype=torch.float32, generator=g) ** 2
        x = (mu.float() + sigma.float() * z / torch.sqrt(chi / 5.0)).contiguous()
        del z
    else:
        mu = torch.empty(k, device=device, dtype=f64).uniform_(-5, 5, generator=g)
        sigma = torch.empty(k, device=device, dtype=f64).uniform_(0.5, 2, generator=g)
        if cid == 2:
            idx = torch.randperm(k, device=device, generator=g)[: max(1, k // 10)]
            sigma[idx] = 1e-3
        x = torch.randn(n, k, device=device, dtype=f64, generator=g)
        x.mul_(sigma).add_(mu)
    b = torch.randn(k, m, device=device, dtype=x.dtype, generator=g)
    off = torch.empty(m, device=device, dtype=x.dtype).uniform_(-3, 3, generator=g)
    y = (x @ b + 0.1 * torch.randn(n, m, device=device, dtype=x.dtype, generator=g) + off).contiguous()
    rng = np.random.default_rng(seed)
    labels = torch.from_numpy(_labels(cid, n, p, rng, seed)).to(device)
    return x, y, labels, p, list(CONFIGS[cid])
