"""Synthetic workloads of BASELINE.json (SURVEY.md §8d recipe): low-rank-plus-noise tensors assembled from the
reference's own seeded primitives.  Config c (1..5):

    G   = random_tensor(K, seed=1000c+1)
    A_n = thin-Q factors from the random_decomposition stream with seed 1000c+2
    X   = G x_0 A_0 ... x_{N-1} A_{N-1}
    E   = random_tensor(L, seed=1000c+3)          (slab-parallel variant for C4/C5: slab i of mode 0 is
                                                    random_tensor(L[1:], 1000c+3+i))
    T   = X + sigma E;  start factors: seed 1000c+4; schedule: Jacobi on optimal_tree(spec); iterations below.

This is input generation for tests and bench — neither the product path nor the oracle.
"""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import List

import numpy as np

from . import hostgen
from .planner import ProblemSpec


@dataclass
class Config:
    index: int
    L: List[int]
    K: List[int]
    sigma: float
    iterations: int
    slab_noise: bool = False

    @property
    def spec(self) -> ProblemSpec:
        return ProblemSpec(list(self.L), list(self.K))

    @property
    def name(self) -> str:
        return "C%d_%s_to_%s" % (self.index, "x".join(map(str, self.L)), "x".join(map(str, self.K)))


CONFIGS = {
    1: Config(1, [200] * 3, [20] * 3, 1e-3, 5),
    2: Config(2, [96] * 4, [10] * 4, 1e-3, 10),
    3: Config(3, [400, 100, 100, 50], [40, 10, 20, 5], 1e-2, 10),
    4: Config(4, [48] * 5, [8] * 5, 1e-3, 10, slab_noise=True),
    5: Config(5, [1600] * 3, [100] * 3, 1e-3, 5, slab_noise=True),
}


def scaled_config(index: int, L, K, iterations=None) -> Config:
    """Same recipe and seeds as config `index` at reduced extents (parity-test sizes)."""
    base = CONFIGS[index]
    return Config(index, list(L), list(K), base.sigma, iterations or base.iterations, base.slab_noise)


def _expand_host(core: np.ndarray, factors) -> np.ndarray:
    z = core
    for n, a in enumerate(factors):
        z = np.moveaxis(np.tensordot(a, z, axes=(1, n)), 0, n)
    return np.ascontiguousarray(z)


def noise_into(cfg: Config, out: np.ndarray, threads: int = 8) -> None:
    """Writes E into `out` (shape L, C-contiguous)."""
    seed = 1000 * cfg.index + 3
    if not cfg.slab_noise:
        hostgen.random_tensor(cfg.L, seed, out.reshape(-1))
        return
    flat = out.reshape(cfg.L[0], -1)

    def one(i):
        hostgen.random_tensor(cfg.L[1:], seed + i, flat[i])

    with ThreadPoolExecutor(max_workers=threads) as pool:  # the C call releases the GIL
        list(pool.map(one, range(cfg.L[0])))


def generating_factors(cfg: Config):
    return hostgen.random_orthonormal_factors(cfg.L, cfg.K, 1000 * cfg.index + 2)


def generating_core(cfg: Config) -> np.ndarray:
    return hostgen.random_tensor(cfg.K, 1000 * cfg.index + 1)


def start_factors(cfg: Config):
    return hostgen.random_orthonormal_factors(cfg.L, cfg.K, 1000 * cfg.index + 4)


def build_tensor_host(cfg: Config, threads: int = 8) -> np.ndarray:
    """T on the host with NumPy (small and medium configs)."""
    t = np.empty(cfg.L, dtype=np.float64)
    noise_into(cfg, t, threads)
    t *= cfg.sigma
    t += _expand_host(generating_core(cfg), generating_factors(cfg))
    return t
