"""BASELINE.json workloads c0–c4 (synthetic, seeded; SURVEY.md §8(d) pins the recipes).

c0/c1 are the reference bars generator (bars.cpp:33-65); c2–c4 draw a
unit-norm×5 random dictionary from RngStream::derived(seed, "wtru") and sample
data with LinearDiscreteModel::generate (linear_discrete.cpp:452-479). The
initial parameters follow BASELINE.json's recipe (W = mean_d + 0.25·std_d·z,
π = 1/H, σ² = mean data variance) and are identical for the oracle and the GPU.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import bsc


@dataclass(frozen=True)
class Workload:
    name: str
    D: int
    H: int
    hprime: int
    gamma: int
    N: int
    iters: int
    seed: int
    kind: str  # "bars" or "random"
    bars_size: int = 0
    pi_true: float = 0.0
    sigma2_true: float = 0.0
    dict_seed: int = 0
    scaling: str = "weak"  # "strong": N is the job's total, sharded over the ranks

    def describe(self) -> dict:
        return dict(workload=self.name, D=self.D, H=self.H, hprime=self.hprime, gamma=self.gamma, N=self.N,
                    seed=self.seed)


CONFIGS = {
    "c0": Workload("c0_bars5x5_exact", 25, 10, 10, 10, 1_000, 50, 0, "bars", bars_size=5),
    "c1": Workload("c1_bars10x10", 100, 20, 10, 4, 10_000, 50, 1, "bars", bars_size=10),
    "c2": Workload("c2_random_D256_H300", 256, 300, 12, 4, 200_000, 20, 2, "random", pi_true=5 / 300,
                   sigma2_true=0.25, dict_seed=2),
    "c3": Workload("c3_random_D576_H1000", 576, 1000, 14, 5, 1_000_000, 10, 3, "random", pi_true=8 / 1000,
                   sigma2_true=0.25, dict_seed=3),
    "c4": Workload("c4_strong_D576_H1000_N4M", 576, 1000, 14, 5, 4_000_000, 10, 4, "random", pi_true=8 / 1000,
                   sigma2_true=0.25, dict_seed=3, scaling="strong"),
    # not a BASELINE config: a shape outside the compile-time lane walks ((10,4), (12,4), (14,5)), to time
    # the run-time-H' state pass (lane_states_kernel<γ>) that every other (H', γ) takes
    "g1": Workload("g1_random_D128_H200_generic", 128, 200, 8, 3, 200_000, 20, 5, "random", pi_true=4 / 200,
                   sigma2_true=0.25, dict_seed=5),
}


class _ProductGen:
    """The package's own fixtures (csrc/fixtures.cpp, the reference's draw order)."""

    @staticmethod
    def random_dictionary(d, h, seed, scale):
        return bsc.random_dictionary(d, h, seed, scale)

    @staticmethod
    def generate(w, pi, sigma2, n, seed):
        return bsc.generate(bsc.BscParams(w, pi, sigma2), n, seed)

    @staticmethod
    def make_bars(size, n, seed):
        return bsc.bars_generate(size, n, seed=seed)


class OracleGen:
    """The same fixtures from the oracle library (bit-identical draws), so that a
    caller timing the reference never maps the product's library."""

    def __init__(self, orc):
        self.o = orc

    def random_dictionary(self, d, h, seed, scale):
        return self.o.random_dictionary(d, h, seed, scale)

    def generate(self, w, pi, sigma2, n, seed):
        return self.o.generate(w, pi, sigma2, n, seed)

    def make_bars(self, size, n, seed):
        return self.o.make_bars(size, n, seed=seed)


# c4 (strong scaling) is generated in fixed blocks of BLOCK points, block b from
# RngStream(block_seed(seed, b)): a rank can draw exactly its rows of the global
# dataset, and every world size (1, 2, 4, 8) shards the same 4M points.
BLOCK = 250_000


def block_seed(seed: int, b: int) -> int:
    return (seed << 20) | b


def truth(w: Workload, gen=None) -> np.ndarray:
    gen = gen or _ProductGen
    if w.kind == "bars":
        _, t = gen.make_bars(w.bars_size, 1, w.seed)
        return t
    return gen.random_dictionary(w.D, w.H, w.dict_seed, 5.0)


def data(w: Workload, n: int | None = None, seed_offset: int = 0, gen=None, rows=None) -> np.ndarray:
    """The workload's data points (first ``n`` of the seeded stream for bars;
    an independent seeded sample of size ``n`` for the random dictionaries).
    Strong-scaling workloads (c4) are blocked: ``rows=(b, e)`` returns global
    rows [b, e) of the N-point dataset, identical whatever the sharding."""
    gen = gen or _ProductGen
    if w.scaling == "strong":
        b, e = rows if rows is not None else (0, w.N if n is None else int(n))
        wt = truth(w, gen)
        parts = []
        for blk in range(b // BLOCK, (e + BLOCK - 1) // BLOCK):
            lo, hi = blk * BLOCK, (blk + 1) * BLOCK
            y = gen.generate(wt, w.pi_true, w.sigma2_true, BLOCK, block_seed(w.seed, blk))
            parts.append(y[max(b, lo) - lo:min(e, hi) - lo])
        return np.ascontiguousarray(np.concatenate(parts)) if len(parts) > 1 else np.ascontiguousarray(parts[0])
    n = w.N if n is None else int(n)
    if w.kind == "bars":
        y, _ = gen.make_bars(w.bars_size, n, w.seed + seed_offset)
        return y
    wt = truth(w, gen)
    return gen.generate(wt, w.pi_true, w.sigma2_true, n, w.seed + seed_offset)


def init(w: Workload, y: np.ndarray, gen_oracle=None) -> bsc.BscParams:
    if gen_oracle is not None:
        wi, pi, s2 = gen_oracle.baseline_init(y, w.H, w.seed)
        return bsc.BscParams(wi, pi, s2)
    return bsc.baseline_init(y, w.H, w.seed)
