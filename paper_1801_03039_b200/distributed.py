"""One process per GPU: row-sharded evaluation with an exact count all-reduce.

The reference parallelises `count_matches` over contiguous row chunks
(make_chunk_plan, fitness.hpp:30-39) and sums per-chunk integer partials
(fitness.hpp:110-116); counts are therefore identical for any partition
(fitness.hpp:17-19).  Here each rank of a torch.distributed group holds the
rows `shard_range(total_rows, world, rank)` of the matrix on its own GPU,
counts its shard with the sm_100a kernel, and the per-series partial counts are
summed with one all-reduce of int64 (NCCL over NVLink on GPUs; any backend
works, the tests use gloo).  Eq. 1 is then applied to the reduced counts with
the reference's arithmetic, so every rank returns bit-identical fitness.
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np

from . import (CbfPopulation, Evaluator, FitnessParams, shard_range)
from ._lib import check, f64p, lib, szp, u64p

LocalCounter = Callable[[CbfPopulation, float], np.ndarray]


def fitness_scores(counts: np.ndarray, offsets: np.ndarray, sigma: int) -> np.ndarray:
    """Eq. 1 (fitness.hpp:124-133) for a whole population on the host, same libm."""
    counts = np.ascontiguousarray(counts, dtype=np.uint64)
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    out = np.empty(len(counts), dtype=np.float64)
    if len(counts):
        check(lib.ebic_fitness_scores_host(counts.ctypes.data_as(u64p), off.ctypes.data_as(szp),
                                           len(counts), int(sigma), out.ctypes.data_as(f64p)))
    return out


class RowShardedEvaluator:
    """Evaluation over a row-sharded matrix, one rank per GPU.

    ``values`` may be the full matrix (each rank keeps its shard) or just this
    rank's rows (``is_shard=True``).  ``local_counter`` overrides the per-shard
    count (tests inject the CPU oracle to exercise the orchestration without a
    GPU); by default it is the B200 kernel through the C ABI.
    """

    def __init__(self, values: np.ndarray, total_rows: Optional[int] = None, group=None,
                 device: Optional[int] = None, is_shard: bool = False,
                 local_counter: Optional[LocalCounter] = None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        total = total_rows if total_rows is not None else values.shape[0]
        self.total_rows = total
        self.lo, self.hi = shard_range(total, self.world, self.rank)
        rows = values if is_shard else values[self.lo:self.hi]
        if rows.shape[0] != self.hi - self.lo:
            raise ValueError("shard rows do not match shard_range")
        self.rows = np.ascontiguousarray(rows, dtype=np.float64)
        self._ev = None
        if local_counter is None:
            dev = device if device is not None else 0
            self._ev = Evaluator(self.rows, devices=[dev], shard=(self.lo, total))
            local_counter = self._ev.count_matches
        self._local = local_counter

    def close(self) -> None:
        if self._ev is not None:
            self._ev.close()
            self._ev = None

    def count_matches(self, pop: CbfPopulation, epsilon: float = 0.0) -> np.ndarray:
        """Global counts (fitness.hpp:100-118), identical on every rank."""
        import torch
        part = np.asarray(self._local(pop, epsilon), dtype=np.uint64)
        t = torch.from_numpy(part.astype(np.int64))
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t.numpy().astype(np.uint64)

    def evaluate_population(self, pop: CbfPopulation, params: FitnessParams,
                            epsilon: float = 0.0) -> np.ndarray:
        """fitness.hpp:135-143 over the whole (sharded) matrix."""
        counts = self.count_matches(pop, epsilon)
        return fitness_scores(counts, pop.offsets, params.sigma)
