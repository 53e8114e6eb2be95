"""One process per GPU: row-sharded evaluation with an exact cross-rank sum.

The reference parallelises `count_matches` over contiguous row chunks
(make_chunk_plan, fitness.hpp:30-39) and sums per-chunk integer partials
(fitness.hpp:110-116); counts are therefore identical for any partition
(fitness.hpp:17-19).  Here each rank of a torch.distributed group holds the
rows `shard_range(total_rows, world, rank)` of the matrix on its own GPU and
counts its shard with the sm_100a kernel.  The cross-rank sum is either

* ``reduce="kernel"`` (default on GPUs): done by the count kernels themselves
  (include/ebic_b200.h, ebic_xgroup_*): each rank's final CTA adds its totals
  into one accumulator on rank 0's GPU through CUDA IPC peer memory; the last
  rank to finish writes whole-matrix counts + Eq. 1 into a shared-memory block
  every rank reads.  torch.distributed only carries the one-time handle
  exchange; or
* ``reduce="collective"``: one all-reduce of int64 partial counts (NCCL over
  NVLink on GPUs; any backend, the CPU tests use gloo), then Eq. 1 with the
  reference's arithmetic.
Either way every rank returns bit-identical counts and fitness.
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np

import ctypes as C
import os
import uuid

from . import (CbfPopulation, Evaluator, FitnessParams, shard_range)
from ._lib import check, f64p, lib, szp, u16p, u64p, vp

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
                 local_counter: Optional[LocalCounter] = None, reduce: str = "kernel",
                 max_series: int = 2048):
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
        if reduce not in ("kernel", "collective"):
            raise ValueError("reduce must be 'kernel' or 'collective'")
        self.rows = np.ascontiguousarray(rows, dtype=np.float64)
        self._ev = None
        self._xg = None
        self._device = device
        self._seq = 0
        self.max_series = int(max_series)
        if local_counter is None:
            dev = device if device is not None else 0
            self._device = dev
            self._ev = Evaluator(self.rows, devices=[dev], shard=(self.lo, total))
            local_counter = self._ev.count_matches
            if reduce == "kernel":
                self._join_group()
        self.reduce = "kernel" if self._xg is not None else "collective"
        self._local = local_counter

    def _join_group(self) -> None:
        """Rank 0 creates the accumulator + shared block; everyone joins.  If
        any rank cannot (no CUDA IPC in the container, no /dev/shm), all ranks
        fall back to the collective."""
        import torch
        handle = (C.c_ubyte * 64)()
        name = f"/ebic_{os.getpid()}_{uuid.uuid4().hex[:12]}"
        ok = 1
        if self.rank == 0:
            ok = int(lib.ebic_xgroup_create(self._ev.handle, self.max_series, name.encode(), handle) == 0)
        obj = [bytes(handle), name, ok]
        self.dist.broadcast_object_list(obj, src=self._src(), group=self.group)
        g = vp()
        ok = 0
        if obj[2]:
            hb = (C.c_ubyte * 64).from_buffer_copy(obj[0])
            ok = int(lib.ebic_xgroup_join(self._ev.handle, hb, obj[1].encode(), self.world,
                                          self.max_series, C.byref(g)) == 0)
        backend = self.dist.get_backend(self.group)
        agree = torch.tensor([ok], dtype=torch.int32,
                             device=torch.device("cuda", self._device) if backend == "nccl" else "cpu")
        self.dist.all_reduce(agree, op=self.dist.ReduceOp.MIN, group=self.group)
        if int(agree.item()):
            self._xg = g
        elif ok:
            check(lib.ebic_xgroup_destroy(g))
        self.dist.barrier(group=self.group)

    def _src(self) -> int:
        """Global rank of the group's rank 0 (broadcast source)."""
        if self.group is None:
            return 0
        return self.dist.get_global_rank(self.group, 0)

    def close(self) -> None:
        if self._xg is not None:
            # the owner (rank 0) frees the shared accumulator last
            if self.rank != 0:
                check(lib.ebic_xgroup_destroy(self._xg))
            self.dist.barrier(group=self.group)
            if self.rank == 0:
                check(lib.ebic_xgroup_destroy(self._xg))
            self._xg = None
        if self._ev is not None:
            self._ev.close()
            self._ev = None

    def _kernel_reduce(self, pop: CbfPopulation, epsilon: float, sigma: int, want_fit: bool):
        P = pop.size()
        off = np.ascontiguousarray(pop.offsets, dtype=np.uint64)
        cols = np.ascontiguousarray(pop.col_indices, dtype=np.uint16)
        if cols.size == 0:
            cols = np.zeros(1, dtype=np.uint16)
        counts = np.zeros(max(P, 1), dtype=np.uint64)
        fit = np.zeros(max(P, 1), dtype=np.float64) if want_fit else None
        self._seq += 1
        check(lib.ebic_xgroup_evaluate(self._xg, off.ctypes.data_as(szp), cols.ctypes.data_as(u16p), P,
                                       int(sigma), float(epsilon), self._seq,
                                       counts.ctypes.data_as(u64p),
                                       fit.ctypes.data_as(f64p) if want_fit else None))
        return counts[:P], (fit[:P] if want_fit else None)

    def _fits_kernel_reduce(self, pop: CbfPopulation) -> bool:
        # one count launch per call (every rank sees the same population, so
        # every rank takes the same branch)
        return (self._xg is not None and 0 < pop.size() <= min(self.max_series, 2048)
                and int(pop.offsets[-1]) <= 8192)

    def count_matches(self, pop: CbfPopulation, epsilon: float = 0.0) -> np.ndarray:
        """Global counts (fitness.hpp:100-118), identical on every rank."""
        if self._fits_kernel_reduce(pop):
            return self._kernel_reduce(pop, epsilon, 4, False)[0]
        import torch
        part = np.asarray(self._local(pop, epsilon), dtype=np.uint64)
        t = torch.from_numpy(part.astype(np.int64))
        if self.dist.get_backend(self.group) == "nccl":
            # NCCL reduces device tensors only: the partials go through this
            # rank's GPU (int64 sums are exact on any backend)
            dev = torch.device("cuda", self._device if self._device is not None
                               else torch.cuda.current_device())
            td = t.to(dev)
            self.dist.all_reduce(td, op=self.dist.ReduceOp.SUM, group=self.group)
            return td.cpu().numpy().astype(np.uint64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t.numpy().astype(np.uint64)

    def evaluate_population(self, pop: CbfPopulation, params: FitnessParams,
                            epsilon: float = 0.0) -> np.ndarray:
        """fitness.hpp:135-143 over the whole (sharded) matrix."""
        if self._fits_kernel_reduce(pop):
            return self._kernel_reduce(pop, epsilon, params.sigma, True)[1]
        counts = self.count_matches(pop, epsilon)
        return fitness_scores(counts, pop.offsets, params.sigma)
