"""B200-native EBIC fitness-evaluation hot path (host-side mirror of the reference API).

The reference (arxiv/paper_1801_03039) is a header-only C++20 library whose
evolutionary loop calls free functions in ``ebic/fitness.hpp`` and
``ebic/expansion.hpp``.  This module mirrors those functions -- same names,
same argument meaning, same exceptions and messages -- on top of the C ABI of
``libebic_b200.so`` (include/ebic_b200.h), whose sm_100a kernels do the work.
The C++ drop-in for the reference's own build is include/ebic/fitness.hpp and
include/ebic/expansion.hpp.

Reference file:line citations are relative to /root/reference/proj/include/ebic/.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import os
from dataclasses import dataclass, field
from typing import Iterable, List, Optional, Sequence

import numpy as np

from ._lib import (CtxInfo, EbicError, check, f64p, fast_count, fast_evaluate, i64p, lib, ptr,
                   szp, u8p, u16p, u64p)

__all__ = [
    "ExpressionMatrix", "CbfPopulation", "ColumnSeries", "RowRange", "ChunkPlan", "FitnessParams",
    "RowFlag", "Bicluster", "ExpansionOptions", "ScenarioSpec", "Pattern", "EbicError",
    "K_MIN_SERIES_LENGTH", "series_has_distinct_columns", "is_valid_series", "encode_population",
    "decode_population", "make_chunk_plan", "default_sigma", "fitness_score", "row_matches",
    "count_matches", "evaluate_population", "assign_rows", "trend_violations",
    "resolve_bicluster", "expand_bicluster", "finalize_biclusters", "Evaluator", "synth_generate",
    "device_count", "shard_range", "TopRankEntry", "TopRankList",
]

ColumnSeries = List[int]
K_MIN_SERIES_LENGTH = 2  # cbf.hpp:18


# ---------------------------------------------------------------------------
# L0 data model (matrix.hpp:21-44, cbf.hpp:15-86, bicluster.hpp:11-22)
# ---------------------------------------------------------------------------
class ExpressionMatrix:
    """Row-major fp64 matrix (matrix.hpp:21-44).  ``values`` is (n_rows, n_cols)."""

    def __init__(self, values: np.ndarray):
        v = np.ascontiguousarray(values, dtype=np.float64)
        if v.ndim != 2:
            raise ValueError("matrix must be 2-D")
        self.values = v

    @property
    def n_rows(self) -> int:
        return self.values.shape[0]

    @property
    def n_cols(self) -> int:
        return self.values.shape[1]

    @staticmethod
    def with_shape(rows: int, cols: int) -> "ExpressionMatrix":
        return ExpressionMatrix(np.zeros((rows, cols)))


@dataclass
class CbfPopulation:
    """Two-array population encoding (cbf.hpp:43-52): offsets[P+1], col_indices."""

    offsets: np.ndarray = field(default_factory=lambda: np.zeros(1, dtype=np.uint64))
    col_indices: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.uint16))

    def size(self) -> int:
        return 0 if len(self.offsets) == 0 else len(self.offsets) - 1

    def individual(self, p: int) -> np.ndarray:
        return self.col_indices[int(self.offsets[p]):int(self.offsets[p + 1])]


def series_has_distinct_columns(s: Sequence[int]) -> bool:  # cbf.hpp:20-30
    return len(set(int(c) for c in s)) == len(s)


def is_valid_series(s: Sequence[int], n_cols: int) -> bool:  # cbf.hpp:32-37
    if len(s) < K_MIN_SERIES_LENGTH:
        return False
    if any(int(c) >= n_cols for c in s):
        return False
    return series_has_distinct_columns(s)


def encode_population(individuals: Sequence[Sequence[int]]) -> CbfPopulation:
    """cbf.hpp:54-68 -- same checks and messages."""
    if len(individuals) == 0:
        raise ValueError("empty population")
    lens = np.fromiter((len(s) for s in individuals), dtype=np.uint64, count=len(individuals))
    for s in individuals:
        if len(s) < K_MIN_SERIES_LENGTH or not series_has_distinct_columns(s):
            raise ValueError("invalid series")
    offsets = np.zeros(len(individuals) + 1, dtype=np.uint64)
    np.cumsum(lens, out=offsets[1:])
    cols = np.fromiter((int(c) for s in individuals for c in s), dtype=np.uint16,
                       count=int(offsets[-1]))
    return CbfPopulation(offsets, cols)


def decode_population(cbf: CbfPopulation) -> List[ColumnSeries]:
    """cbf.hpp:70-86 -- same corruption checks ("corrupt CBF")."""
    off = [int(x) for x in cbf.offsets]
    if len(off) < 2 or off[0] != 0:
        raise RuntimeError("corrupt CBF")
    for i in range(1, len(off)):
        if off[i] <= off[i - 1] or off[i] - off[i - 1] < K_MIN_SERIES_LENGTH:
            raise RuntimeError("corrupt CBF")
    if off[-1] != len(cbf.col_indices):
        raise RuntimeError("corrupt CBF")
    return [[int(c) for c in cbf.individual(p)] for p in range(cbf.size())]


class RowFlag(enum.IntEnum):  # bicluster.hpp:11-15
    kExact = 0
    kNegative = 1
    kApproximate = 2


@dataclass
class Bicluster:  # bicluster.hpp:17-22
    rows: List[int] = field(default_factory=list)
    series: ColumnSeries = field(default_factory=list)
    fitness: float = 0.0
    row_flags: List[RowFlag] = field(default_factory=list)


@dataclass
class ExpansionOptions:  # expansion.hpp:46-49
    allow_negative: bool = True
    approx_violations: int = 1


@dataclass
class FitnessParams:  # fitness.hpp:41-45
    sigma: int = 4


@dataclass
class RowRange:  # fitness.hpp:20-23
    lo: int = 0
    hi: int = 0


@dataclass
class ChunkPlan:  # fitness.hpp:25-28
    chunks: List[RowRange] = field(default_factory=list)
    worker_count: int = 1


def make_chunk_plan(n_rows: int, workers: int = 0) -> ChunkPlan:
    """fitness.hpp:30-39.  On the B200 path chunks map to per-device row shards;
    counts are partition invariant, so the plan never changes results."""
    if n_rows == 0:
        raise ValueError("matrix has no rows")
    if workers == 0:
        workers = max(1, os.cpu_count() or 1)
    chunk = (n_rows + workers - 1) // workers
    return ChunkPlan([RowRange(lo, min(lo + chunk, n_rows)) for lo in range(0, n_rows, chunk)],
                     workers)


def default_sigma(n_rows: int) -> int:  # fitness.hpp:48-52
    return int(lib.ebic_default_sigma(n_rows))


def fitness_score(match_count: int, series_len: int, params: FitnessParams) -> float:
    """fitness.hpp:124-133 (host glibc log/exp2, identical arithmetic)."""
    return float(lib.ebic_fitness_score(int(match_count), int(series_len), int(params.sigma)))


def row_matches(m: ExpressionMatrix, row: int, series: Sequence[int], epsilon: float = 0.0) -> bool:
    """fitness.hpp:57-67 -- single-row predicate (host; not a hot path)."""
    v = m.values[row]
    prev = float(v[series[0]])
    for c in series[1:]:
        cur = float(v[c])
        if not (prev < cur + epsilon):
            return False
        prev = cur
    return True


def trend_violations(m: ExpressionMatrix, row: int, series: Sequence[int],
                     epsilon: float = 0.0) -> int:
    """expansion.hpp:26-33 -- single-row violation count (host)."""
    v = m.values[row]
    return sum(1 for i in range(1, len(series))
               if not (float(v[series[i - 1]]) < float(v[series[i]]) + epsilon))


# ---------------------------------------------------------------------------
# Device context: the evaluation engine (replaces ThreadPool + count_chunk)
# ---------------------------------------------------------------------------
def device_count() -> int:
    n = C.c_int(0)
    check(lib.ebic_device_count(C.byref(n)))
    return n.value


_ONE_COL = np.zeros(1, dtype=np.uint16)


def _as_cbf_arrays(pop: CbfPopulation):
    off, cols = pop.offsets, pop.col_indices
    if off.dtype != np.uint64 or not off.flags.c_contiguous:
        off = np.ascontiguousarray(off, dtype=np.uint64)
    if cols.dtype != np.uint16 or not cols.flags.c_contiguous:
        cols = np.ascontiguousarray(cols, dtype=np.uint16)
    if cols.size == 0:
        cols = _ONE_COL
    return off, cols


def shard_range(total_rows: int, world_size: int, rank: int) -> tuple:
    """Contiguous row shard [lo, hi) of one rank: make_chunk_plan's contiguous
    chunking (fitness.hpp:30-39) with 64-row aligned boundaries, so per-shard
    membership bitmask words concatenate.  Counts are partition invariant
    (fitness.hpp:17-19), so any world size gives identical results."""
    if total_rows == 0:
        raise ValueError("matrix has no rows")
    if world_size <= 0 or not (0 <= rank < world_size):
        raise ValueError("invalid rank")
    per = -(-total_rows // world_size)
    per = -(-per // 64) * 64
    lo = min(rank * per, total_rows)
    return lo, min(lo + per, total_rows)


class Evaluator:
    """One device context holding a matrix (or a row shard of it) in HBM.

    ``devices``: list of CUDA device ids; rows are sharded over them (64-row
    aligned contiguous ranges) and partial counts reduced exactly.
    ``shard=(row_begin, total_rows)``: hold only ``matrix`` rows as the global
    rows [row_begin, row_begin + len) of a total_rows matrix (one process per
    GPU); counts are then partial and must be all-reduced by the caller.
    """

    def __init__(self, matrix, devices: Optional[Sequence[int]] = None,
                 shard: Optional[tuple] = None):
        m = matrix.values if isinstance(matrix, ExpressionMatrix) else np.ascontiguousarray(
            matrix, dtype=np.float64)
        m = np.ascontiguousarray(m, dtype=np.float64)
        if m.ndim != 2:
            raise ValueError("matrix must be 2-D")
        self.n_cols = m.shape[1]
        self._ctx = C.c_void_p()
        if shard is None:
            if m.shape[0] == 0:
                raise ValueError("matrix has no rows")
            devs = (C.c_int * len(devices))(*devices) if devices else None
            check(lib.ebic_ctx_create(ptr(m, f64p), m.shape[0], m.shape[1], devs,
                                      len(devices) if devices else 0, C.byref(self._ctx)))
            self.row_begin, self.total_rows = 0, m.shape[0]
        else:
            row_begin, total_rows = shard
            dev = devices[0] if devices else 0
            check(lib.ebic_ctx_create_shard(ptr(m, f64p), m.shape[0], m.shape[1], total_rows,
                                            row_begin, dev, C.byref(self._ctx)))
            self.row_begin, self.total_rows = row_begin, total_rows
        self.n_rows = m.shape[0]

    @classmethod
    def from_device(cls, d_ptr: int, shard_rows: int, n_cols: int, total_rows: int,
                    row_begin: int, device: int) -> "Evaluator":
        self = cls.__new__(cls)
        self._ctx = C.c_void_p()
        check(lib.ebic_ctx_create_shard_device(C.c_void_p(d_ptr), shard_rows, n_cols, total_rows,
                                               row_begin, device, C.byref(self._ctx)))
        self.n_cols, self.n_rows = n_cols, shard_rows
        self.row_begin, self.total_rows = row_begin, total_rows
        return self

    def close(self) -> None:
        if getattr(self, "_ctx", None) and self._ctx.value:
            check(lib.ebic_ctx_destroy(self._ctx))
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self) -> C.c_void_p:
        return self._ctx

    def info(self) -> CtxInfo:
        i = CtxInfo()
        check(lib.ebic_ctx_get_info(self._ctx, C.byref(i)))
        return i

    # -- fitness.hpp:100-118 ------------------------------------------------
    def count_matches(self, pop: CbfPopulation, epsilon: float = 0.0) -> np.ndarray:
        off, cols = _as_cbf_arrays(pop)
        n = len(off) - 1
        out = np.empty(max(n, 0), dtype=np.uint64)
        if n <= 0:
            return out
        rc = fast_count(self._ctx, off.ctypes.data, cols.ctypes.data, n, float(epsilon),
                        out.ctypes.data)
        if rc:
            check(rc)
        return out

    # -- fitness.hpp:135-143 ------------------------------------------------
    def evaluate_population(self, pop: CbfPopulation, params: FitnessParams,
                            epsilon: float = 0.0, return_counts: bool = False):
        off, cols = _as_cbf_arrays(pop)
        n = max(len(off) - 1, 0)
        fit = np.empty(n, dtype=np.float64)
        counts = np.empty(n, dtype=np.uint64) if return_counts else None
        if n:
            rc = fast_evaluate(self._ctx, off.ctypes.data, cols.ctypes.data, n, int(params.sigma),
                               float(epsilon), counts.ctypes.data if return_counts else None,
                               fit.ctypes.data)
            if rc:
                check(rc)
        return (fit, counts) if return_counts else fit

    # -- membership (expansion.hpp:16-87) ------------------------------------
    def membership_bits(self, pop: CbfPopulation, epsilon: float = 0.0, approx_k: int = 1):
        n = pop.size()
        words = (self.n_rows + 63) // 64
        ex = np.zeros((n, words), dtype=np.uint64)
        ng = np.zeros((n, words), dtype=np.uint64)
        ap = np.zeros((n, words), dtype=np.uint64)
        if n:
            off, cols = _as_cbf_arrays(pop)
            check(lib.ebic_membership_bits(self._ctx, ptr(off, szp), ptr(cols, u16p), n,
                                           float(epsilon), int(approx_k), ptr(ex, u64p),
                                           ptr(ng, u64p), ptr(ap, u64p)))
        return ex, ng, ap

    def assign_rows(self, series: Sequence[int], epsilon: float = 0.0) -> List[int]:
        s = np.ascontiguousarray(series, dtype=np.uint16)
        if s.size == 0:
            raise ValueError("invalid series")
        if int(s.max()) >= self.n_cols:
            raise ValueError("invalid series")
        rows = np.zeros(self.n_rows, dtype=np.uint64)
        n = C.c_size_t(0)
        check(lib.ebic_assign_rows(self._ctx, ptr(s, u16p), s.size, float(epsilon), ptr(rows, u64p),
                                   C.byref(n)))
        return [int(r) for r in rows[:n.value]]

    def resolve_bicluster(self, series: Sequence[int], fitness: float,
                          epsilon: float = 0.0) -> Bicluster:
        rows = self.assign_rows(series, epsilon)
        return Bicluster(rows, [int(c) for c in series], fitness, [RowFlag.kExact] * len(rows))

    def expand_bicluster(self, b: Bicluster, opts: ExpansionOptions,
                         epsilon: float = 0.0) -> Bicluster:
        s = np.ascontiguousarray(b.series, dtype=np.uint16)
        if s.size == 0 or int(s.max()) >= self.n_cols:
            raise ValueError("invalid series")
        core = np.ascontiguousarray(b.rows, dtype=np.uint64)
        flags = np.ascontiguousarray([int(f) for f in b.row_flags], dtype=np.uint8)
        if core.size == 0:
            core = np.zeros(1, dtype=np.uint64)
            flags = np.zeros(1, dtype=np.uint8)
            n_core = 0
        else:
            n_core = len(b.rows)
        cap = self.n_rows + n_core
        rows = np.zeros(cap, dtype=np.uint64)
        rflags = np.zeros(cap, dtype=np.uint8)
        n = C.c_size_t(0)
        check(lib.ebic_expand_bicluster(self._ctx, ptr(s, u16p), s.size, ptr(core, u64p),
                                        ptr(flags, u8p), n_core, int(bool(opts.allow_negative)),
                                        int(opts.approx_violations), float(epsilon),
                                        ptr(rows, u64p), ptr(rflags, u8p), C.byref(n)))
        k = n.value
        return Bicluster([int(r) for r in rows[:k]], list(b.series), b.fitness,
                         [RowFlag(int(f)) for f in rflags[:k]])

    def resolve_expand_batch(self, series_list: Sequence[Sequence[int]], opts: ExpansionOptions,
                             epsilon: float = 0.0):
        """resolve_bicluster + expand_bicluster for many series in one launch.
        Returns a list of (rows, flags) numpy pairs."""
        if len(series_list) == 0:
            return []
        pop = encode_population(series_list)
        off, cols = _as_cbf_arrays(pop)
        n = pop.size()
        rows = np.zeros(n * self.n_rows, dtype=np.uint64)
        flags = np.zeros(n * self.n_rows, dtype=np.uint8)
        counts = np.zeros(n, dtype=np.uint64)
        check(lib.ebic_resolve_expand_batch(self._ctx, ptr(off, szp), ptr(cols, u16p), n,
                                            int(bool(opts.allow_negative)),
                                            int(opts.approx_violations), float(epsilon),
                                            ptr(rows, u64p), ptr(flags, u8p),
                                            counts.ctypes.data_as(szp)))
        out, at = [], 0
        for c in counts:
            c = int(c)
            out.append((rows[at:at + c].copy(), flags[at:at + c].copy()))
            at += c
        return out


# ---------------------------------------------------------------------------
# Reference-signature free functions (fitness.hpp / expansion.hpp / io.hpp).
# The reference passes the matrix on every call; like include/ebic/fitness.hpp
# the device copy is cached per matrix object (matrices are immutable by
# convention, matrix.hpp:18-20).
# ---------------------------------------------------------------------------
_CACHE: dict = {}


def _evaluator_for(m: ExpressionMatrix) -> Evaluator:
    key = id(m)
    hit = _CACHE.get(key)
    if hit is not None and hit[0] is m and hit[1] is m.values:
        return hit[2]
    if len(_CACHE) > 4:
        _CACHE.clear()
    ev = Evaluator(m)
    _CACHE[key] = (m, m.values, ev)
    return ev


def count_matches(m: ExpressionMatrix, pop: CbfPopulation, plan: ChunkPlan,
                  epsilon: float = 0.0) -> List[int]:
    """fitness.hpp:100-118.  ``plan`` is accepted for signature parity; the result
    is partition invariant (fitness.hpp:17-19)."""
    if pop.size() == 0:
        return []
    return [int(c) for c in _evaluator_for(m).count_matches(pop, epsilon)]


def evaluate_population(m: ExpressionMatrix, pop: CbfPopulation, plan: ChunkPlan,
                        params: FitnessParams, epsilon: float = 0.0) -> List[float]:
    """fitness.hpp:135-143."""
    if pop.size() == 0:
        return []
    return [float(f) for f in _evaluator_for(m).evaluate_population(pop, params, epsilon)]


def assign_rows(m: ExpressionMatrix, series: Sequence[int], epsilon: float = 0.0) -> List[int]:
    """expansion.hpp:16-23."""
    return _evaluator_for(m).assign_rows(series, epsilon)


def resolve_bicluster(m: ExpressionMatrix, series: Sequence[int], fitness: float,
                      epsilon: float = 0.0) -> Bicluster:
    """expansion.hpp:36-44."""
    return _evaluator_for(m).resolve_bicluster(series, fitness, epsilon)


def expand_bicluster(m: ExpressionMatrix, b: Bicluster, opts: ExpansionOptions,
                     epsilon: float = 0.0) -> Bicluster:
    """expansion.hpp:56-87."""
    return _evaluator_for(m).expand_bicluster(b, opts, epsilon)


def null_fitness_plateau(n_rows: int, sigma: int) -> float:
    """io.hpp:132-143 (host)."""
    params = FitnessParams(sigma)
    best, factorial = 0.0, 2.0
    for mlen in range(2, 21):
        # std::llround: round half away from zero
        x = n_rows / factorial
        expected = int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))
        best = max(best, fitness_score(expected, mlen, params))
        factorial *= float(mlen + 1)
    return best


def finalize_biclusters(entries: Sequence[tuple], m: ExpressionMatrix, expansion: ExpansionOptions,
                        epsilon: float, min_fitness: float, max_biclusters: int = 100
                        ) -> List[Bicluster]:
    """io.hpp:164-178 with the threshold already resolved (resolve_min_fitness,
    io.hpp:152-160).  ``entries`` = [(series, fitness), ...] in top-rank order.
    All kept series are resolved and expanded in one membership launch."""
    kept = []
    for series, fit in entries:
        if len(kept) >= max_biclusters:
            break
        if fit < min_fitness:
            continue
        kept.append((list(series), fit))
    if not kept:
        return []
    res = _evaluator_for(m).resolve_expand_batch([s for s, _ in kept], expansion, epsilon)
    return [Bicluster([int(r) for r in rows], s, f, [RowFlag(int(x)) for x in flags])
            for (s, f), (rows, flags) in zip(kept, res)]


# ---------------------------------------------------------------------------
# Top-rank list (evolution.hpp:132-218) -- host, exact, via ebic_top_rank_update
# ---------------------------------------------------------------------------
@dataclass
class TopRankEntry:  # evolution.hpp:132-137
    series: List[int]
    fitness: float
    seq: int


class TopRankList:
    """Best biclusters found so far (evolution.hpp:142-218).

    Same admission / eviction / tie semantics as the reference's
    ``TopRankList::update`` (:168-206), computed by ``ebic_top_rank_update``
    (posting-list overlap counting in libebic_b200.so).  The list is held as
    CBF arrays so an update passes it to the library without re-encoding.
    """

    def __init__(self, n_cols: int):
        self.n_cols = int(n_cols)
        self._off = np.zeros(1, dtype=np.uint64)
        self._cols = np.zeros(0, dtype=np.uint16)
        self._fit = np.zeros(0, dtype=np.float64)
        self._seq = np.zeros(0, dtype=np.uint64)
        self._next_seq = C.c_uint64(0)

    def size(self) -> int:
        return len(self._fit)

    __len__ = size

    def empty(self) -> bool:
        return len(self._fit) == 0

    def best_fitness(self) -> float:  # :151
        return float(self._fit[0]) if len(self._fit) else 0.0

    def entries(self) -> List[TopRankEntry]:  # :148
        return [TopRankEntry([int(c) for c in self._cols[int(self._off[i]):int(self._off[i + 1])]],
                             float(self._fit[i]), int(self._seq[i])) for i in range(len(self._fit))]

    @staticmethod
    def overlap(a, b) -> float:  # :154-160 (TopRankEntry or plain series)
        a = a.series if hasattr(a, "series") else a
        b = b.series if hasattr(b, "series") else b
        return len(set(int(x) for x in a) & set(int(x) for x in b)) / min(len(a), len(b))

    def update(self, population, fitness, overlap_threshold: float = 0.75,
               top_rank_capacity: int = 100) -> None:
        """:168-206.  ``population`` is a CbfPopulation or a sequence of series;
        ``overlap_threshold`` may also be an EvolutionConfig-like object."""
        if hasattr(overlap_threshold, "overlap_threshold"):
            cfg = overlap_threshold
            overlap_threshold, top_rank_capacity = cfg.overlap_threshold, cfg.top_rank_capacity
        if not isinstance(population, CbfPopulation):
            lens = np.fromiter((len(s) for s in population), dtype=np.uint64, count=len(population))
            off = np.zeros(len(population) + 1, dtype=np.uint64)
            np.cumsum(lens, out=off[1:])
            cols = np.fromiter((int(c) for s in population for c in s), dtype=np.uint16,
                               count=int(off[-1]))
            population = CbfPopulation(off, cols)
        c_off = np.ascontiguousarray(population.offsets, dtype=np.uint64)
        c_cols = np.ascontiguousarray(population.col_indices, dtype=np.uint16)
        fit = np.ascontiguousarray(fitness, dtype=np.float64)
        n_cand = len(c_off) - 1
        if len(fit) != n_cand:
            raise ValueError("fitness and population sizes differ")
        n_ent = len(self._fit)
        cap = max(1, min(int(top_rank_capacity), n_ent + n_cand))  # output slots
        ref = np.zeros(cap, dtype=np.int64)
        seq = np.zeros(cap, dtype=np.uint64)
        n_out = C.c_size_t(0)
        pad = lambda a: a if a.size else np.zeros(1, dtype=a.dtype)  # noqa: E731
        e_cols, k_cols = pad(self._cols), pad(c_cols)
        check(lib.ebic_top_rank_update(
            self.n_cols, n_ent, ptr(self._off, szp), ptr(e_cols, u16p), ptr(pad(self._fit), f64p),
            ptr(pad(self._seq), u64p), n_cand, ptr(c_off, szp), ptr(k_cols, u16p), ptr(pad(fit), f64p),
            float(overlap_threshold), int(top_rank_capacity), C.byref(self._next_seq),
            ptr(ref, i64p), ptr(seq, u64p), C.byref(n_out)))
        n = n_out.value
        ref, seq = ref[:n], seq[:n]
        # Gather the new list (entries referenced by index, candidates by -(p + 1)).
        segs, new_fit = [], np.empty(n, dtype=np.float64)
        for i, r in enumerate(ref.tolist()):
            if r < 0:
                p = -r - 1
                segs.append(c_cols[int(c_off[p]):int(c_off[p + 1])])
                new_fit[i] = fit[p]
            else:
                segs.append(self._cols[int(self._off[r]):int(self._off[r + 1])])
                new_fit[i] = self._fit[r]
        new_off = np.zeros(n + 1, dtype=np.uint64)
        np.cumsum([len(x) for x in segs], out=new_off[1:])
        new_cols = np.concatenate(segs).astype(np.uint16) if segs else np.zeros(0, dtype=np.uint16)
        self._off, self._cols, self._fit, self._seq = new_off, new_cols, new_fit, seq.copy()


# ---------------------------------------------------------------------------
# Synthetic scenarios (synthgen.hpp:18-223)
# ---------------------------------------------------------------------------
class Pattern(enum.IntEnum):  # synthgen.hpp:18-25
    kTrendPreserving = 0
    kColumnConstant = 1
    kRowConstant = 2
    kShift = 3
    kScale = 4
    kShiftScale = 5


@dataclass
class ScenarioSpec:  # synthgen.hpp:51-61
    n_rows: int = 0
    n_cols: int = 0
    blocks: List[tuple] = field(default_factory=list)  # [(rows, cols), ...]
    pattern: Pattern = Pattern.kTrendPreserving
    overlap_rows: int = 0
    overlap_cols: int = 0
    noise_sd: float = 0.0
    seed: int = 0


def synth_generate(spec: ScenarioSpec) -> ExpressionMatrix:
    """Matrix of ebic::generate(spec) (synthgen.hpp:114-223), bit-identical."""
    out = np.empty((spec.n_rows, spec.n_cols), dtype=np.float64)
    br = np.ascontiguousarray([b[0] for b in spec.blocks] or [0], dtype=np.uint64)
    bc = np.ascontiguousarray([b[1] for b in spec.blocks] or [0], dtype=np.uint64)
    rc = lib.ebic_synth_generate(spec.n_rows, spec.n_cols, len(spec.blocks),
                                 br.ctypes.data_as(szp), bc.ctypes.data_as(szp), int(spec.pattern),
                                 spec.overlap_rows, spec.overlap_cols, float(spec.noise_sd),
                                 int(spec.seed), out.ctypes.data_as(f64p))
    if rc == 1:
        raise ValueError("invalid scenario")
    if rc != 0:
        raise RuntimeError("scenario infeasible")
    return ExpressionMatrix(out)
