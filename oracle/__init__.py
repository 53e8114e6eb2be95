"""TEST INFRASTRUCTURE ONLY -- the parity checker for the B200 hot path.

Two CPU implementations of the reference algorithm:

* ``port``: oracle/ebic_oracle.c, a plain-C restatement of
  /root/reference/proj/include/ebic/fitness.hpp:48-143 and expansion.hpp:16-87
  (built into oracle/_build/liboracle.so; always available).
* ``ref``: the UNMODIFIED reference headers compiled here into
  oracle/_ref/libebic_ref.so by oracle/Makefile (needs /root/reference at build
  time; the built .so travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package -- never the product path.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "_build" / "liboracle.so"
REF_LIB = HERE / "_ref" / "libebic_ref.so"
REF_RUN = HERE / "_ref" / "ebic_ref_run"
DROPIN_RUN = HERE / "_ref" / "ebic_dropin_run"
REFERENCE_INCLUDE = Path("/root/reference/proj/include")

u8p = C.POINTER(C.c_uint8)
u16p = C.POINTER(C.c_uint16)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)
szp = C.POINTER(C.c_size_t)
i64p = C.POINTER(C.c_int64)


def build(ref: bool = True) -> None:
    """make -C oracle oracle [ref] (ref only when the reference is present)."""
    targets = ["oracle"] + (["ref"] if ref and REFERENCE_INCLUDE.exists() else [])
    subprocess.run(["make", "-s", "-C", str(HERE), *targets], check=True)


def _p(a, t):
    return a.ctypes.data_as(t)


class Port:
    """ctypes view of oracle/_build/liboracle.so (the C restatement)."""

    def __init__(self):
        if not PORT_LIB.exists():
            build(ref=False)
        L = C.CDLL(str(PORT_LIB))
        L.orc_default_sigma.restype = C.c_uint64
        L.orc_default_sigma.argtypes = [C.c_size_t]
        L.orc_count_matches.restype = C.c_int
        L.orc_count_matches.argtypes = [f64p, C.c_size_t, C.c_size_t, szp, u16p, C.c_size_t,
                                        C.c_double, C.c_uint, u64p]
        L.orc_fitness_score.restype = C.c_double
        L.orc_fitness_score.argtypes = [C.c_uint64, C.c_size_t, C.c_uint64]
        L.orc_evaluate_population.restype = C.c_int
        L.orc_evaluate_population.argtypes = [f64p, C.c_size_t, C.c_size_t, szp, u16p, C.c_size_t,
                                              C.c_double, C.c_uint64, C.c_uint, u64p, f64p]
        L.orc_row_matches.restype = C.c_int
        L.orc_row_matches.argtypes = [f64p, C.c_size_t, C.c_size_t, u16p, C.c_size_t, C.c_double]
        L.orc_trend_violations.restype = C.c_size_t
        L.orc_trend_violations.argtypes = [f64p, C.c_size_t, C.c_size_t, u16p, C.c_size_t, C.c_double]
        L.orc_assign_rows.restype = C.c_size_t
        L.orc_assign_rows.argtypes = [f64p, C.c_size_t, C.c_size_t, u16p, C.c_size_t, C.c_double, u64p]
        L.orc_membership_bits.restype = None
        L.orc_membership_bits.argtypes = [f64p, C.c_size_t, C.c_size_t, u16p, C.c_size_t, C.c_double,
                                          C.c_size_t, u64p, u64p, u64p]
        L.orc_expand_bicluster.restype = C.c_size_t
        L.orc_top_rank_update.restype = C.c_int
        L.orc_top_rank_update.argtypes = [C.c_size_t, C.c_size_t, szp, u16p, f64p, u64p, C.c_size_t,
                                          szp, u16p, f64p, C.c_double, C.c_size_t, u64p, i64p,
                                          u64p, szp]
        L.orc_expand_bicluster.argtypes = [f64p, C.c_size_t, C.c_size_t, u16p, C.c_size_t, u64p, u8p,
                                           C.c_size_t, C.c_int, C.c_size_t, C.c_double, u64p, u8p]
        self.lib = L

    def count_matches(self, values, offsets, cols, eps=0.0, workers=1):
        v = np.ascontiguousarray(values, dtype=np.float64)
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        c = np.ascontiguousarray(cols, dtype=np.uint16)
        if c.size == 0:
            c = np.zeros(1, dtype=np.uint16)
        n = len(off) - 1
        out = np.zeros(max(n, 1), dtype=np.uint64)
        rc = self.lib.orc_count_matches(_p(v, f64p), v.shape[0], v.shape[1], _p(off, szp),
                                        _p(c, u16p), n, float(eps), workers, _p(out, u64p))
        if rc == -1:
            raise ValueError("matrix has no rows")
        return out[:n]

    def evaluate_population(self, values, offsets, cols, sigma, eps=0.0, workers=1):
        v = np.ascontiguousarray(values, dtype=np.float64)
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        c = np.ascontiguousarray(cols, dtype=np.uint16)
        if c.size == 0:
            c = np.zeros(1, dtype=np.uint16)
        n = len(off) - 1
        counts = np.zeros(max(n, 1), dtype=np.uint64)
        fit = np.zeros(max(n, 1), dtype=np.float64)
        rc = self.lib.orc_evaluate_population(_p(v, f64p), v.shape[0], v.shape[1], _p(off, szp),
                                              _p(c, u16p), n, float(eps), int(sigma), workers,
                                              _p(counts, u64p), _p(fit, f64p))
        if rc == -1:
            raise ValueError("matrix has no rows")
        return counts[:n], fit[:n]

    def fitness_score(self, count, length, sigma):
        return self.lib.orc_fitness_score(int(count), int(length), int(sigma))

    def default_sigma(self, n_rows):
        return int(self.lib.orc_default_sigma(n_rows))

    def row_matches(self, values, row, series, eps=0.0):
        v = np.ascontiguousarray(values, dtype=np.float64)
        s = np.ascontiguousarray(series, dtype=np.uint16)
        return bool(self.lib.orc_row_matches(_p(v, f64p), v.shape[1], row, _p(s, u16p), s.size, float(eps)))

    def trend_violations(self, values, row, series, eps=0.0):
        v = np.ascontiguousarray(values, dtype=np.float64)
        s = np.ascontiguousarray(series, dtype=np.uint16)
        return int(self.lib.orc_trend_violations(_p(v, f64p), v.shape[1], row, _p(s, u16p), s.size, float(eps)))

    def assign_rows(self, values, series, eps=0.0):
        v = np.ascontiguousarray(values, dtype=np.float64)
        s = np.ascontiguousarray(series, dtype=np.uint16)
        out = np.zeros(v.shape[0], dtype=np.uint64)
        n = self.lib.orc_assign_rows(_p(v, f64p), v.shape[0], v.shape[1], _p(s, u16p), s.size,
                                     float(eps), _p(out, u64p))
        return [int(r) for r in out[:n]]

    def membership_bits(self, values, series, eps=0.0, approx_k=1):
        v = np.ascontiguousarray(values, dtype=np.float64)
        s = np.ascontiguousarray(series, dtype=np.uint16)
        words = (v.shape[0] + 63) // 64
        ex = np.zeros(words, dtype=np.uint64)
        ng = np.zeros(words, dtype=np.uint64)
        ap = np.zeros(words, dtype=np.uint64)
        self.lib.orc_membership_bits(_p(v, f64p), v.shape[0], v.shape[1], _p(s, u16p), s.size,
                                     float(eps), int(approx_k), _p(ex, u64p), _p(ng, u64p), _p(ap, u64p))
        return ex, ng, ap

    def expand_bicluster(self, values, series, core_rows, core_flags, allow_negative=True,
                         approx_k=1, eps=0.0):
        v = np.ascontiguousarray(values, dtype=np.float64)
        s = np.ascontiguousarray(series, dtype=np.uint16)
        cr = np.ascontiguousarray(core_rows if len(core_rows) else [0], dtype=np.uint64)
        cf = np.ascontiguousarray(core_flags if len(core_flags) else [0], dtype=np.uint8)
        cap = v.shape[0] + len(core_rows)
        ro = np.zeros(cap, dtype=np.uint64)
        fo = np.zeros(cap, dtype=np.uint8)
        n = self.lib.orc_expand_bicluster(_p(v, f64p), v.shape[0], v.shape[1], _p(s, u16p), s.size,
                                          _p(cr, u64p), _p(cf, u8p), len(core_rows),
                                          int(bool(allow_negative)), int(approx_k), float(eps),
                                          _p(ro, u64p), _p(fo, u8p))
        return [int(r) for r in ro[:n]], [int(f) for f in fo[:n]]


    def top_rank_update(self, n_cols, entries, cand_off, cand_cols, cand_fit, threshold, capacity,
                        next_seq):
        """evolution.hpp:168-206 in the stateless ebic_top_rank_update form.
        entries = (offsets, cols, fitness, seq) arrays.  Returns (ref, seq, next_seq)."""
        e_off, e_cols, e_fit, e_seq = (np.ascontiguousarray(entries[0], dtype=np.uint64),
                                       np.ascontiguousarray(entries[1], dtype=np.uint16),
                                       np.ascontiguousarray(entries[2], dtype=np.float64),
                                       np.ascontiguousarray(entries[3], dtype=np.uint64))
        k_off = np.ascontiguousarray(cand_off, dtype=np.uint64)
        k_cols = np.ascontiguousarray(cand_cols, dtype=np.uint16)
        k_fit = np.ascontiguousarray(cand_fit, dtype=np.float64)
        pad = lambda a: a if a.size else np.zeros(1, dtype=a.dtype)  # noqa: E731
        n_e, n_c = len(e_fit), len(k_fit)
        cap = max(1, min(capacity, n_e + n_c))
        ref = np.zeros(cap, dtype=np.int64)
        seq = np.zeros(cap, dtype=np.uint64)
        nxt = C.c_uint64(next_seq)
        n = C.c_size_t(0)
        self.lib.orc_top_rank_update(n_cols, n_e, _p(e_off, szp), _p(pad(e_cols), u16p),
                                     _p(pad(e_fit), f64p), _p(pad(e_seq), u64p), n_c, _p(k_off, szp),
                                     _p(pad(k_cols), u16p), _p(pad(k_fit), f64p), float(threshold),
                                     capacity, C.byref(nxt), _p(ref, i64p), _p(seq, u64p), C.byref(n))
        return ref[:n.value], seq[:n.value], nxt.value


class Ref:
    """ctypes view of oracle/_ref/libebic_ref.so (reference headers, compiled here)."""

    def __init__(self):
        if not REF_LIB.exists():
            raise FileNotFoundError(f"{REF_LIB} not built (needs /root/reference at build time)")
        L = C.CDLL(str(REF_LIB))
        L.ref_matrix_create.restype = C.c_void_p
        L.ref_matrix_create.argtypes = [f64p, C.c_size_t, C.c_size_t]
        L.ref_matrix_destroy.restype = None
        L.ref_matrix_destroy.argtypes = [C.c_void_p]
        L.ref_count_matches.restype = C.c_int
        L.ref_count_matches.argtypes = [C.c_void_p, szp, u16p, C.c_size_t, C.c_double, C.c_uint, u64p]
        L.ref_evaluate_population.restype = C.c_int
        L.ref_evaluate_population.argtypes = [C.c_void_p, szp, u16p, C.c_size_t, C.c_uint64,
                                              C.c_double, C.c_uint, f64p]
        L.ref_fitness_score.restype = C.c_double
        L.ref_fitness_score.argtypes = [C.c_uint64, C.c_size_t, C.c_uint64]
        L.ref_default_sigma.restype = C.c_uint64
        L.ref_default_sigma.argtypes = [C.c_size_t]
        L.ref_assign_rows.restype = C.c_size_t
        L.ref_assign_rows.argtypes = [C.c_void_p, u16p, C.c_size_t, C.c_double, u64p]
        L.ref_expand_bicluster.restype = C.c_size_t
        L.ref_expand_bicluster.argtypes = [C.c_void_p, u16p, C.c_size_t, u64p, u8p, C.c_size_t,
                                           C.c_int, C.c_size_t, C.c_double, u64p, u8p]
        L.ref_generate.restype = C.c_int
        L.ref_generate.argtypes = [C.c_size_t, C.c_size_t, C.c_size_t, szp, szp, C.c_int,
                                   C.c_size_t, C.c_size_t, C.c_double, C.c_uint64, f64p]
        L.ref_derive_seed.restype = C.c_uint64
        L.ref_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_toprank_create.restype = C.c_void_p
        L.ref_toprank_create.argtypes = [C.c_size_t]
        L.ref_toprank_destroy.argtypes = [C.c_void_p]
        L.ref_toprank_update.argtypes = [C.c_void_p, szp, u16p, C.c_size_t, f64p, C.c_double,
                                         C.c_size_t]
        L.ref_toprank_size.restype = C.c_size_t
        L.ref_toprank_size.argtypes = [C.c_void_p]
        L.ref_toprank_entries.restype = C.c_size_t
        L.ref_toprank_entries.argtypes = [C.c_void_p, szp, u16p, f64p, u64p]
        L.ref_toprank_time.restype = C.c_double
        L.ref_toprank_time.argtypes = [C.c_size_t, C.c_size_t, szp, szp, u16p, f64p, C.c_double,
                                       C.c_size_t, C.c_int]
        L.ref_run_population_trace.restype = C.c_long
        L.ref_run_population_trace.argtypes = [C.c_void_p, C.c_size_t, C.c_size_t, C.c_uint64,
                                               C.c_double, C.c_uint64, C.c_uint, C.c_char_p]
        L.ref_run_trace.restype = C.c_long
        L.ref_run_trace.argtypes = [C.c_void_p, C.c_size_t, C.c_size_t, C.c_uint64, C.c_double,
                                    C.c_uint64, C.c_uint, C.c_size_t, C.c_char_p]
        L.ref_run_trace_sel.restype = C.c_long
        L.ref_run_trace_sel.argtypes = [C.c_void_p, C.c_size_t, C.c_size_t, C.c_uint64, C.c_double,
                                        C.c_uint64, C.c_uint, C.c_size_t, C.c_size_t, C.c_char_p]
        self.lib = L

    class Matrix:
        def __init__(self, ref, values):
            v = np.ascontiguousarray(values, dtype=np.float64)
            self.ref, self.shape = ref, v.shape
            self.h = ref.lib.ref_matrix_create(_p(v, f64p), v.shape[0], v.shape[1])

        def __del__(self):
            try:
                self.ref.lib.ref_matrix_destroy(self.h)
            except Exception:
                pass

    def matrix(self, values):
        return Ref.Matrix(self, values)

    def count_matches(self, m, offsets, cols, eps=0.0, workers=1):
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        c = np.ascontiguousarray(cols, dtype=np.uint16)
        if c.size == 0:
            c = np.zeros(1, dtype=np.uint16)
        n = len(off) - 1
        out = np.zeros(max(n, 1), dtype=np.uint64)
        rc = self.lib.ref_count_matches(m.h, _p(off, szp), _p(c, u16p), n, float(eps), workers,
                                        _p(out, u64p))
        if rc != 0:
            raise ValueError("reference count_matches failed")
        return out[:n]

    def evaluate_population(self, m, offsets, cols, sigma, eps=0.0, workers=1):
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        c = np.ascontiguousarray(cols, dtype=np.uint16)
        n = len(off) - 1
        out = np.zeros(max(n, 1), dtype=np.float64)
        rc = self.lib.ref_evaluate_population(m.h, _p(off, szp), _p(c, u16p), n, int(sigma),
                                              float(eps), workers, _p(out, f64p))
        if rc != 0:
            raise ValueError("reference evaluate_population failed")
        return out[:n]

    def assign_rows(self, m, series, eps=0.0):
        s = np.ascontiguousarray(series, dtype=np.uint16)
        out = np.zeros(m.shape[0], dtype=np.uint64)
        n = self.lib.ref_assign_rows(m.h, _p(s, u16p), s.size, float(eps), _p(out, u64p))
        return [int(r) for r in out[:n]]

    def expand_bicluster(self, m, series, core_rows, core_flags, allow_negative=True, approx_k=1,
                         eps=0.0):
        s = np.ascontiguousarray(series, dtype=np.uint16)
        cr = np.ascontiguousarray(core_rows if len(core_rows) else [0], dtype=np.uint64)
        cf = np.ascontiguousarray(core_flags if len(core_flags) else [0], dtype=np.uint8)
        cap = m.shape[0] + len(core_rows)
        ro = np.zeros(cap, dtype=np.uint64)
        fo = np.zeros(cap, dtype=np.uint8)
        n = self.lib.ref_expand_bicluster(m.h, _p(s, u16p), s.size, _p(cr, u64p), _p(cf, u8p),
                                          len(core_rows), int(bool(allow_negative)), int(approx_k),
                                          float(eps), _p(ro, u64p), _p(fo, u8p))
        return [int(r) for r in ro[:n]], [int(f) for f in fo[:n]]

    def generate(self, n_rows, n_cols, blocks, pattern=0, overlap_rows=0, overlap_cols=0,
                 noise_sd=0.0, seed=0):
        out = np.empty((n_rows, n_cols), dtype=np.float64)
        br = np.ascontiguousarray([b[0] for b in blocks] or [0], dtype=np.uint64)
        bc = np.ascontiguousarray([b[1] for b in blocks] or [0], dtype=np.uint64)
        rc = self.lib.ref_generate(n_rows, n_cols, len(blocks), _p(br, szp), _p(bc, szp), pattern,
                                   overlap_rows, overlap_cols, float(noise_sd), seed, _p(out, f64p))
        if rc != 0:
            raise RuntimeError("scenario infeasible")
        return out

    def run_trace(self, m, path, population=600, iterations=10, rng_seed=1, eps=0.0, sigma=0,
                  threads=1, max_batches=0):
        n = self.lib.ref_run_trace(m.h, population, iterations, rng_seed, float(eps), sigma,
                                   threads, max_batches, str(path).encode())
        if n < 0:
            raise RuntimeError("reference run failed")
        return n


    def run_trace_sel(self, m, path, population=600, iterations=10, rng_seed=1, eps=0.0, sigma=0,
                      threads=1, record_first=0, record_every=0):
        n = self.lib.ref_run_trace_sel(m.h, population, iterations, rng_seed, float(eps), sigma,
                                       threads, record_first, record_every, str(path).encode())
        if n < 0:
            raise RuntimeError("reference run failed")
        return n

    class TopRank:
        """The reference's own TopRankList (evolution.hpp:142-218)."""

        def __init__(self, ref, n_cols):
            self.ref = ref
            self.h = ref.lib.ref_toprank_create(n_cols)

        def __del__(self):
            try:
                self.ref.lib.ref_toprank_destroy(self.h)
            except Exception:
                pass

        def update(self, off, cols, fit, threshold=0.75, capacity=100):
            off = np.ascontiguousarray(off, dtype=np.uint64)
            cols = np.ascontiguousarray(cols, dtype=np.uint16)
            fit = np.ascontiguousarray(fit, dtype=np.float64)
            pad = lambda a: a if a.size else np.zeros(1, dtype=a.dtype)  # noqa: E731
            self.ref.lib.ref_toprank_update(self.h, _p(off, szp), _p(pad(cols), u16p), len(fit),
                                            _p(pad(fit), f64p), float(threshold), capacity)

        def entries(self):
            """-> (offsets u64, cols u16, fitness f64, seq u64)."""
            L = self.ref.lib
            n = L.ref_toprank_size(self.h)
            total = L.ref_toprank_entries(self.h, None, None, None, None)
            off = np.zeros(n + 1, dtype=np.uint64)
            cols = np.zeros(max(total, 1), dtype=np.uint16)
            fit = np.zeros(max(n, 1), dtype=np.float64)
            seq = np.zeros(max(n, 1), dtype=np.uint64)
            L.ref_toprank_entries(self.h, _p(off, szp), _p(cols, u16p), _p(fit, f64p), _p(seq, u64p))
            return off, cols[:total], fit[:n], seq[:n]

    def run_population_trace(self, m, path, population=600, iterations=10, rng_seed=1, eps=0.0,
                             sigma=0, threads=1):
        n = self.lib.ref_run_population_trace(m.h, population, iterations, rng_seed, float(eps),
                                              sigma, threads, str(path).encode())
        if n < 0:
            raise RuntimeError("reference run failed")
        return n

    def top_rank(self, n_cols):
        return Ref.TopRank(self, n_cols)

    def top_rank_time(self, n_cols, updates, threshold=0.75, capacity=100, reps=3):
        """Mean us per TopRankList::update replaying [(off, cols, fit), ...]."""
        sizes = np.array([len(f) for _, _, f in updates], dtype=np.uint64)
        offs, colss, fits, base = [np.zeros(1, dtype=np.uint64)], [], [], 0
        for off, cols, fit in updates:
            offs.append(np.asarray(off[1:], dtype=np.uint64) + base)
            base += int(off[-1])
            colss.append(np.asarray(cols, dtype=np.uint16))
            fits.append(np.asarray(fit, dtype=np.float64))
        off = np.concatenate(offs)
        cols = np.concatenate(colss)
        fit = np.concatenate(fits)
        return self.lib.ref_toprank_time(n_cols, len(updates), _p(sizes, szp), _p(off, szp),
                                         _p(cols, u16p), _p(fit, f64p), float(threshold), capacity,
                                         reps)


def read_population_trace(path):
    """Parse a ref_run_population_trace file -> list of (offsets u64, cols u16, fitness f64)."""
    data = Path(path).read_bytes()
    at, out = 0, []
    while at < len(data):
        P = int(np.frombuffer(data, np.uint64, 1, at)[0]); at += 8
        off = np.frombuffer(data, np.uint64, P + 1, at).copy(); at += 8 * (P + 1)
        L = int(off[-1])
        cols = np.frombuffer(data, np.uint16, L, at).copy(); at += 2 * L
        fit = np.frombuffer(data, np.float64, P, at).copy(); at += 8 * P
        out.append((off, cols, fit))
    return out


def read_trace(path):
    """Parse a ref_run_trace file -> list of (offsets u64, cols u16, counts u64)."""
    data = Path(path).read_bytes()
    at, out = 0, []
    while at < len(data):
        P = int(np.frombuffer(data, np.uint64, 1, at)[0]); at += 8
        off = np.frombuffer(data, np.uint64, P + 1, at).copy(); at += 8 * (P + 1)
        L = int(off[-1])
        cols = np.frombuffer(data, np.uint16, L, at).copy(); at += 2 * L
        counts = np.frombuffer(data, np.uint64, P, at).copy(); at += 8 * P
        out.append((off, cols, counts))
    return out


def read_trace_sel(path):
    """Parse a ref_run_trace_sel file -> list of (batch index, offsets, cols, counts)."""
    data = Path(path).read_bytes()
    at, out = 0, []
    while at < len(data):
        k = int(np.frombuffer(data, np.uint64, 1, at)[0]); at += 8
        P = int(np.frombuffer(data, np.uint64, 1, at)[0]); at += 8
        off = np.frombuffer(data, np.uint64, P + 1, at).copy(); at += 8 * (P + 1)
        L = int(off[-1])
        cols = np.frombuffer(data, np.uint16, L, at).copy(); at += 2 * L
        counts = np.frombuffer(data, np.uint64, P, at).copy(); at += 8 * P
        out.append((k, off, cols, counts))
    return out
