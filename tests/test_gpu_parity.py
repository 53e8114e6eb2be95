"""GPU parity: the sm_100a path through the C ABI against the reference.

Every comparison is exact: counts ==, fitness bitwise == (fp64 bit patterns),
membership rows/flags ==.  Expected values come from the reference itself
(golden fixtures generated from the unmodified reference headers) or from the
CPU oracle (oracle/ebic_oracle.c, pinned to the reference by
tests/test_oracle_golden.py) on the same seeded inputs.
"""
import os
from contextlib import contextmanager

import numpy as np
import pytest

import oracle
import paper_1801_03039_b200 as eb
from golden_io import STEADY_NAMES, TRACE_NAMES, acceptance, expansion_cases, fitness_trials, trace

pytestmark = pytest.mark.gpu
port = oracle.Port()

# Every count-kernel configuration the library can select: the exact rank
# tile (default; 1 or 2 planes by eps / NaN presence, 16, 24 or 31 consumer warps),
# the fp64 tile (rows-per-tile x rows-per-lane), and the unstaged direct kernel.
KERNEL_CONFIGS = ([dict(), dict(EBIC_NCW="16"), dict(EBIC_NCW="24"), dict(EBIC_NCW="32"), dict(EBIC_NO_COLLAPSE="1"),
                   dict(EBIC_NO_COLLAPSE="1", EBIC_NCW="16"), dict(EBIC_NO_COLLAPSE="1", EBIC_NCW="32"), dict(EBIC_SPG="4"),
                   dict(EBIC_SPG="4", EBIC_NO_COLLAPSE="1")] +
                  [dict(EBIC_LAYOUT_F64="1", EBIC_RPG=str(g), EBIC_RPL=str(l))
                   for g in (32, 16, 8, 4) for l in (1, 2)] +
                  [dict(EBIC_LAYOUT_F64="1", EBIC_NCW="16"), dict(EBIC_LAYOUT_F64="1", EBIC_NCW="32"), dict(EBIC_FORCE_DIRECT="1")] +
                  # K1v2 (default for rank layouts) vs the v1 tile kernel, and K1v2's own knobs
                  [dict(EBIC_KERNEL="1"), dict(EBIC_KERNEL="1", EBIC_NO_COLLAPSE="1"), dict(EBIC_COMPACT="1"), dict(EBIC_COMPACT="0"),
                   dict(EBIC_COMPACT="1", EBIC_GAP="2"), dict(EBIC_STAGES="1"), dict(EBIC_COMPACT="1", EBIC_NO_COLLAPSE="1"),
                   dict(EBIC_PACK="0"), dict(EBIC_PACK="0", EBIC_COMPACT="1"),
                   # K1s (series per CTA; default for short launches) against K1v2, and its shapes
                   dict(EBIC_SPLIT="0"), dict(EBIC_SPLIT="1"), dict(EBIC_SPLIT="1", EBIC_NO_COLLAPSE="1"),
                   dict(EBIC_SPLIT="1", EBIC_PACK="0"), dict(EBIC_SPLIT="1", EBIC_GRID="1000"),
                   dict(EBIC_SPLIT="1", EBIC_GRID="3"),
                   # five rows per 64-bit word (default above 510 columns) also on narrow matrices
                   dict(EBIC_PACK="12"), dict(EBIC_PACK="12", EBIC_SPLIT="0", EBIC_COMPACT="1"),
                   dict(EBIC_PACK="12", EBIC_SPLIT="1")])


@contextmanager
def env(**kw):
    old = {k: os.environ.get(k) for k in kw}
    os.environ.update(kw)
    try:
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def cbf(series):
    off = np.zeros(len(series) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(s) for s in series])
    return eb.CbfPopulation(off, np.array([c for s in series for c in s], dtype=np.uint16))


def bits_equal(a, b):
    return (np.asarray(a, np.float64).view(np.uint64) == np.asarray(b, np.float64).view(np.uint64)).all()


def random_population(rng, n_cols, P, max_len=9):
    return [list(map(int, rng.choice(n_cols, size=int(rng.integers(2, min(n_cols, max_len) + 1)),
                                     replace=False))) for _ in range(P)]


# ---------------------------------------------------------------------------
def test_smoke_small():
    rng = np.random.default_rng(0)
    v = rng.standard_normal((300, 30))
    pop = cbf(random_population(rng, 30, 200))
    with eb.Evaluator(v) as ev:
        fit, counts = ev.evaluate_population(pop, eb.FitnessParams(6), 0.0, return_counts=True)
        info = ev.info()
    c, f = port.evaluate_population(v, pop.offsets, pop.col_indices, 6, 0.0)
    assert (counts == c).all() and bits_equal(fit, f)
    assert info.rows_per_tile > 0 and info.grid > 0


def test_acceptance_golden_all_eps():  # acceptance_main.cpp:233-292
    z = acceptance()
    pop = eb.CbfPopulation(z["offsets"], z["cols"])
    with eb.Evaluator(z["values"]) as ev:
        for i, eps in enumerate(z["eps"]):
            assert (ev.count_matches(pop, eps) == z[f"counts_{i}"]).all()
            fit = ev.evaluate_population(pop, eb.FitnessParams(int(z["sigma"])), eps)
            assert bits_equal(fit, z[f"fitness_{i}"])


def test_fitness_trials_golden():  # test_fitness.cpp:111-137
    for v, off, cols, eps, counts in fitness_trials():
        with eb.Evaluator(v) as ev:
            assert (ev.count_matches(eb.CbfPopulation(off, cols), eps) == counts).all()


@pytest.mark.parametrize("name", TRACE_NAMES + STEADY_NAMES)
def test_trace_golden(name):
    """Every batch of a recorded reference GA run: counts and fitness bit-exact."""
    t = trace(name)
    with eb.Evaluator(t.matrix()) as ev:
        for off, cols, counts, fit in t.batches:
            f, c = ev.evaluate_population(eb.CbfPopulation(off, cols), eb.FitnessParams(t.sigma),
                                          t.eps, return_counts=True)
            assert (c == counts).all()
            assert bits_equal(f, fit)


@pytest.mark.parametrize("cfg", KERNEL_CONFIGS, ids=lambda d: "-".join(f"{k}={v}" for k, v in d.items()) or "default")
@pytest.mark.parametrize("name", ["c1", "c1e", "c3", "c4"])
def test_every_kernel_config_on_traces(cfg, name):
    t = trace(name)
    v = t.matrix()
    with env(**cfg):
        with eb.Evaluator(v) as ev:
            for off, cols, counts, fit in t.batches[:3]:
                f, c = ev.evaluate_population(eb.CbfPopulation(off, cols), eb.FitnessParams(t.sigma),
                                              t.eps, return_counts=True)
                assert (c == counts).all()
                assert bits_equal(f, fit)


# Scheduling, reduction and staging knobs (results must not depend on them).
SCHEDULE_CONFIGS = [dict(EBIC_GRID="37"), dict(EBIC_GRID="300"), dict(EBIC_SCHED_STATIC="1"),
                    dict(EBIC_MAX_PARTS="1"), dict(EBIC_REDUCE_TREE="1"), dict(EBIC_SLICE="64"),
                    dict(EBIC_STAGES="2"), dict(EBIC_HOST_COPY="1"), dict(EBIC_GRAPH="0"),
                    dict(EBIC_REDUCE_TREE="1", EBIC_GRID="37", EBIC_HOST_COPY="1")]


@pytest.mark.parametrize("name", ["c4", "c3", "c1e"])
@pytest.mark.parametrize("cfg", SCHEDULE_CONFIGS, ids=lambda d: "-".join(f"{k}={v}" for k, v in d.items()))
def test_schedule_knobs_on_traces(cfg, name):
    t = trace(name)
    v = t.matrix()
    with env(**cfg):
        with eb.Evaluator(v) as ev:
            for rep in range(2):  # the second pass reuses the graph / ring / tables
                for off, cols, counts, fit in t.batches[:3]:
                    f, c = ev.evaluate_population(eb.CbfPopulation(off, cols), eb.FitnessParams(t.sigma),
                                                  t.eps, return_counts=True)
                    assert (c == counts).all()
                    assert bits_equal(f, fit)


@pytest.mark.parametrize("cfg", KERNEL_CONFIGS[:8] + KERNEL_CONFIGS[10:11] + KERNEL_CONFIGS[-1:], ids=str)
def test_edge_cases_vs_oracle(cfg):
    """Ragged row counts, ties, +-0, NaN/inf cells, odd eps values, len-1 series."""
    rng = np.random.default_rng(7)
    with env(**cfg):
        for rows in (1, 2, 15, 16, 17, 31, 33, 63, 64, 65, 127, 129, 1000, 4097):
            n_cols = int(rng.integers(3, 90))
            v = np.round(rng.standard_normal((rows, n_cols)), 1)
            flat = v.ravel()
            k = max(1, flat.size // 50)
            flat[rng.choice(flat.size, k, replace=False)] = rng.choice(
                [np.nan, np.inf, -np.inf, 0.0, -0.0], k)
            series = random_population(rng, n_cols, int(rng.integers(1, 300)))
            series[0] = [series[0][0]]  # length-1 series: no adjacent pair -> every row matches
            pop = cbf(series)
            with eb.Evaluator(v) as ev:
                for eps in (0.0, -0.0, 1e-9, 0.1, -0.05, np.inf, np.nan, 1e300):
                    got = ev.count_matches(pop, eps)
                    want = port.count_matches(v, pop.offsets, pop.col_indices, eps)
                    assert (got == want).all(), (rows, n_cols, eps)


V2_CONFIGS = [dict(), dict(EBIC_NO_COLLAPSE="1"), dict(EBIC_COMPACT="1"), dict(EBIC_COMPACT="0"),
              dict(EBIC_COMPACT="1", EBIC_GAP="1"), dict(EBIC_COMPACT="1", EBIC_GAP="2"),
              dict(EBIC_COMPACT="1", EBIC_NO_COLLAPSE="1"), dict(EBIC_STAGES="1"), dict(EBIC_COMPACT="1", EBIC_STAGES="1"),
              dict(EBIC_GRID="7"), dict(EBIC_COMPACT="1", EBIC_GRID="7")]


@pytest.mark.parametrize("cfg", V2_CONFIGS, ids=lambda d: "-".join(f"{k}={v}" for k, v in d.items()) or "default")
def test_v2_column_runs_vs_oracle(cfg):
    """K1v2 stages only the launch's referenced columns, as runs of consecutive
    columns: every column (one run, a 1000-column stage that fits only once),
    every other column (the most runs), the two edge columns, one tail block,
    a single repeated column, and random sets -- over 1 tile and many."""
    rng = np.random.default_rng(21)
    n_cols = 1000
    pops = {
        "all": [list(map(int, rng.permutation(n_cols)[:8])) for _ in range(40)] +
               [list(range(k, n_cols, 125)) for k in range(125)],
        "every_other": [list(map(int, rng.choice(np.arange(0, n_cols, 2), size=int(rng.integers(2, 9)),
                                                 replace=False))) for _ in range(300)] +
                       [list(range(k, n_cols, 250)) for k in range(0, 250, 2)],
        "edges": [[0, n_cols - 1], [n_cols - 1, 0]] * 20,
        "tail": [list(map(int, rng.choice(np.arange(n_cols - 64, n_cols), size=int(rng.integers(2, 12)),
                                          replace=False))) for _ in range(200)],
        "one_col": [[5, 5, 5], [5, 5]] * 9,
        "random": random_population(rng, n_cols, 700, max_len=14),
    }
    with env(**cfg):
        for rows in (700, 13000):
            v = np.round(rng.standard_normal((rows, n_cols)), 2)
            with eb.Evaluator(v) as ev:
                for name, series in pops.items():
                    pop = cbf(series)
                    for eps in (0.0, 1e-9, 0.05):
                        got = ev.count_matches(pop, eps)
                        want = port.count_matches(v, pop.offsets, pop.col_indices, eps)
                        assert (got == want).all(), (rows, name, eps)


@pytest.mark.parametrize("grid", ["", "40", "148", "4000"])
def test_split_kernel_partition_vs_oracle(grid):
    """K1s splits series x row tiles by length-weighted units: series split
    over 2+ CTAs (partial sums, arrival counters), CTA ranges shorter than one
    series (some CTAs in a series' span hold none of its tiles), few CTAs with
    many series per CTA, length-0/1 series, many more CTAs than work."""
    rng = np.random.default_rng(44)
    cfg = dict(EBIC_SPLIT="1", **({"EBIC_GRID": grid} if grid else {}))
    with env(**cfg):
        for rows, n_cols in ((40, 30), (960, 100), (5000, 400)):
            v = np.round(rng.standard_normal((rows, n_cols)), 1)
            series = random_population(rng, n_cols, 300, max_len=20) + [[], [3], [7, 7], list(range(n_cols))[:25]]
            rng.shuffle(series)
            pop = cbf(series)
            with eb.Evaluator(v) as ev:
                for eps in (0.0, 1e-9, 0.05):
                    for rep in range(2):  # the accumulators must come back zeroed
                        got = ev.count_matches(pop, eps)
                        want = port.count_matches(v, pop.offsets, pop.col_indices, eps)
                        assert (got == want).all(), (grid, rows, eps, rep)
                    f, c = ev.evaluate_population(pop, eb.FitnessParams(max(4, rows // 50)), eps, return_counts=True)
                    _, wf = port.evaluate_population(v, pop.offsets, pop.col_indices, max(4, rows // 50), eps)
                    assert bits_equal(f, wf)
                    assert ev.info().kernel == 3


PACK_CONFIGS = [dict(), dict(EBIC_SPLIT="0"), dict(EBIC_COMPACT="1"), dict(EBIC_COMPACT="0", EBIC_SPLIT="0"),
                dict(EBIC_GRID="7", EBIC_SPLIT="0"), dict(EBIC_COMPACT="1", EBIC_GRID="7"), dict(EBIC_STAGES="1"),
                dict(EBIC_V2_NP="4", EBIC_SPLIT="0"), dict(EBIC_SPLIT="1", EBIC_GRID="1000"),
                dict(EBIC_SPLIT="1", EBIC_GRID="5"), dict(EBIC_PACK="12", EBIC_SPLIT="0"),
                dict(EBIC_PACK="12", EBIC_SPLIT="1"), dict(EBIC_PACK="12", EBIC_COMPACT="1", EBIC_SPLIT="0")]


@pytest.mark.parametrize("cfg", PACK_CONFIGS, ids=lambda d: "-".join(f"{k}={v}" for k, v in d.items()) or "default")
def test_v2_packed_ranks_vs_oracle(cfg):
    """Matrices of <= 510 columns stream one rank plane packed three rows per
    word (96-row tiles, 10-bit fields): ragged row counts around the 96-row
    tile and 64-row mask-word boundaries, the widest packable matrix, ties,
    strict and collapsed tests, dirty rows straddling two mask words."""
    rng = np.random.default_rng(33)
    with env(**cfg):
        for rows, n_cols in ((1, 5), (95, 40), (96, 40), (97, 40), (191, 510), (1000, 510), (13000, 300),
                             (4097, 97)):
            v = np.round(rng.standard_normal((rows, n_cols)), 1)  # many ties
            for r in rng.choice(rows, size=min(rows, 9), replace=False):  # eps-close pairs: dirty rows
                a, b = rng.choice(n_cols, size=2, replace=False) if n_cols > 1 else (0, 0)
                v[r, b] = v[r, a] + 0.5e-6
            series = random_population(rng, n_cols, 600, max_len=12)
            pop = cbf(series)
            with eb.Evaluator(v) as ev:
                for eps in (0.0, 1e-6, 0.05):
                    got = ev.count_matches(pop, eps)
                    want = port.count_matches(v, pop.offsets, pop.col_indices, eps)
                    assert (got == want).all(), (rows, n_cols, eps)
                    if eps == 0.0:
                        assert ev.info().layout == (6 if os.environ.get("EBIC_PACK") == "12" else 4), ev.info().layout
                f = ev.evaluate_population(pop, eb.FitnessParams(max(4, rows // 50)), 1e-6)
                _, wf = port.evaluate_population(v, pop.offsets, pop.col_indices, max(4, rows // 50), 1e-6)
                assert bits_equal(f, wf)


@pytest.mark.parametrize("cfg", [dict(EBIC_SPLIT="0"), dict(EBIC_SPLIT="1"), dict(EBIC_COMPACT="1"),
                                 dict(EBIC_KERNEL="1")], ids=str)
def test_host_cbf_staging_without_cta0(cfg):
    """Host-buffer calls: the population is copied to the device by CTA 0 and
    published with a flag.  EBIC_DEBUG_MODE=4 suppresses the flag, so every
    other CTA must take its own copy after the 20 us wait -- the result may
    not depend on CTA 0 being scheduled first."""
    t = trace("c4")
    with env(EBIC_DEBUG_MODE="4", **cfg):
        with eb.Evaluator(t.matrix()) as ev:
            for off, cols, counts, fit in t.batches[:3]:
                f, c = ev.evaluate_population(eb.CbfPopulation(off, cols), eb.FitnessParams(t.sigma), t.eps,
                                              return_counts=True)
                assert (c == counts).all() and bits_equal(f, fit)


def test_empty_population_and_errors():
    v = np.random.default_rng(1).standard_normal((100, 10))
    with eb.Evaluator(v) as ev:
        assert ev.count_matches(eb.CbfPopulation()).size == 0
        with pytest.raises(ValueError, match="invalid series"):
            ev.count_matches(cbf([[0, 10]]))
        with pytest.raises(RuntimeError, match="corrupt CBF"):
            ev.count_matches(eb.CbfPopulation(np.array([0, 3, 2], np.uint64),
                                              np.array([0, 1, 2], np.uint16)))
    with pytest.raises(ValueError, match="matrix has no rows"):
        eb.Evaluator(np.zeros((0, 5)))


def test_large_population_is_split_exactly():
    """P above one launch's shared-memory work list (4096 series)."""
    rng = np.random.default_rng(3)
    v = rng.standard_normal((3000, 120))
    pop = cbf(random_population(rng, 120, 9000))
    with eb.Evaluator(v) as ev:
        f, c = ev.evaluate_population(pop, eb.FitnessParams(60), 1e-9, return_counts=True)
    wc, wf = port.evaluate_population(v, pop.offsets, pop.col_indices, 60, 1e-9)
    assert (c == wc).all() and bits_equal(f, wf)


def test_wide_matrix_direct_path():
    """Many columns: config selection falls back to the unstaged kernel."""
    rng = np.random.default_rng(4)
    v = rng.standard_normal((700, 9000))
    pop = cbf(random_population(rng, 9000, 400, max_len=12))
    with eb.Evaluator(v) as ev:
        got = ev.count_matches(pop, 0.05)
    assert (got == port.count_matches(v, pop.offsets, pop.col_indices, 0.05)).all()


@pytest.mark.parametrize("xshard", ["1", "0"])
@pytest.mark.parametrize("devices,name", [([0, 0, 0], "c3"), ([0, 0], "c4"), ([0] * 5, "c1e"), ([0, 0], "c5")])
def test_row_shards_on_one_device_are_partition_invariant(xshard, devices, name):
    """Several 64-row-aligned shards on one GPU.  EBIC_XSHARD=1: every shard's
    kernel adds its totals into one accumulator and the last to finish writes
    counts + fitness (no launch waits for another, so the shards may run in any
    order); EBIC_XSHARD=0: exact host reduction."""
    t = trace(name)
    v = t.matrix()
    with env(EBIC_XSHARD=xshard), eb.Evaluator(v, devices=devices) as ev:
        assert ev.info().n_shards >= 2  # 64-row aligned: fewer shards than devices on small matrices
        for rep in range(2):
            for off, cols, counts, fit in t.batches[:4]:
                f, c = ev.evaluate_population(eb.CbfPopulation(off, cols), eb.FitnessParams(t.sigma),
                                              t.eps, return_counts=True)
                assert (c == counts).all() and bits_equal(f, fit)
                c2 = ev.count_matches(eb.CbfPopulation(off, cols), t.eps)
                assert (c2 == counts).all()


def test_shard_contexts_sum_to_whole():
    """One-process-per-GPU layout: per-shard partial counts + reduction == reference."""
    t = trace("c2_scale")
    v = t.matrix()
    bounds = [0, 320, 640, 1000]
    off, cols, counts, fit = t.batches[2]
    pop = eb.CbfPopulation(off, cols)
    total = np.zeros_like(counts)
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        with eb.Evaluator(v[lo:hi], shard=(lo, v.shape[0])) as ev:
            total += ev.count_matches(pop, t.eps)
    assert (total == counts).all()


def test_device_pointer_api_with_fused_fitness():
    import torch
    from paper_1801_03039_b200 import _lib
    t = trace("c1e")
    v = t.matrix()
    with eb.Evaluator(v) as ev:
        for off, cols, counts, fit in t.batches[:3]:
            d_off = torch.from_numpy(off.astype(np.int64)).cuda()
            d_cols = torch.from_numpy(cols.astype(np.int16)).cuda()
            d_cnt = torch.zeros(len(counts), dtype=torch.int64, device="cuda")
            d_fit = torch.zeros(len(counts), dtype=torch.float64, device="cuda")
            st = torch.cuda.current_stream().cuda_stream
            _lib.check(_lib.lib.ebic_count_matches_device(
                ev.handle, d_off.data_ptr(), d_cols.data_ptr(), len(counts), int(off[-1]), t.eps,
                t.sigma, d_cnt.data_ptr(), d_fit.data_ptr(), st))
            torch.cuda.synchronize()
            assert (d_cnt.cpu().numpy().astype(np.uint64) == counts).all()
            assert bits_equal(d_fit.cpu().numpy(), fit)
            d_fit2 = torch.zeros_like(d_fit)
            _lib.check(_lib.lib.ebic_fitness_device(ev.handle, d_cnt.data_ptr(), d_off.data_ptr(),
                                                    len(counts), t.sigma, d_fit2.data_ptr(), st))
            torch.cuda.synchronize()
            assert bits_equal(d_fit2.cpu().numpy(), fit)


# ---- membership (Steps 6-7) ------------------------------------------------
def test_expansion_golden():
    for case in expansion_cases():
        with eb.Evaluator(case["matrix"]) as ev:
            core = ev.resolve_bicluster(case["series"], 1.0, case["eps"])
            assert core.rows == [int(r) for r in case["core"]]
            grown = ev.expand_bicluster(core, eb.ExpansionOptions(case["allow_negative"],
                                                                  case["approx_k"]), case["eps"])
            assert grown.rows == [int(r) for r in case["rows"]]
            assert [int(f) for f in grown.row_flags] == [int(f) for f in case["flags"]]
            (rows, flags), = ev.resolve_expand_batch(
                [list(map(int, case["series"]))],
                eb.ExpansionOptions(case["allow_negative"], case["approx_k"]), case["eps"])
            assert list(rows) == [int(r) for r in case["rows"]]
            assert list(flags) == [int(f) for f in case["flags"]]


@pytest.mark.parametrize("devices", [[0], [0, 0, 0]])
def test_membership_bits_vs_oracle(devices):
    rng = np.random.default_rng(8)
    for rows in (1, 63, 64, 65, 200, 1000, 5001):
        n_cols = int(rng.integers(3, 40))
        v = np.round(rng.standard_normal((rows, n_cols)), 1)
        series = random_population(rng, n_cols, 20)
        with eb.Evaluator(v, devices=devices) as ev:
            for eps, k in ((0.0, 1), (0.1, 2), (1e-9, 0)):
                ex, ng, ap = ev.membership_bits(cbf(series), eps, k)
                for i, s in enumerate(series):
                    e2, n2, a2 = port.membership_bits(v, s, eps, k)
                    assert (ex[i] == e2).all() and (ng[i] == n2).all() and (ap[i] == a2).all()


def test_expand_with_arbitrary_core_vs_oracle():
    rng = np.random.default_rng(9)
    v = np.round(rng.standard_normal((700, 12)), 1)
    with eb.Evaluator(v) as ev:
        for trial in range(30):
            s = random_population(rng, 12, 1)[0]
            core = sorted(map(int, rng.choice(700, size=int(rng.integers(0, 40)), replace=False)))
            flags = [int(x) for x in rng.integers(0, 3, size=len(core))]
            b = eb.Bicluster(core, s, 2.0, [eb.RowFlag(f) for f in flags])
            for opts in (eb.ExpansionOptions(), eb.ExpansionOptions(False, 2), eb.ExpansionOptions(True, 0)):
                g = ev.expand_bicluster(b, opts, 0.05)
                wr, wf = port.expand_bicluster(v, s, core, flags, opts.allow_negative,
                                               opts.approx_violations, 0.05)
                assert g.rows == wr and [int(f) for f in g.row_flags] == wf


def test_finalize_biclusters_c4_top_series():
    """io.hpp:164-178 over the C4 matrix: one batched launch for 100 series."""
    t = trace("c4")
    v = t.matrix()
    off, cols, counts, fit = t.batches[-1]
    order = np.argsort(-fit, kind="stable")[:100]
    series = [list(map(int, cols[int(off[i]):int(off[i + 1])])) for i in order]
    entries = [(s, float(fit[i])) for s, i in zip(series, order)]
    m = eb.ExpressionMatrix(v)
    out = eb.finalize_biclusters(entries, m, eb.ExpansionOptions(), t.eps, 0.0)
    assert len(out) == 100
    for b in out:  # every finalized bicluster
        core = port.assign_rows(v, b.series, t.eps)
        wr, wf = port.expand_bicluster(v, b.series, core, [0] * len(core), True, 1, t.eps)
        assert b.rows == wr and [int(f) for f in b.row_flags] == wf


@pytest.mark.parametrize("n_dirty", [0, 1, 7, 40, 3000])
def test_collapsed_rank_layout_with_dirty_rows(n_dirty):
    """eps > 0 with clean rows uses the one-plane collapsed layout (<= test);
    rows holding two values closer than eps (or NaN) cannot be represented and
    are evaluated exactly in fp64 by the kernel.  Too many of them: two planes."""
    rng = np.random.default_rng(100 + n_dirty)
    rows, n_cols, eps = 6000, 60, 1e-6
    v = rng.standard_normal((rows, n_cols))
    dirty = rng.choice(rows, size=n_dirty, replace=False)
    for k, r in enumerate(dirty):
        a, b = rng.choice(n_cols, size=2, replace=False)
        if k % 5 == 4:
            v[r, a] = np.nan
        else:
            v[r, b] = v[r, a] + eps * [0.5, 1.0, 0.999, 0.25][k % 4]  # inside (v_a, v_a + eps]
    series = random_population(rng, n_cols, 700)
    pop = cbf(series)
    with eb.Evaluator(v) as ev:
        for e in (eps, 2 * eps, 1e-9):
            got = ev.count_matches(pop, e)
            want = port.count_matches(v, pop.offsets, pop.col_indices, e)
            assert (got == want).all(), (n_dirty, e)
            f = ev.evaluate_population(pop, eb.FitnessParams(120), e)
            _, wf = port.evaluate_population(v, pop.offsets, pop.col_indices, 120, e)
            assert bits_equal(f, wf)
        info = ev.info()
    # 5: the collapsed plane packed three rows per word (n_cols <= 510)
    assert info.layout == (5 if n_dirty <= 64 else 2)


@pytest.mark.parametrize("cfg", [dict(), dict(EBIC_NO_COLLAPSE="1"), dict(EBIC_LAYOUT_F64="1"),
                                 dict(EBIC_FORCE_DIRECT="1")], ids=str)
def test_repeated_columns_inside_a_series(cfg):
    """count_chunk (fitness.hpp:71-93) takes any column list: a repeated column
    compares a value with itself (v < v + eps), exactly as the reference."""
    rng = np.random.default_rng(31)
    rows, n_cols = 2000, 40
    v = np.round(rng.standard_normal((rows, n_cols)), 2)
    series = [list(map(int, rng.choice(n_cols, size=int(rng.integers(2, 9)), replace=True)))
              for _ in range(800)]
    pop = cbf(series)
    with env(**cfg), eb.Evaluator(v) as ev:
        for e in (0.0, 1e-9, 0.01, -0.01):
            got = ev.count_matches(pop, e)
            want = port.count_matches(v, pop.offsets, pop.col_indices, e)
            assert (got == want).all(), e


@pytest.mark.parametrize("cfg", [dict(), dict(EBIC_NO_COLLAPSE="1"), dict(EBIC_LAYOUT_F64="1")], ids=str)
def test_long_series_and_overflow_length_bucket(cfg):
    """Lengths 13-62 (generic walk) and >= 63 (the work list's overflow bucket,
    listed in a separate pass) next to short ones, across several launches."""
    rng = np.random.default_rng(77)
    rows, n_cols = 3000, 300
    v = np.round(rng.standard_normal((rows, n_cols)), 1)
    # mostly increasing rows for some column orders so long series still match
    v[:500] = np.sort(v[:500], axis=1)
    lens = list(rng.integers(2, 12, size=300)) + list(rng.integers(13, 63, size=120)) + \
        list(rng.integers(63, 250, size=40)) + [63, 64, 127, 250]
    rng.shuffle(lens)
    series = []
    for L in lens:
        if rng.random() < 0.3:  # ascending columns: matches the sorted rows
            series.append(sorted(map(int, rng.choice(n_cols, size=int(L), replace=False))))
        else:
            series.append(list(map(int, rng.choice(n_cols, size=int(L), replace=False))))
    pop = cbf(series)
    with env(**cfg), eb.Evaluator(v) as ev:
        for e in (0.0, 1e-9, 0.05):
            got = ev.count_matches(pop, e)
            want = port.count_matches(v, pop.offsets, pop.col_indices, e)
            assert (got == want).all(), e
            assert got.max() > 0


def test_many_rows():
    """4.2M rows (65,600 row tiles): tile indexing, shard padding and counts
    far above one tile, against the oracle on a small population."""
    rng = np.random.default_rng(5)
    rows, n_cols = 4_200_007, 24
    v = rng.standard_normal((rows, n_cols)).astype(np.float64)
    series = random_population(rng, n_cols, 40, max_len=6)
    pop = cbf(series)
    with eb.Evaluator(v) as ev:
        for e in (0.0, 0.3):
            got = ev.count_matches(pop, e)
            want = port.count_matches(v, pop.offsets, pop.col_indices, e)
            assert (got == want).all(), e


@pytest.mark.parametrize("n_cols", [1400, 2047, 2048, 2049])
def test_wide_matrix_layout_boundaries(n_cols):
    """Around the widths where the staged tiles stop fitting shared memory
    (1-plane rank rows of 32: ~1700 columns for two stages) and where the rank
    layout is no longer built (2048 columns, 2C keys sorted per row): every
    fallback (fp64 tile, direct kernel) stays exact."""
    rng = np.random.default_rng(n_cols)
    v = rng.standard_normal((700, n_cols))
    v[:, 5] = v[:, 7]  # ties
    pop = cbf(random_population(rng, n_cols, 300, max_len=9))
    with eb.Evaluator(v) as ev:
        for e in (0.0, 1e-9, 0.3):
            got = ev.count_matches(pop, e)
            assert (got == port.count_matches(v, pop.offsets, pop.col_indices, e)).all(), e


def test_device_batch_limits():
    """The device-pointer API takes up to 2048 series / 8192 columns per call
    and rejects larger batches with the documented message."""
    import torch
    from paper_1801_03039_b200 import _lib
    rng = np.random.default_rng(11)
    v = rng.standard_normal((900, 64))
    with eb.Evaluator(v) as ev:
        for P in (2048, 2049):
            series = [rng.choice(64, size=4, replace=False) for _ in range(P)]
            pop = cbf(series)
            d_off = torch.from_numpy(pop.offsets.astype(np.int64)).cuda()
            d_cols = torch.from_numpy(pop.col_indices.astype(np.int16)).cuda()
            d_cnt = torch.zeros(P, dtype=torch.int64, device="cuda")
            st = torch.cuda.current_stream().cuda_stream
            rc = _lib.lib.ebic_count_matches_device(ev.handle, d_off.data_ptr(), d_cols.data_ptr(), P,
                                                    int(pop.offsets[-1]), 0.0, 0, d_cnt.data_ptr(), None, st)
            if P == 2048:
                _lib.check(rc)
                torch.cuda.synchronize()
                want = port.count_matches(v, pop.offsets, pop.col_indices, 0.0)
                assert (d_cnt.cpu().numpy().astype(np.uint64) == want).all()
            else:
                assert rc != 0 and "2048 series" in _lib.lib.ebic_last_error().decode()
            # the host path splits any size exactly
            assert (ev.count_matches(pop, 0.0) == port.count_matches(v, pop.offsets, pop.col_indices, 0.0)).all()
