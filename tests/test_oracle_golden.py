"""Pins the CPU oracle (oracle/ebic_oracle.c) to the reference.

1. Known-answer tests restated from the reference's own unit tests.
2. Golden vectors produced by the reference itself (tests/golden/make_golden.py).
3. When oracle/_ref (reference headers compiled here) is present, a seeded
   differential sweep oracle == reference.
"""
import math

import numpy as np
import pytest

import oracle
from golden_io import TRACE_NAMES, acceptance, expansion_cases, fitness_trials, trace

port = oracle.Port()


def cbf(series):
    off = np.zeros(len(series) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(s) for s in series])
    return off, np.array([c for s in series for c in s], dtype=np.uint16)


# ---- KATs restated from proj/tests/test_fitness.cpp ------------------------
def test_default_sigma_kat():  # test_fitness.cpp:27-34
    for n, s in [(150, 4), (100, 4), (250, 5), (1000, 20), (25000, 500), (1, 4)]:
        assert port.default_sigma(n) == s


def test_fitness_zero_below_two_rows():  # test_fitness.cpp:36-41
    for c in (0, 1, 2):
        assert port.fitness_score(c, 5, 4) == 0.0


def test_fitness_closed_form():  # test_fitness.cpp:43-71
    assert math.isclose(port.fitness_score(10, 5, 4), 5 * math.log(9.0), rel_tol=1e-12)
    assert math.isclose(port.fitness_score(3, 7, 4), 2 ** -1 * 7 * math.log(2.0), rel_tol=1e-12)
    for sigma in (2, 4, 20):
        for count in range(65):
            for ln in range(2, 25):
                exp = 0.0 if count <= 1 else 2.0 ** min(count - sigma, 0) * ln * math.log(count - 1)
                got = port.fitness_score(count, ln, sigma)
                if exp == 0.0:
                    assert got == 0.0
                else:
                    assert math.isclose(got, exp, rel_tol=1e-9)


def test_fitness_monotone():  # test_fitness.cpp:73-79
    f = port.fitness_score
    assert f(10, 5, 4) > f(9, 5, 4)
    assert f(10, 6, 4) > f(10, 5, 4)
    assert f(3, 5, 4) < f(4, 5, 4) / 1.5


def test_row_matches_kat():  # test_fitness.cpp:81-92
    m = np.array([[1, 2, 3], [3, 2, 1], [1, 1, 2]], dtype=np.float64)
    s = [0, 1, 2]
    assert port.row_matches(m, 0, s)
    assert not port.row_matches(m, 1, s)
    assert not port.row_matches(m, 2, s)
    assert port.row_matches(m, 2, s, 1e-9)
    assert not port.row_matches(m, 1, s, 1.0)
    assert port.row_matches(m, 1, s, 1.01 + 1e-12)


def test_count_matches_no_rows():  # fitness.hpp:31
    with pytest.raises(ValueError, match="matrix has no rows"):
        port.count_matches(np.zeros((0, 3)), *cbf([[0, 1]]))


# ---- KATs restated from proj/tests/test_expansion.cpp ----------------------
def test_assign_rows_kat():  # test_expansion.cpp:39-45
    m = np.array([[1, 2], [2, 1], [3, 4]], dtype=np.float64)
    assert port.assign_rows(m, [0, 1]) == [0, 2]
    assert port.assign_rows(m, [1, 0]) == [1]


def test_violations_kat():  # test_expansion.cpp:64-89
    m = np.array([[1, 2, 3, 4], [1, 2, 4, 3], [2, 1, 4, 3], [4, 3, 2, 1]], dtype=np.float64)
    assert [port.trend_violations(m, r, [0, 1, 2, 3]) for r in range(4)] == [0, 1, 2, 3]
    tie = np.array([[4, 4]], dtype=np.float64)
    assert port.trend_violations(tie, 0, [0, 1]) == 1
    assert port.trend_violations(tie, 0, [0, 1], 0.5) == 0


def test_expansion_kat():  # test_expansion.cpp:100-118
    m = np.array([[1, 2, 3, 4], [4, 3, 2, 1], [1, 2, 4, 3], [2, 1, 4, 3], [5, 1, 2, 3],
                  [1, 1, 1, 1]], dtype=np.float64)
    core = port.assign_rows(m, [0, 1, 2, 3])
    assert core == [0]
    rows, flags = port.expand_bicluster(m, [0, 1, 2, 3], core, [0])
    assert rows == [0, 1, 2, 4]
    assert flags == [0, 1, 2, 2]


def test_negative_outranks_approximate():  # test_expansion.cpp:120-134
    m = np.array([[1, 2], [2, 1]], dtype=np.float64)
    assert port.expand_bicluster(m, [0, 1], [0], [0], True, 1) == ([0, 1], [0, 1])
    assert port.expand_bicluster(m, [0, 1], [0], [0], False, 1) == ([0, 1], [0, 2])


# ---- golden vectors from the reference -------------------------------------
def test_acceptance_match_counts_golden():  # acceptance_main.cpp:233-292
    z = acceptance()
    for i, eps in enumerate(z["eps"]):
        for workers in (1, 2, 3, 8):
            got = port.count_matches(z["values"], z["offsets"], z["cols"], eps, workers)
            assert (got == z[f"counts_{i}"]).all()
        _, fit = port.evaluate_population(z["values"], z["offsets"], z["cols"], int(z["sigma"]), eps)
        assert (fit.view(np.uint64) == z[f"fitness_{i}"].view(np.uint64)).all()


def test_fitness_trials_golden():  # test_fitness.cpp:111-137
    n = 0
    for v, off, cols, eps, counts in fitness_trials():
        for workers in (1, 2, 3, 8):
            assert (port.count_matches(v, off, cols, eps, workers) == counts).all()
        n += 1
    assert n == 100


def test_expansion_golden():
    n = 0
    for case in expansion_cases():
        v = case["matrix"]
        core = port.assign_rows(v, case["series"], case["eps"])
        assert core == [int(r) for r in case["core"]]
        rows, flags = port.expand_bicluster(v, case["series"], core, [0] * len(core),
                                            case["allow_negative"], case["approx_k"], case["eps"])
        assert rows == [int(r) for r in case["rows"]]
        assert flags == [int(f) for f in case["flags"]]
        n += 1
    assert n == 48


@pytest.mark.parametrize("name", [t for t in TRACE_NAMES if t not in ("c4", "c5")])
def test_trace_golden(name):
    t = trace(name)
    v = t.matrix()
    for off, cols, counts, fit in t.batches:
        c, f = port.evaluate_population(v, off, cols, t.sigma, t.eps)
        assert (c == counts).all()
        assert (f.view(np.uint64) == fit.view(np.uint64)).all()


def test_trace_c4_first_batch_golden():
    t = trace("c4")
    v = t.matrix()
    off, cols, counts, fit = t.batches[0]
    c, f = port.evaluate_population(v, off, cols, t.sigma, t.eps)
    assert (c == counts).all()
    assert (f.view(np.uint64) == fit.view(np.uint64)).all()


# ---- direct differential check against the compiled reference --------------
@pytest.mark.skipif(not oracle.REF_LIB.exists(), reason="oracle/_ref not built")
def test_port_equals_reference_sweep():
    ref = oracle.Ref()
    rng = np.random.default_rng(11)
    for trial in range(40):
        R, Cn = int(rng.integers(1, 400)), int(rng.integers(3, 60))
        v = rng.standard_normal((R, Cn))
        if trial % 3 == 0:
            v = np.round(v, 1)
        P = int(rng.integers(1, 60))
        series = [list(rng.choice(Cn, size=int(rng.integers(2, min(Cn, 9) + 1)), replace=False))
                  for _ in range(P)]
        off, cols = cbf(series)
        eps = [0.0, 1e-9, 0.1, 0.5][trial % 4]
        m = ref.matrix(v)
        assert (port.count_matches(v, off, cols, eps, 3) == ref.count_matches(m, off, cols, eps, 3)).all()
        _, f = port.evaluate_population(v, off, cols, 7, eps)
        assert (f.view(np.uint64) == ref.evaluate_population(m, off, cols, 7, eps).view(np.uint64)).all()
