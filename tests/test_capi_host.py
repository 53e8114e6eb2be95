"""CPU-side checks of the product library and its host logic (no GPU calls).

- libebic_b200.so loads and exports every entry point include/ebic_b200.h declares.
- Host mirror of the reference data model: CBF encode/decode, chunk plans,
  sigma, Eq. 1 (bit-exact vs the oracle), error strings.
- The synthetic generator is bit-identical to the reference's ebic::generate.
"""
import re
from pathlib import Path

import numpy as np
import pytest

import oracle
import paper_1801_03039_b200 as eb
from paper_1801_03039_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
port = oracle.Port()


def declared_symbols():
    text = (ROOT / "include" / "ebic_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ebic_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    decl = declared_symbols()
    assert len(decl) >= 19
    for name in decl:
        assert hasattr(_lib.lib, name), name
    assert sorted(_lib.EXPORTED) == decl


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_abi_version():
    assert _lib.lib.ebic_abi_version() == 2


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(eb.EbicError, match="no CUDA device"):
        eb.Evaluator(np.zeros((4, 3)))


def test_cbf_fig2_kat():  # test_datamodel.cpp:108-118
    pop = eb.encode_population([[1, 4, 2], [4, 2], [2, 3, 5, 1, 4]])
    assert list(pop.offsets) == [0, 3, 5, 10]
    assert list(pop.col_indices) == [1, 4, 2, 4, 2, 2, 3, 5, 1, 4]
    assert pop.size() == 3
    assert list(pop.individual(1)) == [4, 2]


def test_cbf_round_trip():  # test_datamodel.cpp:120-136
    rng = np.random.default_rng(99)
    for _ in range(300):
        n_cols = int(rng.integers(3, 43))
        series = [list(map(int, rng.choice(n_cols, size=int(rng.integers(2, min(n_cols, 6) + 1)),
                                           replace=False))) for _ in range(int(rng.integers(1, 13)))]
        assert eb.decode_population(eb.encode_population(series)) == series


def test_cbf_errors():  # test_datamodel.cpp:138-165
    with pytest.raises(ValueError, match="empty population"):
        eb.encode_population([])
    with pytest.raises(ValueError, match="invalid series"):
        eb.encode_population([[3]])
    with pytest.raises(ValueError, match="invalid series"):
        eb.encode_population([[3, 3]])
    good = eb.CbfPopulation(np.array([0, 2, 4], np.uint64), np.array([0, 1, 1, 2], np.uint16))
    eb.decode_population(good)
    for off in ([1, 2, 4], [0, 2, 3], [0, 1, 4], [0, 4, 4]):
        with pytest.raises(RuntimeError, match="corrupt CBF"):
            eb.decode_population(eb.CbfPopulation(np.array(off, np.uint64), good.col_indices))


def test_series_validity():  # test_datamodel.cpp:167+
    assert eb.is_valid_series([0, 1], 4)
    assert not eb.is_valid_series([0], 4)
    assert not eb.is_valid_series([0, 0], 4)
    assert not eb.is_valid_series([0, 4], 4)


def test_chunk_plan_partitions():  # test_fitness.cpp:94-109
    for rows in (1, 2, 7, 100, 1001):
        for workers in (1, 2, 3, 8, 64):
            plan = eb.make_chunk_plan(rows, workers)
            lo = 0
            for r in plan.chunks:
                assert r.lo == lo and r.hi > r.lo
                lo = r.hi
            assert lo == rows and len(plan.chunks) <= workers
    with pytest.raises(ValueError, match="matrix has no rows"):
        eb.make_chunk_plan(0, 2)


def test_sigma_and_fitness_bit_exact_vs_oracle():
    for n in (1, 100, 150, 250, 1000, 20000, 25000, 200000):
        assert eb.default_sigma(n) == port.default_sigma(n)
    rng = np.random.default_rng(3)
    for sigma in (2, 4, 20, 400, 4000):
        for _ in range(400):
            c = int(rng.integers(0, 300000))
            ln = int(rng.integers(2, 40))
            a = eb.fitness_score(c, ln, eb.FitnessParams(sigma))
            b = port.fitness_score(c, ln, sigma)
            assert np.float64(a).view(np.uint64) == np.float64(b).view(np.uint64)


def test_host_row_predicates_match_oracle():
    rng = np.random.default_rng(5)
    v = np.round(rng.standard_normal((50, 8)), 1)
    m = eb.ExpressionMatrix(v)
    for _ in range(50):
        s = list(map(int, rng.choice(8, size=int(rng.integers(2, 6)), replace=False)))
        for eps in (0.0, 0.1):
            for r in range(50):
                assert eb.row_matches(m, r, s, eps) == port.row_matches(v, r, s, eps)
                assert eb.trend_violations(m, r, s, eps) == port.trend_violations(v, r, s, eps)


@pytest.mark.skipif(not oracle.REF_LIB.exists(), reason="oracle/_ref not built")
def test_synth_generate_matches_reference_generator():
    ref = oracle.Ref()
    for pat in range(6):
        for (rows, cols, blocks, ov) in [(300, 40, [(30, 8), (30, 8)], 3), (150, 100, [(15, 15)] * 3, 0)]:
            noise = 0.2 if pat % 2 else 0.0
            spec = eb.ScenarioSpec(rows, cols, blocks, eb.Pattern(pat), ov, ov, noise, 100 + pat)
            a = eb.synth_generate(spec).values
            b = ref.generate(rows, cols, blocks, pat, ov, ov, noise, 100 + pat)
            assert (a.view(np.uint64) == b.view(np.uint64)).all()


@pytest.mark.parametrize("pat", range(6))
def test_synth_generate_bulk_path_matches_reference(pat):
    """Matrices above 2^17 cells take the multi-threaded background fill
    (raw engine draws in order, Box-Muller pairs in parallel); odd cell counts
    and a spare normal left by the pattern draws (odd column / row counts)
    exercise its edges."""
    ref = oracle.Ref()
    for (rows, cols) in [(1001, 263), (700, 401), (640, 512)]:
        blocks = [(40, 9), (35, 7)]
        noise = 0.3 if pat % 2 else 0.0
        spec = eb.ScenarioSpec(rows, cols, blocks, eb.Pattern(pat), 2, 2, noise, 7 + pat)
        a = eb.synth_generate(spec).values
        b = ref.generate(rows, cols, blocks, pat, 2, 2, noise, 7 + pat)
        assert (a.view(np.uint64) == b.view(np.uint64)).all(), (rows, cols)


def test_synth_generate_errors():
    with pytest.raises(ValueError):
        eb.synth_generate(eb.ScenarioSpec(0, 10, [], eb.Pattern(0)))
    with pytest.raises(RuntimeError):
        eb.synth_generate(eb.ScenarioSpec(10, 10, [(20, 2)], eb.Pattern(0)))


def test_null_fitness_plateau_matches_reference_formula():
    # io.hpp:132-143 restated on the host; value must exceed the fitness of any
    # junk series of length 2 on a 500-row matrix.
    p = eb.null_fitness_plateau(500, 10)
    assert p >= eb.fitness_score(250, 2, eb.FitnessParams(10))


def test_cross_rank_group_rejects_bad_arguments():
    """ebic_xgroup_* argument checks run before any device work."""
    import ctypes as C
    h = (C.c_ubyte * 64)()
    g = _lib.vp()
    L = _lib.lib
    assert L.ebic_xgroup_create(None, 16, b"/x", h) == _lib.EBIC_ERR_INVALID_ARGUMENT
    assert L.ebic_xgroup_join(None, h, b"/x", 2, 16, C.byref(g)) == _lib.EBIC_ERR_INVALID_ARGUMENT
    assert L.ebic_xgroup_count(None, None, None, 1, 1, 0.0, 4, 0, 1, None) == _lib.EBIC_ERR_INVALID_ARGUMENT
    assert L.ebic_xgroup_wait(None, 1, 1, None, None) == _lib.EBIC_ERR_INVALID_ARGUMENT
    assert L.ebic_xgroup_evaluate(None, None, None, 1, 4, 0.0, 1, None, None) == _lib.EBIC_ERR_INVALID_ARGUMENT
    assert L.ebic_xgroup_destroy(None) == 0
