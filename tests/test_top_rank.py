"""TopRankList::update (evolution.hpp:168-206) -- SURVEY.md §8(f) rank 1.

The product implementation is ebic_top_rank_update in libebic_b200.so (host
C++, csrc/toprank.cpp), reached through the Python mirror TopRankList and the
shadow include/ebic/evolution.hpp.  It is checked, update by update, against:

* tests/golden/top_rank_updates.npz -- populations exactly as the reference GA
  hands them to its top-rank list (C1 for 60 generations, C4 for 12), plus
  random streams with many fitness ties and column collisions, with the
  reference TopRankList's entries (series, fitness, seq) after every update;
* the C restatement oracle/ebic_oracle.c:orc_top_rank_update (pinned to the
  same fixture);
* the compiled reference itself (oracle/_ref) on fresh random streams.
Host-only code: these run on CPU.
"""
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_1801_03039_b200 import CbfPopulation, TopRankList

GOLDEN = Path(__file__).resolve().parent / "golden" / "top_rank_updates.npz"


def _split(sizes, lens, cols, *per_item):
    """Per-update (offsets, cols, *per-item arrays) from concatenated fixture arrays."""
    out, li, ci = [], 0, 0
    for n in sizes.tolist():
        ln = lens[li:li + n].astype(np.uint64)
        off = np.zeros(n + 1, dtype=np.uint64)
        np.cumsum(ln, out=off[1:])
        c = cols[ci:ci + int(off[-1])]
        out.append((off, c, *[a[li:li + n] for a in per_item]))
        li += n
        ci += int(off[-1])
    return out


def golden_streams():
    z = np.load(GOLDEN)
    for i, name in enumerate(z["names"].tolist()):
        pops = _split(z[f"s{i}_pop_sizes"], z[f"s{i}_pop_lens"], z[f"s{i}_pop_cols"],
                      z[f"s{i}_pop_fitness"])
        tops = _split(z[f"s{i}_top_sizes"], z[f"s{i}_top_lens"], z[f"s{i}_top_cols"],
                      z[f"s{i}_top_fitness"], z[f"s{i}_top_seq"])
        yield (name, int(z["n_cols"][i]), float(z["threshold"][i]), int(z["capacity"][i]),
               pops, tops)


STREAMS = list(golden_streams())


def _same(top: TopRankList, expected) -> bool:
    off, cols, fit, seq = expected
    return (np.array_equal(top._off, off) and np.array_equal(top._cols, cols)
            and np.array_equal(top._fit, fit) and np.array_equal(top._seq, seq))


@pytest.mark.parametrize("stream", STREAMS, ids=[s[0] for s in STREAMS])
def test_library_matches_reference_fixture(stream):
    name, n_cols, thr, cap, pops, tops = stream
    top = TopRankList(n_cols)
    for u, ((off, cols, fit), expected) in enumerate(zip(pops, tops)):
        top.update(CbfPopulation(off, cols), fit, thr, cap)
        assert _same(top, expected), f"{name}: update {u} differs"
    assert top.best_fitness() == (float(tops[-1][2][0]) if len(tops[-1][2]) else 0.0)


@pytest.mark.parametrize("stream", STREAMS, ids=[s[0] for s in STREAMS])
def test_oracle_matches_reference_fixture(stream):
    """Pins the C restatement to the reference's own outputs."""
    name, n_cols, thr, cap, pops, tops = stream
    port = oracle.Port()
    ent = (np.zeros(1, np.uint64), np.zeros(0, np.uint16), np.zeros(0), np.zeros(0, np.uint64))
    nseq = 0
    for u, ((off, cols, fit), (e_off, e_cols, e_fit, e_seq)) in enumerate(zip(pops, tops)):
        ref, seq, nseq = port.top_rank_update(n_cols, ent, off, cols, fit, thr, cap, nseq)
        segs, fits = [], []
        for r in ref.tolist():
            if r < 0:
                segs.append(cols[int(off[-r - 1]):int(off[-r])]); fits.append(fit[-r - 1])
            else:
                segs.append(ent[1][int(ent[0][r]):int(ent[0][r + 1])]); fits.append(ent[2][r])
        new_off = np.zeros(len(segs) + 1, dtype=np.uint64)
        np.cumsum([len(x) for x in segs], out=new_off[1:])
        ent = (new_off, np.concatenate(segs).astype(np.uint16) if segs else np.zeros(0, np.uint16),
               np.array(fits, dtype=np.float64), seq.copy())
        assert np.array_equal(ent[0], e_off) and np.array_equal(ent[1], e_cols), f"{name}: {u}"
        assert np.array_equal(ent[2], e_fit) and np.array_equal(ent[3], e_seq), f"{name}: {u}"


def _random_stream(rng, dup_columns=False):
    n_cols = int(rng.integers(4, 300))
    thr = float(rng.choice([0.75, 0.5, 1.0, 0.1, 0.34, 0.999]))
    cap = int(rng.choice([1, 2, 7, 100]))
    ups = []
    for _ in range(int(rng.integers(1, 8))):
        P = int(rng.integers(0, 300))
        pool = rng.choice(n_cols, size=min(n_cols, int(rng.integers(2, 50))), replace=False)
        series = [rng.choice(pool, size=int(rng.integers(2, 12)) if dup_columns else
                             min(len(pool), int(rng.integers(2, 12))), replace=dup_columns)
                  for _ in range(P)]
        off = np.zeros(P + 1, dtype=np.uint64)
        off[1:] = np.cumsum([len(x) for x in series]) if P else []
        cols = np.concatenate(series).astype(np.uint16) if P else np.zeros(0, np.uint16)
        fit = rng.integers(-3, 8, size=P).astype(np.float64) * rng.choice([1.0, 0.1, 1e-300])
        ups.append((off, cols, fit))
    return n_cols, thr, cap, ups


@pytest.mark.skipif(not oracle.REF_LIB.exists(), reason="oracle/_ref not built")
@pytest.mark.parametrize("dups", [False, True])
def test_library_matches_compiled_reference_random(dups):
    ref = oracle.Ref()
    for seed in range(60):
        n_cols, thr, cap, ups = _random_stream(np.random.default_rng(1000 * dups + seed), dups)
        mine, theirs = TopRankList(n_cols), ref.top_rank(n_cols)
        for off, cols, fit in ups:
            mine.update(CbfPopulation(off, cols), fit, thr, cap)
            theirs.update(off, cols, fit, thr, cap)
            assert _same(mine, theirs.entries()), f"seed {seed}"


def test_series_list_input_and_entries_view():
    top = TopRankList(10)
    top.update([[0, 1, 2], [0, 1, 3], [5, 6], [7, 8]], [3.0, 2.0, 2.0, -1.0], 0.5, 100)
    # [0,1,3] overlaps [0,1,2] by 2/3 > 0.5 and has lower fitness: blocked.
    assert [(e.series, e.fitness, e.seq) for e in top.entries()] == [([0, 1, 2], 3.0, 0),
                                                                  ([5, 6], 2.0, 1)]
    top.update([[0, 1, 4, 5]], [4.0], 0.5, 100)  # evicts [0,1,2] (2/3 > 0.5), keeps [5,6] (1/2)
    assert [(e.series, e.seq) for e in top.entries()] == [([0, 1, 4, 5], 2), ([5, 6], 1)]
    assert TopRankList.overlap([0, 1, 4, 5], [5, 6]) == 0.5
    assert TopRankList.overlap(top.entries()[0], top.entries()[1]) == 0.5
    assert len(top) == 2 and not top.empty() and top.best_fitness() == 4.0


@pytest.mark.skipif(not oracle.REF_LIB.exists(), reason="oracle/_ref not built")
@pytest.mark.parametrize("thr,cap", [(0.0, 100), (1.5, 100), (-0.5, 100), (float("nan"), 100),
                                     (0.75, 0), (-1.0, 3)])
def test_unvalidated_config_matches_reference(thr, cap):
    """update() does not validate cfg (run() does, evolution.hpp:41-63): out-of-range
    thresholds and a zero capacity behave exactly as in the reference."""
    ref = oracle.Ref()
    for seed in range(10):
        n_cols, _, _, ups = _random_stream(np.random.default_rng(7000 + seed))
        mine, theirs = TopRankList(n_cols), ref.top_rank(n_cols)
        for off, cols, fit in ups:
            mine.update(CbfPopulation(off, cols), fit, thr, cap)
            theirs.update(off, cols, fit, thr, cap)
            assert _same(mine, theirs.entries()), f"seed {seed}"


def test_column_out_of_range_is_rejected():
    top = TopRankList(10)
    with pytest.raises(ValueError, match="column out of range"):
        top.update([[0, 12]], [1.0], 0.75, 100)


def _raw_update(n_cols, entries, off, cols, fit, thr, cap, next_seq):
    """ebic_top_rank_update called directly (entries in any order)."""
    import ctypes as C
    from paper_1801_03039_b200 import _lib as L
    e_off, e_cols, e_fit, e_seq = (np.ascontiguousarray(entries[0], np.uint64),
                                   np.ascontiguousarray(entries[1], np.uint16),
                                   np.ascontiguousarray(entries[2], np.float64),
                                   np.ascontiguousarray(entries[3], np.uint64))
    pad = lambda a: a if a.size else np.zeros(1, dtype=a.dtype)  # noqa: E731
    p = lambda a, t: a.ctypes.data_as(t)  # noqa: E731
    k_off, k_cols, k_fit = (np.ascontiguousarray(off, np.uint64), pad(np.ascontiguousarray(cols, np.uint16)),
                            np.ascontiguousarray(fit, np.float64))
    n_e, n_c = len(e_fit), len(k_fit)
    slots = max(1, min(cap, n_e + n_c))
    ref, seq = np.zeros(slots, np.int64), np.zeros(slots, np.uint64)
    nxt, n = C.c_uint64(next_seq), C.c_size_t(0)
    L.check(L.lib.ebic_top_rank_update(n_cols, n_e, p(e_off, L.szp), p(pad(e_cols), L.u16p), p(pad(e_fit), L.f64p),
                                       p(pad(e_seq), L.u64p), n_c, p(k_off, L.szp), p(k_cols, L.u16p),
                                       p(pad(k_fit), L.f64p), float(thr), cap, C.byref(nxt), p(ref, L.i64p),
                                       p(seq, L.u64p), C.byref(n)))
    return ref[:n.value], seq[:n.value], nxt.value


@pytest.mark.parametrize("shuffled", [False, True])
def test_entries_in_any_order_match_oracle(shuffled):
    """The final order is a merge when the entries keep the list's own order
    (fitness desc, seq asc) and a sort otherwise; both agree with the oracle."""
    port = oracle.Port()
    for seed in range(40):
        rng = np.random.default_rng(9100 + seed)
        n_cols = int(rng.integers(6, 80))
        def pop(n):
            series = [rng.choice(n_cols, size=int(rng.integers(2, 6)), replace=False) for _ in range(n)]
            off = np.zeros(n + 1, np.uint64)
            off[1:] = np.cumsum([len(s) for s in series]) if n else []
            cols = np.concatenate(series).astype(np.uint16) if n else np.zeros(0, np.uint16)
            return off, cols, rng.integers(1, 6, size=n).astype(np.float64)
        n_e = int(rng.integers(0, 30))
        e_off, e_cols, e_fit = pop(n_e)
        e_seq = rng.permutation(1000)[:n_e].astype(np.uint64)
        if not shuffled:  # the list's own invariant
            order = sorted(range(n_e), key=lambda i: (-e_fit[i], e_seq[i]))
            segs = [e_cols[int(e_off[i]):int(e_off[i + 1])] for i in order]
            e_off = np.zeros(n_e + 1, np.uint64)
            e_off[1:] = np.cumsum([len(s) for s in segs]) if n_e else []
            e_cols = np.concatenate(segs).astype(np.uint16) if n_e else np.zeros(0, np.uint16)
            e_fit, e_seq = e_fit[order], e_seq[order]
        off, cols, fit = pop(int(rng.integers(0, 40)))
        thr, cap = float(rng.choice([0.3, 0.5, 0.75, 1.0])), int(rng.choice([3, 10, 100]))
        ent = (e_off, e_cols, e_fit, e_seq)
        got = _raw_update(n_cols, ent, off, cols, fit, thr, cap, 1000)
        want = port.top_rank_update(n_cols, ent, off, cols, fit, thr, cap, 1000)
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1]), seed
        assert got[2] == want[2], seed
