#!/usr/bin/env python
"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Runs in the build container only (needs oracle/_ref/libebic_ref.so, which
oracle/Makefile compiles from the unmodified headers under /root/reference).
Every expected value in the fixtures is produced by the reference's own
functions (count_matches, evaluate_population / fitness_score, assign_rows,
expand_bicluster, the GA run() loop via RunHooks::on_evaluate); the inputs are
the reference tests' own input streams where those exist.

    python tests/golden/make_golden.py            # all fixtures
    python tests/golden/make_golden.py --only c4  # one trace
"""
from __future__ import annotations

import argparse
import ctypes as C
import hashlib
import json
import os
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402

OUT = Path(__file__).resolve().parent

# BASELINE.json configs (SURVEY.md §8d / Appendix B mapping).
TRACES = {
    # name: (rows, cols, blocks, pattern, overlap, noise, seed, eps, batches, population)
    "c1": (500, 100, [(50, 10)] * 3, 0, 0, 0.0, 1, 0.0, 30, 600),
    "c1e": (500, 100, [(50, 10)] * 3, 0, 0, 0.0, 1, 1e-9, 30, 600),
    "c2_shift": (1000, 100, [(100, 10)] * 3, 3, 0, 0.0, 2, 1e-9, 10, 600),
    "c2_scale": (1000, 100, [(100, 10)] * 3, 4, 0, 0.0, 3, 1e-9, 10, 600),
    "c2_shiftscale": (1000, 100, [(100, 10)] * 3, 5, 0, 0.0, 4, 1e-9, 10, 600),
    "c3": (5000, 200, [(200, 20)] * 5, 0, 5, 0.0, 5, 1e-9, 10, 600),
    "c3_noise": (5000, 200, [(200, 20)] * 5, 0, 5, 0.35, 6, 0.2, 6, 600),
    "c4": (20000, 500, [(600, 20)] * 5, 0, 0, 0.0, 2026, 1e-9, 8, 600),
    "c5": (200000, 1000, [(6000, 30)] * 5, 0, 0, 0.0, 2027, 1e-9, 3, 600),
}


# Steady-state traces (late-run batches): the early
# generations plus a sparse sample of the run up to `iterations`.
STEADY = {
    # name: (base trace, iterations, record_first, record_every)
    "c4ss": ("c4", 5000, 8, 250),
    "c5ss": ("c5", 1000, 50, 100),
}


def sha(values: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(values, dtype=np.float64).tobytes()).hexdigest()


def fixture_acceptance(ref: oracle.Ref) -> None:
    """acceptance_main.cpp:233-271 -- 300x30, 500 series, eps in {0, 0.1, 0.5}."""
    v = np.zeros(300 * 30)
    off = np.zeros(501, dtype=np.uint64)
    cols = np.zeros(3500, dtype=np.uint16)
    ref.lib.ref_fixture_acceptance_match_counts(v.ctypes.data_as(oracle.f64p),
                                                off.ctypes.data_as(oracle.szp),
                                                cols.ctypes.data_as(oracle.u16p))
    v = v.reshape(300, 30)
    cols = cols[:int(off[-1])]
    m = ref.matrix(v)
    out = dict(values=v, offsets=off, cols=cols, eps=np.array([0.0, 0.1, 0.5]))
    sigma = int(ref.lib.ref_default_sigma(300))
    out["sigma"] = np.array(sigma)
    for i, eps in enumerate([0.0, 0.1, 0.5]):
        counts = {w: ref.count_matches(m, off, cols, eps, workers=w) for w in (1, 2, 3, 8)}
        for w in (2, 3, 8):
            assert (counts[w] == counts[1]).all()
        out[f"counts_{i}"] = counts[1]
        out[f"fitness_{i}"] = ref.evaluate_population(m, off, cols, sigma, eps, workers=2)
    np.savez_compressed(OUT / "acceptance_match_counts.npz", **out)


def fixture_fitness_trials(ref: oracle.Ref) -> None:
    """test_fitness.cpp:111-137 -- the 100 chunk-invariance trials of Rng(4242)."""
    vals, offs, cols, meta, counts = [], [], [], [], []
    L = ref.lib
    L.ref_fixture_fitness_trial.argtypes = [C.c_int, oracle.szp, oracle.szp, C.POINTER(C.c_double),
                                           oracle.szp, oracle.f64p, oracle.szp, oracle.u16p]
    for t in range(100):
        r, c, n = C.c_size_t(), C.c_size_t(), C.c_size_t()
        e = C.c_double()
        v = np.zeros(124 * 22)
        o = np.zeros(11, dtype=np.uint64)
        s = np.zeros(60, dtype=np.uint16)
        L.ref_fixture_fitness_trial(t, C.byref(r), C.byref(c), C.byref(e), C.byref(n),
                                    v.ctypes.data_as(oracle.f64p), o.ctypes.data_as(oracle.szp),
                                    s.ctypes.data_as(oracle.u16p))
        R, Cc, N = r.value, c.value, n.value
        v = v[:R * Cc].reshape(R, Cc)
        o = o[:N + 1]
        s = s[:int(o[-1])]
        m = ref.matrix(v)
        got = {w: ref.count_matches(m, o, s, e.value, workers=w) for w in (1, 2, 3, 8)}
        for w in (2, 3, 8):
            assert (got[w] == got[1]).all()
        vals.append(v.ravel()); offs.append(o); cols.append(s); counts.append(got[1])
        meta.append((R, Cc, N, e.value))
    np.savez_compressed(
        OUT / "fitness_trials.npz",
        values=np.concatenate(vals), offsets=np.concatenate(offs), cols=np.concatenate(cols),
        counts=np.concatenate(counts),
        shape=np.array([(m[0], m[1], m[2]) for m in meta], dtype=np.uint64),
        eps=np.array([m[3] for m in meta]))


# (rows, cols, blocks, pattern, overlap_rows, overlap_cols, noise, seed)
C3LIKE = (5000, 200, [(200, 20)] * 5, 0, 5, 5, 0.2, 77)


def fixture_expansion(ref: oracle.Ref) -> None:
    """test_expansion.cpp:148-188 matrices (Rng seeds 46/48) plus a C3-shaped scenario
    with overlaps and noise; reference assign_rows + expand_bicluster results for
    several options and epsilons."""
    cases = []
    L = ref.lib
    L.ref_fixture_random_matrix.argtypes = [C.c_size_t, C.c_size_t, C.c_uint64, oracle.f64p]

    def rand_matrix(rows, cols, seed):
        v = np.zeros(rows * cols)
        L.ref_fixture_random_matrix(rows, cols, seed, v.ctypes.data_as(oracle.f64p))
        return v.reshape(rows, cols)

    mats = {
        "rand80x10": rand_matrix(80, 10, 46),
        "rand60x9": rand_matrix(60, 9, 48),
        "c3like": ref.generate(*C3LIKE),
        "ties": np.round(rand_matrix(300, 12, 5), 1),
    }
    rng = np.random.default_rng(2024)
    out = {}
    k = 0
    for name, v in mats.items():
        m = ref.matrix(v)
        if name == "c3like":  # regenerated bit-identically by synth_generate in the tests
            out["c3like_sha256"] = np.array(sha(v))
        else:
            out[f"m_{name}"] = v
        for trial in range(12):
            ncols = v.shape[1]
            ln = int(rng.integers(2, min(ncols, 8) + 1))
            series = rng.choice(ncols, size=ln, replace=False).astype(np.uint16)
            eps = [0.0, 1e-9, 0.1][trial % 3]
            allow_neg = trial % 4 != 3
            approx_k = [1, 0, 2, 1][trial % 4]
            core = ref.assign_rows(m, series, eps)
            rows, flags = ref.expand_bicluster(m, series, core, [0] * len(core), allow_neg,
                                               approx_k, eps)
            out[f"c{k}_series"] = series
            out[f"c{k}_core"] = np.array(core, dtype=np.uint64)
            out[f"c{k}_rows"] = np.array(rows, dtype=np.uint64)
            out[f"c{k}_flags"] = np.array(flags, dtype=np.uint8)
            out[f"c{k}_meta"] = np.array([eps, float(allow_neg), float(approx_k)])
            out[f"c{k}_matrix"] = np.array(name)
            k += 1
    out["n_cases"] = np.array(k)
    np.savez_compressed(OUT / "expansion_cases.npz", **out)


def fixture_trace(ref: oracle.Ref, name: str) -> None:
    rows, cols, blocks, pattern, overlap, noise, seed, eps, batches, pop = TRACES[name]
    v = ref.generate(rows, cols, blocks, pattern, overlap, overlap, noise, seed)
    m = ref.matrix(v)
    sigma = int(ref.lib.ref_default_sigma(rows))
    with tempfile.TemporaryDirectory() as td:
        path = Path(td) / "trace.bin"
        n = ref.run_trace(m, path, population=pop, iterations=batches - 1, rng_seed=1, eps=eps,
                          sigma=0, threads=8, max_batches=batches)
        trace = oracle.read_trace(path)
    assert n == len(trace)
    lens, cols_all, counts, fits, sizes = [], [], [], [], []
    for off, c, cnt in trace:
        lens.append(np.diff(off).astype(np.uint16))
        cols_all.append(c)
        counts.append(cnt)
        fits.append(ref.evaluate_population(m, off, c, sigma, eps, workers=8))
        sizes.append(len(cnt))
    np.savez_compressed(
        OUT / f"trace_{name}.npz",
        spec=np.array(json.dumps(dict(rows=rows, cols=cols, blocks=blocks, pattern=pattern,
                                      overlap=overlap, noise=noise, seed=seed))),
        matrix_sha256=np.array(sha(v)), eps=np.array(eps), sigma=np.array(sigma),
        batch_sizes=np.array(sizes, dtype=np.uint32), lens=np.concatenate(lens),
        cols=np.concatenate(cols_all), counts=np.concatenate(counts).astype(np.uint32),
        fitness=np.concatenate(fits))
    print(f"trace {name}: {len(trace)} batches, {sum(sizes)} series", flush=True)


def fixture_trace_steady(ref: oracle.Ref, name: str) -> None:
    base, iterations, first, every = STEADY[name]
    rows, cols, blocks, pattern, overlap, noise, seed, eps, _, pop = TRACES[base]
    v = ref.generate(rows, cols, blocks, pattern, overlap, overlap, noise, seed)
    m = ref.matrix(v)
    sigma = int(ref.lib.ref_default_sigma(rows))
    threads = os.cpu_count() or 8
    with tempfile.TemporaryDirectory() as td:
        path = Path(td) / "trace.bin"
        n = ref.run_trace_sel(m, path, population=pop, iterations=iterations, rng_seed=1, eps=eps,
                              sigma=0, threads=threads, record_first=first, record_every=every)
        trace = oracle.read_trace_sel(path)
    assert n == len(trace)
    gens, lens, cols_all, counts, fits, sizes = [], [], [], [], [], []
    for k, off, c, cnt in trace:
        gens.append(k)
        lens.append(np.diff(off).astype(np.uint16))
        cols_all.append(c)
        counts.append(cnt)
        fits.append(ref.evaluate_population(m, off, c, sigma, eps, workers=threads))
        sizes.append(len(cnt))
    np.savez_compressed(
        OUT / f"trace_{name}.npz",
        spec=np.array(json.dumps(dict(rows=rows, cols=cols, blocks=blocks, pattern=pattern,
                                      overlap=overlap, noise=noise, seed=seed))),
        matrix_sha256=np.array(sha(v)), eps=np.array(eps), sigma=np.array(sigma),
        generations=np.array(gens, dtype=np.uint32), iterations=np.array(iterations),
        batch_sizes=np.array(sizes, dtype=np.uint32), lens=np.concatenate(lens),
        cols=np.concatenate(cols_all), counts=np.concatenate(counts).astype(np.uint32),
        fitness=np.concatenate(fits))
    print(f"trace {name}: {len(trace)} batches (generations {gens[0]}..{gens[-1]}), "
          f"{sum(sizes)} series", flush=True)


# TopRankList::update sequences: whole populations as the
# reference GA passes them to the list (elite clones + novel), and the random
# stress streams with many fitness ties and column collisions.
TOP_RANK_RUNS = {
    # name: (rows, cols, blocks, seed, eps, generations, threshold, capacity)
    "c1": (500, 100, [(50, 10)] * 3, 1, 0.0, 60, 0.75, 100),
    "c4": (20000, 500, [(600, 20)] * 5, 2026, 1e-9, 12, 0.75, 100),
}


def _stress_updates(seed: int):
    rng = np.random.default_rng(seed)
    n_cols = int(rng.integers(6, 140))
    thr = float(rng.choice([0.75, 0.5, 1.0, 0.25, 0.6]))
    cap = int(rng.choice([1, 3, 20, 100]))
    ups = []
    for _ in range(int(rng.integers(2, 10))):
        P = int(rng.integers(1, 200))
        pool = rng.choice(n_cols, size=min(n_cols, int(rng.integers(4, 40))), replace=False)
        series = [rng.choice(pool, size=min(len(pool), int(rng.integers(2, 10))), replace=False)
                  for _ in range(P)]
        off = np.zeros(P + 1, dtype=np.uint64)
        off[1:] = np.cumsum([len(x) for x in series])
        fit = rng.integers(-2, 10, size=P).astype(np.float64) * 0.25
        ups.append((off, np.concatenate(series).astype(np.uint16), fit))
    return n_cols, thr, cap, ups


def fixture_top_rank(ref: oracle.Ref) -> None:
    streams = []
    for name, (rows, cols, blocks, seed, eps, gens, thr, cap) in TOP_RANK_RUNS.items():
        v = ref.generate(rows, cols, blocks, 0, 0, 0, 0.0, seed)
        m = ref.matrix(v)
        with tempfile.TemporaryDirectory() as td:
            path = Path(td) / "pop.bin"
            ref.run_population_trace(m, path, population=600, iterations=gens - 1, rng_seed=1,
                                     eps=eps, sigma=0, threads=8)
            streams.append((name, cols, thr, cap, oracle.read_population_trace(path)))
    for k in range(24):
        n_cols, thr, cap, ups = _stress_updates(100 + k)
        streams.append((f"stress{k}", n_cols, thr, cap, ups))
    out = {"names": np.array([s[0] for s in streams]),
           "n_cols": np.array([s[1] for s in streams], dtype=np.uint32),
           "threshold": np.array([s[2] for s in streams]),
           "capacity": np.array([s[3] for s in streams], dtype=np.uint32)}
    for i, (name, n_cols, thr, cap, ups) in enumerate(streams):
        t = ref.top_rank(n_cols)
        p_sizes, p_lens, p_cols, p_fit = [], [], [], []
        e_sizes, e_lens, e_cols, e_fit, e_seq = [], [], [], [], []
        for off, c, fit in ups:
            t.update(off, c, fit, thr, cap)
            eo, ec, ef, es = t.entries()
            p_sizes.append(len(fit)); p_lens.append(np.diff(off)); p_cols.append(c); p_fit.append(fit)
            e_sizes.append(len(ef)); e_lens.append(np.diff(eo)); e_cols.append(ec)
            e_fit.append(ef); e_seq.append(es)
        out[f"s{i}_pop_sizes"] = np.array(p_sizes, dtype=np.uint32)
        out[f"s{i}_pop_lens"] = np.concatenate(p_lens).astype(np.uint16)
        out[f"s{i}_pop_cols"] = np.concatenate(p_cols).astype(np.uint16)
        out[f"s{i}_pop_fitness"] = np.concatenate(p_fit)
        out[f"s{i}_top_sizes"] = np.array(e_sizes, dtype=np.uint32)
        out[f"s{i}_top_lens"] = np.concatenate(e_lens).astype(np.uint16)
        out[f"s{i}_top_cols"] = np.concatenate(e_cols).astype(np.uint16)
        out[f"s{i}_top_fitness"] = np.concatenate(e_fit)
        out[f"s{i}_top_seq"] = np.concatenate(e_seq).astype(np.uint64)
        print(f"top_rank {name}: {len(ups)} updates, final size {e_sizes[-1]}", flush=True)
    np.savez_compressed(OUT / "top_rank_updates.npz", **out)


def fixture_dropin_json() -> None:
    """Reference `ebic run` output (byte-exact target for the drop-in binary)."""
    args = ["rows=500", "cols=100", "blocks=50x10,50x10,50x10", "seed=1", "population=600",
            "iterations=300", "rng_seed=42", "epsilon=1e-9", "overlap_threshold=0.5",
            "threshold=none", "threads=1"]
    with tempfile.TemporaryDirectory() as td:
        out = Path(td) / "ref.json"
        subprocess.run([str(oracle.REF_RUN), *args, f"out={out}"], check=True)
        (OUT / "dropin_c1.json").write_bytes(out.read_bytes())
    (OUT / "dropin_c1.args").write_text(" ".join(args) + "\n")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    oracle.build(ref=True)
    ref = oracle.Ref()
    jobs = {"acceptance": lambda: fixture_acceptance(ref),
            "trials": lambda: fixture_fitness_trials(ref),
            "expansion": lambda: fixture_expansion(ref),
            "dropin": fixture_dropin_json,
            "top_rank": lambda: fixture_top_rank(ref)}
    for t in TRACES:
        jobs[t] = (lambda t=t: fixture_trace(ref, t))
    for t in STEADY:
        jobs[t] = (lambda t=t: fixture_trace_steady(ref, t))
    for name, job in jobs.items():
        if a.only and name != a.only:
            continue
        job()
        print("ok", name, flush=True)


if __name__ == "__main__":
    main()
