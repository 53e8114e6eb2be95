"""Drop-in proof: the reference's own GA + Steps 6-7 + JSON writer, compiled
against the repo's shadowing include/ebic/{fitness,expansion}.hpp and linked to
libebic_b200.so (oracle/_ref/ebic_dropin_run), must write byte-identical
results to the pure reference CPU build (oracle/_ref/ebic_ref_run / the
committed golden JSON) -- the reference's own determinism check
(acceptance_main.cpp:407-442) applied across implementations.
"""
import os
import subprocess
from pathlib import Path

import pytest

import oracle

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"

needs_dropin = pytest.mark.skipif(not oracle.DROPIN_RUN.exists(),
                                  reason="oracle/_ref/ebic_dropin_run not built")


def run(binary, args, out, env=None):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([str(binary), *args, f"out={out}"], capture_output=True, text=True, env=e,
                       timeout=900)
    assert r.returncode == 0, r.stderr
    return Path(out).read_bytes()


@needs_dropin
@pytest.mark.parametrize("gpus", ["0", "0,0,0"])
def test_dropin_matches_golden_json(tmp_path, gpus):
    args = (GOLDEN / "dropin_c1.args").read_text().split()
    got = run(oracle.DROPIN_RUN, args, tmp_path / "b200.json", {"EBIC_GPUS": gpus})
    assert got == (GOLDEN / "dropin_c1.json").read_bytes()


CONFIGS = {
    "c2_shift_approx2": ["rows=1000", "cols=100", "blocks=100x10,100x10,100x10", "pattern=shift",
                         "seed=2", "population=600", "iterations=80", "rng_seed=3", "epsilon=1e-9",
                         "approx=2", "threshold=none"],
    "c3_overlap_negative": ["rows=5000", "cols=200", "blocks=200x20,200x20,200x20,200x20,200x20",
                            "overlap=5", "seed=5", "population=600", "iterations=60", "rng_seed=1",
                            "epsilon=1e-9", "threshold=none"],
    "c3_noise_eps": ["rows=5000", "cols=200", "blocks=200x20,200x20,200x20", "noise=0.35", "seed=6",
                     "population=400", "iterations=60", "rng_seed=9", "epsilon=0.2",
                     "allow_negative=0"],
    # every other generator pattern, eps = 0, wide tabu keys (> 256 columns),
    # a narrow matrix that ends through the tabu list, another overlap threshold
    "scale_eps0": ["rows=1500", "cols=120", "blocks=120x12,120x12", "pattern=scale", "seed=11",
                   "population=500", "iterations=50", "rng_seed=4", "epsilon=0", "threshold=none"],
    "shift_scale_wide": ["rows=2000", "cols=300", "blocks=150x15,150x15", "pattern=shift_scale",
                         "seed=12", "population=600", "iterations=50", "rng_seed=5", "epsilon=1e-9",
                         "threshold=none"],
    "column_constant": ["rows=800", "cols=60", "blocks=80x8,80x8", "pattern=column_constant", "seed=13",
                        "population=300", "iterations=40", "rng_seed=6", "epsilon=1e-9"],
    "row_constant_overlap": ["rows=800", "cols=60", "blocks=80x8,80x8,80x8", "pattern=row_constant",
                             "overlap=2", "seed=14", "population=300", "iterations=40", "rng_seed=7",
                             "epsilon=1e-9", "overlap_threshold=0.3", "threshold=none"],
    "narrow_tabu_end": ["rows=300", "cols=6", "blocks=30x3", "seed=15", "population=200",
                        "iterations=400", "rng_seed=8", "epsilon=0", "threshold=none"],
}


@needs_dropin
@pytest.mark.skipif(not oracle.REF_RUN.exists(), reason="oracle/_ref/ebic_ref_run not built")
@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_dropin_matches_reference_binary(tmp_path, name):
    args = CONFIGS[name]
    want = run(oracle.REF_RUN, args + ["threads=8"], tmp_path / "ref.json")
    got = run(oracle.DROPIN_RUN, args, tmp_path / "b200.json")
    assert got == want
