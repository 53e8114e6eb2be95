"""TopRankList::update, reference vs drop-in, on recorded GA population streams.

Records the populations the reference GA hands to its top-rank list
(oracle Ref.run_population_trace: C1 for 300 generations, C4 for 30) and
replays them through oracle/_ref/toprank_time_ref (reference evolution.hpp)
and oracle/_ref/toprank_time_dropin (shadow evolution.hpp -> ebic_top_rank_update).
Both print mean us/update and a digest of the final list (must agree).
When tools/probes/build.sh has run, build_generation is timed on the same
streams too (reference vs shadow headers, digest of the children).
usage: python tools/toprank_compare.py > gpurun_out/toprank_compare.log
"""
import json
import os
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402

RUNS = {"c1": (500, 100, [(50, 10)] * 3, 1, 0.0, 300),
        "c4": (20000, 500, [(600, 20)] * 5, 2026, 1e-9, 30)}

ref = oracle.Ref()
with tempfile.TemporaryDirectory() as td:
    for name, (rows, cols, blocks, seed, eps, gens) in RUNS.items():
        m = ref.matrix(ref.generate(rows, cols, blocks, 0, 0, 0, 0.0, seed))
        path = Path(td) / f"{name}.bin"
        ref.run_population_trace(m, path, population=600, iterations=gens - 1, rng_seed=1, eps=eps,
                                 sigma=0, threads=os.cpu_count() or 1)
        out = {}
        for impl in ("ref", "dropin"):
            r = subprocess.run([str(oracle.HERE / "_ref" / f"toprank_time_{impl}"), str(path), "5"],
                               capture_output=True, text=True, check=True)
            out[impl] = json.loads(r.stdout)
        bg = {}
        for impl in ("ref", "dropin"):  # build_generation on the same stream (tools/probes/build.sh)
            exe = ROOT / "tools" / "probes" / f"build_gen_compare_{impl}"
            if exe.exists():
                r = subprocess.run([str(exe), str(path)], capture_output=True, text=True, check=True)
                bg[impl] = r.stdout.split()  # "build_generation us <t> digest <d>"
        if len(bg) == 2:
            print(json.dumps({"stream": name, "build_generation_reference_us": float(bg["ref"][2]),
                              "build_generation_dropin_us": float(bg["dropin"][2]),
                              "children_equal": bg["ref"][4] == bg["dropin"][4]}), flush=True)
        print(json.dumps({"stream": name, "updates": out["ref"]["updates"],
                          "reference_us_per_update": out["ref"]["us_per_update"],
                          "dropin_us_per_update": out["dropin"]["us_per_update"],
                          "speedup": round(out["ref"]["us_per_update"] / out["dropin"]["us_per_update"], 2),
                          "digests_equal": out["ref"]["digest"] == out["dropin"]["digest"]}), flush=True)
