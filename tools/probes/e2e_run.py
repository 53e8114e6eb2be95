"""Runs the C++ e2e driver on a trace under several env settings (diagnostics).
usage: python tools/probes/e2e_run.py c4 "EBIC_X=1" "EBIC_X=0 EBIC_Y=2" ..."""
import json, os, subprocess, sys, tempfile
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from golden_io import trace
t = trace(sys.argv[1] if len(sys.argv) > 1 else "c4")
exe = ROOT / "paper_1801_03039_b200" / "ebic_e2e_driver"
with tempfile.TemporaryDirectory() as td:
    path = Path(td) / "b.bin"
    with open(path, "wb") as f:
        for off, cols, counts, fit in (t.steady_batches() if sys.argv[1].endswith("ss") else t.batches):
            f.write(np.uint64(len(off) - 1).tobytes()); f.write(off.astype(np.uint64).tobytes())
            f.write(cols.astype(np.uint16).tobytes()); f.write(counts.astype(np.uint64).tobytes())
            f.write(fit.astype(np.float64).tobytes())
    s = t.spec
    for envs in [a.split() for a in sys.argv[2:]] or [[]]:
        env = dict(os.environ); env.update(e.split("=") for e in envs)
        cmd = [str(exe), str(path), str(s["rows"]), str(s["cols"]), str(len(s["blocks"])), str(s["blocks"][0][0]),
               str(s["blocks"][0][1]), str(s["pattern"]), str(s["overlap"]), repr(float(s["noise"])), str(s["seed"]),
               repr(float(t.eps)), str(t.sigma), "1000", "5"]
        r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=300)
        print(envs, r.stdout.strip()[-600:], r.stderr.strip()[-300:], flush=True)
