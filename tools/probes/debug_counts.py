"""Count mismatches of the C3/C4 traces under several kernel configurations."""
import os
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import paper_1801_03039_b200 as eb  # noqa: E402
from golden_io import trace  # noqa: E402

for name in ["c3", "c4"]:
    t = trace(name)
    v = t.matrix()
    for cfg in [{}, {"EBIC_SCHED_STATIC": "1"}, {"EBIC_MAX_PARTS": "1"}, {"EBIC_MAX_PARTS": "2"}, {"EBIC_MAX_PARTS": "2", "EBIC_SCHED_STATIC": "1"}]:
        for k in ["EBIC_STAGES", "EBIC_GRID", "EBIC_NCW", "EBIC_LAYOUT_F64", "EBIC_SCHED_STATIC", "EBIC_MAX_PARTS"]:
            os.environ.pop(k, None)
        os.environ.update(cfg)
        with eb.Evaluator(v) as ev:
            off, cols, counts, fit = t.batches[1]
            c = ev.count_matches(eb.CbfPopulation(off, cols), t.eps)
            bad = np.nonzero(c != counts)[0]
            info = ev.info()
            print(name, cfg, "grid", info.grid, "stages", info.stages, "mismatch", len(bad),
                  "diff sum", int((c.astype(np.int64) - counts.astype(np.int64)).sum()),
                  "ex", [(int(i), int(c[i]), int(counts[i])) for i in bad[:4]], flush=True)
