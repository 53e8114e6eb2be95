"""Per-CTA tile-phase end times of the count kernel (EBIC_PHASE_TIMING=1)."""
import ctypes as C
import os
import sys
from pathlib import Path
import numpy as np
os.environ["EBIC_PHASE_TIMING"] = "1"
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import paper_1801_03039_b200 as eb  # noqa: E402
from paper_1801_03039_b200 import _lib  # noqa: E402
from golden_io import trace  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
t = trace(name)
v = t.matrix()
with eb.Evaluator(v) as ev:
    off, cols, counts, fit = t.batches[1]
    pop = eb.CbfPopulation(off, cols)
    for _ in range(3):
        ev.count_matches(pop, t.eps)
    st = np.zeros((4096, 8), dtype=np.uint64)
    n = C.c_size_t(0)
    _lib.check(_lib.lib.ebic_ctx_phase_times(ev.handle, st.ctypes.data_as(_lib.u64p), 4096, C.byref(n)))
    st = st[:n.value].astype(np.int64)
    t0 = st[:, 0].min()
    tiles = (st[:, 2] - t0) / 1e3
    pro = (st[:, 1] - st[:, 0]) / 1e3
    start = (st[:, 0] - t0) / 1e3
    print("ctas", n.value, "tiles_done min/median/max", tiles.min(), np.median(tiles), tiles.max())
    order = np.argsort(tiles)
    print("slowest 12 CTAs (idx, tiles_done, start, prologue):")
    for i in order[-12:]:
        print(int(i), round(float(tiles[i]), 2), round(float(start[i]), 2), round(float(pro[i]), 2))
    print("fastest 6:", [(int(i), round(float(tiles[i]), 2)) for i in order[:6]])
    G = n.value
    print("mean tiles_done by CTA index decile:", [round(float(tiles[k * G // 10:(k + 1) * G // 10].mean()), 2) for k in range(10)])
