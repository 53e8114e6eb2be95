"""Phase stamps (EBIC_PHASE_TIMING=1) of the count kernel on the host path
(Evaluator.evaluate_population: CBF staged in-kernel from mapped memory) and on
the device path (ebic_count_matches_device), C4 by default."""
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

t = trace(sys.argv[1] if len(sys.argv) > 1 else "c4")


def summary(ev):
    st = np.zeros((4096, 8), dtype=np.uint64)
    n = C.c_size_t(0)
    _lib.check(_lib.lib.ebic_ctx_phase_times(ev.handle, st.ctypes.data_as(_lib.u64p), 4096, C.byref(n)))
    st = st[:n.value].astype(np.int64)
    t0 = st[:, 0].min()
    r = lambda k: (st[:, k] - t0) / 1e3  # noqa: E731
    fin = st[:, 7] > 0
    return {"start_spread": r(0).max(), "cta0_prologue_end": r(1)[0], "prologue_end_med": np.median(r(1)),
            "prologue_end_max": r(1).max(), "tiles_done_min": r(2).min(), "tiles_done_med": np.median(r(2)),
            "tiles_done_max": r(2).max(), "flushed_max": r(4).max(), "arrived_max": r(5).max(),
            "final_start": r(7)[fin].max() if fin.any() else None, "end_max": r(3).max()}


with eb.Evaluator(t.matrix()) as ev:
    params = eb.FitnessParams(t.sigma)
    for k in range(8):
        off, cols, _, _ = t.batches[k % len(t.batches)]
        ev.evaluate_population(eb.CbfPopulation(off, cols), params, t.eps)
    print("host path  :", {k: (round(float(v), 2) if v is not None else None) for k, v in summary(ev).items()})
    import torch
    off, cols, _, _ = t.batches[-1]
    d_off = torch.from_numpy(off.astype(np.int64)).cuda()
    d_cols = torch.from_numpy(cols.view(np.int16)).cuda()
    P, L = len(off) - 1, int(off[-1])
    cnt = torch.zeros(P, dtype=torch.int64, device="cuda")
    fit = torch.zeros(P, dtype=torch.float64, device="cuda")
    for _ in range(4):
        _lib.check(_lib.lib.ebic_count_matches_device(ev.handle, d_off.data_ptr(), d_cols.data_ptr(), P, L,
                                                      t.eps, t.sigma, cnt.data_ptr(), fit.data_ptr(), None))
        torch.cuda.synchronize()
    print("device path:", {k: (round(float(v), 2) if v is not None else None) for k, v in summary(ev).items()})
