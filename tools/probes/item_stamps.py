"""Per-item timeline of CTA 0 in K1v2 (EBIC_PHASE_TIMING=1, device path):
producer wait-for-free-stage / issue-done, consumer warp 0 wait-for-data /
walk-done, for one workload.  usage: python tools/probes/item_stamps.py [c5ss] [host] [rows=N]"""
import ctypes as C
import os
import sys
from pathlib import Path
import numpy as np
os.environ["EBIC_PHASE_TIMING"] = "1"
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import torch  # noqa: E402
import paper_1801_03039_b200 as eb  # noqa: E402
from paper_1801_03039_b200 import _lib  # noqa: E402
from golden_io import trace  # noqa: E402

t = trace(sys.argv[1] if len(sys.argv) > 1 else "c5ss")
host = "host" in sys.argv[2:]  # the host-buffer API (CTA-0 population pull)
rows = [int(a[5:]) for a in sys.argv[2:] if a.startswith("rows=")]  # rows=N: the first N rows only (a shard's size)
off, cols, _, _ = t.batches[-1]
with eb.Evaluator(t.matrix()[:rows[0]] if rows else t.matrix()) as ev:
    d_off = torch.from_numpy(off.astype(np.int64)).cuda()
    d_cols = torch.from_numpy(cols.view(np.int16)).cuda()
    P, L = len(off) - 1, int(off[-1])
    cnt = torch.zeros(P, dtype=torch.int64, device="cuda")
    fit = torch.zeros(P, dtype=torch.float64, device="cuda")
    for _ in range(4):
        if host:
            ev.evaluate_population(eb.CbfPopulation(off, cols), eb.FitnessParams(t.sigma), t.eps)
        else:
            _lib.check(_lib.lib.ebic_count_matches_device(ev.handle, d_off.data_ptr(), d_cols.data_ptr(), P, L,
                                                          t.eps, t.sigma, cnt.data_ptr(), fit.data_ptr(), None))
        torch.cuda.synchronize()
    st = np.zeros((4096, 8), dtype=np.uint64)
    n = C.c_size_t(0)
    _lib.check(_lib.lib.ebic_ctx_phase_times(ev.handle, st.ctypes.data_as(_lib.u64p), 4096, C.byref(n)))
    st = st.astype(np.int64)
    t0 = st[:n.value, 0].min()
    it = st[512:576]
    pr = st[600]
    print("CTA0 prologue: start->item tiles", (pr[0] - st[0, 0]) / 1e3, "barriers 1..5 at",
          [round((pr[k] - st[0, 0]) / 1e3, 2) for k in range(1, 6)], "(us from CTA 0 start)")
    pd = st[601]
    print("  phase D (thread 0): slots done", (pd[0] - st[0, 0]) / 1e3, "dummies done", (pd[1] - st[0, 0]) / 1e3,
          "after barrier 4a", (pd[2] - st[0, 0]) / 1e3)
    print("CTA0 prologue end", (st[0, 1] - t0) / 1e3, "walk end", (st[0, 2] - t0) / 1e3, "kernel end", (st[:n.value, 3].max() - t0) / 1e3)
    a = st[:n.value]
    q = lambda col: np.percentile((a[:, col] - t0) / 1e3, [0, 50, 100]).round(2).tolist()  # noqa: E731
    print("all CTAs (min/median/max us): start", q(0), "prologue end", q(1), "walk end", q(2),
          "reds done", q(4), "ticket", q(5), "end", q(3))
    order = np.argsort(a[:, 2])[::-1][:6]  # the latest walks (CTA G-1 also fixes up the first dirty row)
    print("latest walk ends (CTA: prologue end, walk end, us):",
          [(int(c), round((a[c, 1] - t0) / 1e3, 2), round((a[c, 2] - t0) / 1e3, 2)) for c in order])
    last = a[a[:, 7] >= t0]  # (rows of CTAs that were last in earlier launches keep stale stamps)
    if len(last):
        k = int(np.argmax(last[:, 7]))
        print("last CTA: enters final sum", round((last[k, 7] - t0) / 1e3, 2), "ends", round((last[k, 3] - t0) / 1e3, 2))
    print("item  prod_start  stage_free  issued   cons_wait  data_in  walk_done   (us from first CTA start)")
    for k in range(64):
        r = it[k]
        if r[3] == 0 and r[0] == 0:
            continue
        f = lambda x: f"{(x - t0) / 1e3:9.2f}" if x else "        -"  # noqa: E731
        print(f"{k:4d} {f(r[0])} {f(r[1])} {f(r[2])} {f(r[3])} {f(r[4])} {f(r[5])}")
