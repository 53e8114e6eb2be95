"""Host-side cost breakdown of one e2e evaluate_population call (GPU box)."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import torch  # noqa: E402
import paper_1801_03039_b200 as eb  # noqa: E402
from paper_1801_03039_b200 import _lib  # noqa: E402
from golden_io import trace  # noqa: E402

t = trace("c4")
v = t.matrix()
ev = eb.Evaluator(v)
pops = [eb.CbfPopulation(off, cols) for off, cols, _, _ in t.batches]
params = eb.FitnessParams(t.sigma)


def timeit(name, fn, n=300):
    for _ in range(20):
        fn(0)
    ts = []
    for k in range(n):
        a = time.perf_counter()
        fn(k)
        ts.append(time.perf_counter() - a)
    ts = np.array(ts) * 1e6
    print(f"{name:<55} median {np.median(ts):8.2f} us  p10 {np.percentile(ts, 10):8.2f}")


timeit("Evaluator.evaluate_population (public API)", lambda k: ev.evaluate_population(pops[k % 8], params, t.eps))
offs = [np.ascontiguousarray(p.offsets, dtype=np.uint64) for p in pops]
cols = [np.ascontiguousarray(p.col_indices, dtype=np.uint16) for p in pops]
outs = [np.zeros(p.size(), np.float64) for p in pops]
cnts = [np.zeros(p.size(), np.uint64) for p in pops]
args = [(o.ctypes.data_as(_lib.szp), c.ctypes.data_as(_lib.u16p), len(o) - 1, f.ctypes.data_as(_lib.f64p), n.ctypes.data_as(_lib.u64p)) for o, c, f, n in zip(offs, cols, outs, cnts)]
L = _lib.lib
h = ev.handle


def raw(k):
    a = args[k % 8]
    L.ebic_evaluate_population(h, a[0], a[1], a[2], t.sigma, t.eps, a[4], a[3])


timeit("raw ctypes ebic_evaluate_population (pre-converted)", raw)
one = eb.encode_population([[0, 1]])
o1 = np.ascontiguousarray(one.offsets); c1 = np.ascontiguousarray(one.col_indices)
f1 = np.zeros(1); n1 = np.zeros(1, np.uint64)
timeit("raw ctypes, P=1", lambda k: L.ebic_evaluate_population(h, o1.ctypes.data_as(_lib.szp), c1.ctypes.data_as(_lib.u16p), 1, t.sigma, t.eps, n1.ctypes.data_as(_lib.u64p), f1.ctypes.data_as(_lib.f64p)))
timeit("ctypes no-op (ebic_abi_version)", lambda k: L.ebic_abi_version())
d_off = [torch.from_numpy(o.astype(np.int64)).cuda() for o in offs]
d_cols = [torch.from_numpy(c.view(np.int16)).cuda() for c in cols]
d_cnt = torch.zeros(700, dtype=torch.int64, device="cuda")
d_fit = torch.zeros(700, dtype=torch.float64, device="cuda")


def dev(k):
    i = k % 8
    L.ebic_count_matches_device(h, d_off[i].data_ptr(), d_cols[i].data_ptr(), len(offs[i]) - 1, int(offs[i][-1]), t.eps, t.sigma, d_cnt.data_ptr(), d_fit.data_ptr(), None)
    torch.cuda.synchronize()


timeit("device API launch + synchronize (L2 warm)", dev)
