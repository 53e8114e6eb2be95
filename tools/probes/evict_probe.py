"""Count-kernel step time (C4, device path, CUDA events) after different
pre-step kernels: L2 evicted by a read with no / the count kernel's shared
memory, an empty kernel (L2 warm), nothing."""
import ctypes as C, sys
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import paper_1801_03039_b200 as eb
from paper_1801_03039_b200 import _lib
from golden_io import trace
lib = C.CDLL(str(ROOT / "tools/probes/libevict_probe.so"))
lib.evict.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_int, C.c_void_p]
lib.empty.argtypes = [C.c_void_p, C.c_void_p]
t = trace("c4"); ev = eb.Evaluator(t.matrix())
dev = torch.device("cuda"); st = torch.cuda.Stream(); sh = st.cuda_stream
bs = []
for off, cols, _, _ in t.batches:
    bs.append((torch.from_numpy(off.astype(np.int64)).to(dev), torch.from_numpy(cols.view(np.int16)).to(dev), len(off) - 1, int(off[-1])))
cnt = torch.zeros(2048, dtype=torch.int64, device=dev); fit = torch.zeros(2048, dtype=torch.float64, device=dev)
buf = torch.zeros(128 << 20, dtype=torch.float32, device=dev); sink = torch.zeros(1, device=dev)
def step(b):
    _lib.check(_lib.lib.ebic_count_matches_device(ev.handle, b[0].data_ptr(), b[1].data_ptr(), b[2], b[3], t.eps, t.sigma, cnt.data_ptr(), fit.data_ptr(), sh))
modes = {"evict_small_smem": lambda: lib.evict(buf.data_ptr(), buf.numel() * 4, sink.data_ptr(), 0, sh),
         "evict_big_smem": lambda: lib.evict(buf.data_ptr(), buf.numel() * 4, sink.data_ptr(), 1, sh),
         "empty_kernel": lambda: lib.empty(sink.data_ptr(), sh),
         "nothing": lambda: None}
with torch.cuda.stream(st):
    for name, pre in modes.items():
        for k in range(5): pre(); step(bs[k % len(bs)])
        torch.cuda.synchronize()
        tot = 0.0
        for k in range(400):
            pre()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st); step(bs[k % len(bs)]); e1.record(st)
            torch.cuda._sleep(50_000)
            e1.synchronize(); tot += e0.elapsed_time(e1)
        print(f"{name:18s} {1e3 * tot / 400:.2f} us/step", flush=True)
