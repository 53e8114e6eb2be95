#!/usr/bin/env python
"""Per-shard count-kernel cost of the config-5 row sharding (GPU box; not a
bench line).

usage: python tools/shard_probe.py [c5ss] [N ...]      (default N = 1 2 4 8)

For each N the 200,000 x 1000 matrix is split into N 64-row-aligned shards
exactly as ``RowShardedEvaluator`` / ``bench.py --gpus N`` split it; every
shard gets its own context (``ebic_ctx_create_shard``) on the one GPU here and
is timed alone, per launch, with CUDA events (L2 evicted before every launch,
and back to back), on the steady-state batches.  The shards' partial counts
are summed on the host and compared with the reference trace (bit-exact
row-sharded counts at every N).  What one GPU cannot show is the cross-GPU
exchange: the step at N GPUs is the slowest shard's launch plus the in-kernel
cross-rank sum."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    import torch
    import paper_1801_03039_b200 as eb
    from paper_1801_03039_b200 import _lib
    from golden_io import trace

    name = sys.argv[1] if len(sys.argv) > 1 else "c5ss"
    ns = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
    t = trace(name)
    batches = t.steady_batches() if name.endswith("ss") else t.batches
    values = t.matrix()
    R = values.shape[0]
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    bs = []
    for off, cols, counts, _ in batches:
        bs.append(dict(P=len(off) - 1, L=int(off[-1]), want=counts.astype(np.uint64),
                       off=torch.from_numpy(off.astype(np.int64)).to(dev),
                       cols=torch.from_numpy(cols.view(np.int16)).to(dev),
                       counts=torch.zeros(len(off) - 1, dtype=torch.int64, device=dev)))
    flush = torch.zeros(128 << 20, dtype=torch.float32, device=dev)
    sink = torch.zeros(1, dtype=torch.float32, device=dev)
    for n in ns:
        per = -(-R // n)
        per = -(-per // 64) * 64
        bounds = [(b, min(R, b + per)) for b in range(0, R, per)]
        sums = [np.zeros(b["P"], dtype=np.uint64) for b in bs]
        shard_us = []
        for lo, hi in bounds:
            ev = eb.Evaluator(values[lo:hi], devices=[0], shard=(lo, R))

            def step(b):
                _lib.check(_lib.lib.ebic_count_matches_device(
                    ev.handle, b["off"].data_ptr(), b["cols"].data_ptr(), b["P"], b["L"], t.eps, t.sigma,
                    b["counts"].data_ptr(), None, stream.cuda_stream))

            for i, b in enumerate(bs):
                step(b)
                torch.cuda.synchronize()
                sums[i] += b["counts"].cpu().numpy().astype(np.uint64)
            k = max(40, 4 * len(bs))
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
            for j in range(k):
                torch.sum(flush, dim=0, keepdim=True, out=sink)
                torch.cuda._sleep(100_000)
                evs[j][0].record(stream)
                step(bs[j % len(bs)])
                evs[j][1].record(stream)
            torch.cuda.synchronize()
            evicted = float(np.mean([a.elapsed_time(e) * 1e3 for a, e in evs]))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.sum(flush, dim=0, keepdim=True, out=sink)
            e0.record(stream)
            for j in range(k):
                step(bs[j % len(bs)])
            e1.record(stream)
            torch.cuda.synchronize()
            shard_us.append((hi - lo, evicted, e0.elapsed_time(e1) * 1e3 / k))
            ev.close()
        parity = all(bool((s == b["want"]).all()) for s, b in zip(sums, bs))
        worst = max(shard_us, key=lambda x: x[1])
        print(json.dumps({"workload": name, "n_shards": n, "rows_per_shard": bounds[0][1] - bounds[0][0],
                          "parity_summed_counts": parity,
                          "slowest_shard_us_evicted": round(worst[1], 2),
                          "slowest_shard_us_back_to_back": round(max(x[2] for x in shard_us), 2),
                          "per_shard": [[r, round(a, 2), round(b, 2)] for r, a, b in shard_us]}), flush=True)


if __name__ == "__main__":
    main()
