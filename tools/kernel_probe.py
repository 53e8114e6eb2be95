#!/usr/bin/env python
"""Count-kernel timing under EBIC_* knob variants (GPU box; not a bench line).

usage: python tools/kernel_probe.py WORKLOAD [VARIANT ...]
  WORKLOAD  a trace name (c4, c5, c4ss, c5ss, ...); steady-state traces replay
            their batches of generation >= 250 (all batches otherwise)
  VARIANT   "" (defaults) or space-separated K=V knobs, e.g. "EBIC_DEBUG_MODE=1"

Per variant: a fresh context (knobs are read at creation), parity of counts
and fitness against the reference trace (skipped for EBIC_DEBUG_MODE != 0),
then per-launch CUDA-event times with L2 evicted before every launch (as
bench.py's `value`), the same without the eviction (warm L2), and back to
back without eviction.  Prints one JSON line
per variant."""
import json
import os
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

    name = sys.argv[1]
    variants = sys.argv[2:] or [""]
    if name.startswith("synth:"):
        # synth:ROWS,COLS,P,LEN -- N(0,1) matrix, P random series of LEN columns
        # (no reference counts: parity is not checked)
        R, Cc, P, L = map(int, name[6:].split(","))
        rng = np.random.default_rng(11)
        values = rng.standard_normal((R, Cc))
        cols = np.concatenate([rng.choice(Cc, size=L, replace=False) for _ in range(P)]).astype(np.uint16)
        off = np.arange(P + 1, dtype=np.uint64) * L

        class T:
            eps, sigma = 1e-9, max(4, -(-R // 50))
        t = T()
        batches = [(off, cols, None, None)]
    else:
        t = trace(name)
        batches = t.steady_batches() if name.endswith("ss") else t.batches
        values = t.matrix()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    bs = []
    for off, cols, counts, fit in batches:
        bs.append(dict(P=len(off) - 1, L=int(off[-1]), want=(counts, fit),
                       off=torch.from_numpy(off.astype(np.int64)).to(dev),
                       cols=torch.from_numpy(cols.view(np.int16)).to(dev),
                       counts=torch.zeros(len(off) - 1, dtype=torch.int64, device=dev),
                       fit=torch.zeros(len(off) - 1, dtype=torch.float64, device=dev)))
    flush = torch.zeros(128 << 20, dtype=torch.float32, device=dev)
    sink = torch.zeros(1, dtype=torch.float32, device=dev)
    base_env = dict(os.environ)
    for var in variants:
        os.environ.clear()
        os.environ.update(base_env)
        for kv in var.split():
            k, v = kv.split("=", 1)
            os.environ[k] = v
        ev = eb.Evaluator(values, devices=[0])

        def step(b):
            _lib.check(_lib.lib.ebic_count_matches_device(
                ev.handle, b["off"].data_ptr(), b["cols"].data_ptr(), b["P"], b["L"], t.eps, t.sigma,
                b["counts"].data_ptr(), b["fit"].data_ptr(), stream.cuda_stream))

        for b in bs:
            step(b)
        torch.cuda.synchronize()
        parity = None
        if os.environ.get("EBIC_DEBUG_MODE", "0") == "0" and bs[0]["want"][0] is not None:
            parity = True
            for b in bs:
                step(b)
                torch.cuda.synchronize()
                c = b["counts"].cpu().numpy().astype(np.uint64)
                f = b["fit"].cpu().numpy()
                parity &= bool((c == b["want"][0]).all() and (f.view(np.uint64) == b["want"][1].view(np.uint64)).all())
        n = max(40, 4 * len(bs))
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for k in range(n):
            torch.sum(flush, dim=0, keepdim=True, out=sink)
            torch.cuda._sleep(100_000)
            evs[k][0].record(stream)
            step(bs[k % len(bs)])
            evs[k][1].record(stream)
        torch.cuda.synchronize()
        per = [a.elapsed_time(b) * 1e3 for a, b in evs]
        # same per-step events without the eviction: L2 keeps the code, the
        # CBF, the rank tiles and the stripes (the GA's own case between
        # generations); separates the cold-L2 cost from the launch floor
        for k in range(n):
            torch.cuda._sleep(100_000)
            evs[k][0].record(stream)
            step(bs[k % len(bs)])
            evs[k][1].record(stream)
        torch.cuda.synchronize()
        warm = [a.elapsed_time(b) * 1e3 for a, b in evs]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.sum(flush, dim=0, keepdim=True, out=sink)
        e0.record(stream)
        for k in range(n):
            step(bs[k % len(bs)])
        e1.record(stream)
        torch.cuda.synchronize()
        info = ev.info()
        series = float(np.mean([b["P"] for b in bs]))
        print(json.dumps({"workload": name, "variant": var, "parity": parity,
                          "us_evicted_mean": float(np.mean(per)), "us_evicted_min": float(np.min(per)),
                          "us_warm_mean": float(np.mean(warm)),
                          "us_back_to_back": e0.elapsed_time(e1) * 1e3 / n,
                          "mbic_per_s": series / float(np.mean(per)),
                          "rows_per_tile": info.rows_per_tile, "stages": info.stages,
                          "layout": info.layout, "warps": info.consumer_warps}), flush=True)
        ev.close()


if __name__ == "__main__":
    main()
