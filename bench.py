#!/usr/bin/env python
"""Benchmark of the EBIC fitness-evaluation hot path on B200.

Metric (BASELINE.json): biclusters evaluated/sec (+ fitness-kernel GB/s vs
roofline).  A step is one generation's novel batch (P = 575 series, the
reference's `series_evaluated` unit, evolution.hpp:486,506) evaluated against
every row of the matrix: per-series match counts + Eq. 1 fitness
(fitness.hpp:100-143).

Workload (default, N=1): BASELINE config 4 -- the 20,000 x 500 synthetic
matrix (ebic::generate, 5 planted 600x20 trend blocks, seed 2026; regenerated
bit-identically by the product generator) and the novel batches of a real
reference GA run on it (tests/golden/trace_c4.npz, recorded through
RunHooks::on_evaluate), eps = 1e-9, sigma = default 400.

Arms
  (default)          the B200 path.  `value`: inputs resident in HBM, one count
                     kernel (fused fitness) per step, CUDA events on the launch
                     stream, L2 flushed between steps (outside the events).
                     `e2e`: the public API with host buffers
                     (Evaluator.evaluate_population -> ebic_evaluate_population:
                     pinned H2D of the CBF, kernel, D2H of counts + fitness).
  --impl reference   the reference's own CPU implementation (oracle/_ref, the
                     unmodified headers compiled here) on all host threads.

Multi-GPU: `bench.py --gpus N` re-executes itself under torch.distributed.run
as N ranks when WORLD_SIZE is unset (the driver may also launch it with
torchrun itself); a run whose WORLD_SIZE differs from --gpus is refused, and
NCCL ranks need N visible GPUs (--backend gloo lets ranks share one GPU, for
tests).  One process per GPU: rows are sharded (64-row aligned);
each rank counts its shard.  `e2e` (host buffers, the public C ABI) sums
across ranks inside the count kernels: every rank's final CTA adds into rank
0's accumulator through CUDA IPC peer memory and the last one writes counts +
Eq. 1 into a shared-memory block all ranks read.  `value` (inputs resident in
HBM) uses the same in-kernel sum with a host wait per step (--reduce kernel,
default: one launch per step and no collective), or all-reduces the counts
with NCCL and runs the Eq. 1 kernel on them (--reduce collective; also the
fallback when CUDA IPC is unavailable).  Time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

METRIC = "biclusters evaluated/sec"
UNIT = "biclusters/s"

WORKLOADS = {
    # name: (trace fixture, first generation replayed).  C4 / C5 replay the
    # steady state of long reference runs (tests/golden/make_golden.py STEADY:
    # C4 generations 250..5000 of 5000, every 250th; C5 generations 100..1000
    # of 1000, every 100th); "c4early" / "c5early" the first generations.
    "c4": ("c4ss", 250),
    "c5": ("c5ss", 50),
    "c4early": ("c4", 0),
    "c5early": ("c5", 0),
    "c3": ("c3", 0),
    "c1": ("c1e", 0),
}


def load_workload(name: str):
    import copy
    from golden_io import trace
    tname, min_gen = WORKLOADS[name]
    t = copy.copy(trace(tname))
    if min_gen:
        keep = [g >= min_gen for g in t.generations]
        t.batches = [b for b, k in zip(t.batches, keep) if k]
        t.generations = [g for g, k in zip(t.generations, keep) if k]
    return t


def hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int = 0):
        self.dev = device_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = [r.split(",") for r in out.strip().splitlines() if r.strip()]
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                smax.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for i, n in enumerate(names):
                if len(r) > 4 + i and "Active" in r[4 + i] and "Not" not in r[4 + i]:
                    reasons.add(n)
        busy = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# bytes per matrix cell of the layout the count kernel streams (ebic_ctx_info.layout)
# (4, 5: one plane packed three rows per 32-bit word, 128 B per 96 rows;
#  6, 7: five rows per 64-bit word, 128 B per 80 rows)
LAYOUT_CELL_BYTES = {0: 8, 1: 2, 2: 4, 3: 2, 4: 4 / 3, 5: 4 / 3, 6: 1.6, 7: 1.6}
LAYOUT_NAMES = {0: "fp64", 1: "rank16x1", 2: "rank16x2", 3: "rank16x1c", 4: "rank10x3", 5: "rank10x3c",
                6: "rank12x5", 7: "rank12x5c"}


def algorithmic_bytes(rows: int, off: np.ndarray, cols: np.ndarray, cell_bytes: int) -> int:
    """rows x U x b_elem (cells of the U distinct columns the
    launch references, at the element width of the layout actually streamed:
    8 for fp64, 4 for the two-plane exact rank layout, 2 for one plane)
    + CBF in + counts/fitness out."""
    P = len(off) - 1
    U = len(np.unique(cols))
    return round(rows * U * cell_bytes) + (P + 1) * 8 + len(cols) * 2 + P * 8 * 2


# ---------------------------------------------------------------------------
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference(t, values, batches, steps, warmup, budget_s=60.0, threads=None, single_budget_s=None):
    """The reference CPU implementation on this host (oracle/_ref when built,
    else the C restatement).  Each step evaluates a bounded sample of a batch
    (a prefix of its series) so the whole run stays within ~budget_s.
    SURVEY.md §8(d): timed with T = nproc threads (`value`) and with T = 1
    (`value_1t`, a smaller sample), after >= 2 s of multi-threaded warm-up."""
    import oracle
    threads = threads or os.cpu_count() or 1
    if oracle.REF_LIB.exists():
        ref = oracle.Ref()
        m = ref.matrix(values)
        kind = "reference"

        def run(off, cols, workers):
            return ref.evaluate_population(m, off, cols, t.sigma, t.eps, workers=workers)
    else:
        port = oracle.Port()
        kind, threads = "port", 1

        def run(off, cols, workers):
            return port.evaluate_population(values, off, cols, t.sigma, t.eps)[1]

    # Warm-up: >= 2 s of multi-threaded work (cold vCPUs).
    t0 = time.perf_counter()
    full = []
    while time.perf_counter() - t0 < 2.0 or len(full) < max(1, warmup):
        off, cols, _, _ = batches[len(full) % len(batches)]
        a = time.perf_counter()
        run(off, cols, threads)
        full.append((time.perf_counter() - a) / (len(off) - 1))
    per_series = min(full)
    P = len(batches[0][0]) - 1

    def timed(workers, budget, per):
        sample = int(max(1, min(P, budget / max(steps, 1) / per)))
        done = 0
        a = time.perf_counter()
        for k in range(steps):
            off, cols, _, _ = batches[k % len(batches)]
            n = min(sample, len(off) - 1)
            sub_off = off[:n + 1]
            run(sub_off, cols[:int(sub_off[-1])], workers)
            done += n
        return done / (time.perf_counter() - a), sample

    value, sample = timed(threads, budget_s, per_series)
    out = {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
           "sample": f"{steps} steps x first {sample} of {P} series of a {t.name.upper()} GA batch "
                     f"(all {values.shape[0]} rows, eps={t.eps}); {threads} threads",
           "cpu_model": cpu_model(), "nproc": os.cpu_count()}
    if single_budget_s and threads > 1:
        # one thread is ~threads x slower per series: scale the estimate
        v1, s1 = timed(1, single_budget_s, per_series * threads)
        out["value_1t"] = v1
        out["sample_1t"] = f"{steps} steps x first {s1} series, 1 thread"
    return out


# ---------------------------------------------------------------------------
def run_reference_arm(args):
    """The reference's own CPU implementation (oracle/_ref) on all host
    threads, on the same workload.  Nothing from the product package is
    loaded: the input matrix comes from the reference's `ebic::generate`."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    t = load_workload(args.workload)
    values = t.matrix_reference()
    cb = cpu_reference(t, values, t.batches, args.steps, args.warmup,
                       single_budget_s=min(20.0, args.cpu_budget))
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": None, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(t, args, args.gpus, args.gpus),
        "cpu_baseline": cb,
        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(t, args, world=1, devices=1):
    s = t.spec
    gens = list(getattr(t, "generations", []))
    return {"workload": f"{args.workload}: synthetic {s['rows']}x{s['cols']} "
                        f"({len(s['blocks'])} planted {s['blocks'][0][0]}x{s['blocks'][0][1]} trend blocks, "
                        f"seed {s['seed']}), reference GA novel batches (population 600)"
                        + (f", generations {gens[0]}..{gens[-1]} of a {t.iterations}-generation run"
                           if gens else ""),
            "rows": s["rows"], "cols": s["cols"],
            "series_per_step": round(float(np.mean([len(b[0]) - 1 for b in t.batches])), 1),
            "eps": t.eps, "sigma": t.sigma, "l2": "evicted between timed steps (512 MB read, outside the timed events)",
            "parallelism": f"rows sharded over {world} rank(s) on {devices} GPU(s)"
                           + ("" if world == 1 and not args.force_sharded else
                              ("; value: cross-rank sum inside the count kernels (CUDA IPC peer memory)"
                               if args.reduce == "kernel" else "; value: NCCL all-reduce of counts")
                              + "; e2e: cross-rank sum inside the count kernels")}


# ---------------------------------------------------------------------------
def large_roofline(args, peak, evict, sharded=False, world=1, rank=0, backend="nccl"):
    """BASELINE config 5 (200,000 x 1000, the scaling-sweep matrix).

    * Roofline of the count kernel (one GPU): its tile (400 MB in the rank
      layout) exceeds the 126 MB L2, so back-to-back launches between one
      event pair are HBM-cold and the per-launch overhead is amortised.
      Reported beside the headline C4 line (where one step is ~10 us of HBM
      time plus a ~5.5 us event/launch floor).
    * `row_sharded`: the config-5 sweep itself -- rows sharded over the ranks
      (1 at N=1), every step one count launch per rank plus, at N>1, the NCCL
      all-reduce of the counts and the Eq. 1 kernel; per-step CUDA events with
      L2 evicted before each step (a shard of 200,000/N rows fits L2 at N=8),
      max over ranks.  Same measurement at every N, so the driver's N-sweep
      of this key is the config-5 scaling curve."""
    import torch
    import torch.distributed as dist
    import paper_1801_03039_b200 as eb
    from paper_1801_03039_b200 import _lib
    t = load_workload("c5")
    values = t.matrix()
    R = values.shape[0]
    dev = torch.device("cuda", torch.cuda.current_device())
    lo, hi = eb.shard_range(R, world, rank) if sharded else (0, R)
    if sharded:
        ev = eb.Evaluator(values[lo:hi], devices=[dev.index], shard=(lo, R))
    else:
        ev = eb.Evaluator(values, devices=[dev.index])
    del values
    stream = torch.cuda.current_stream(dev)
    bs = []
    for off, cols, counts, fit in t.batches:
        bs.append(dict(P=len(off) - 1, L=int(off[-1]), off_np=off, cols_np=cols, want=counts,
                       off=torch.from_numpy(off.astype(np.int64)).to(dev),
                       cols=torch.from_numpy(cols.view(np.int16)).to(dev),
                       counts=torch.zeros(len(off) - 1, dtype=torch.int64, device=dev),
                       fit=torch.zeros(len(off) - 1, dtype=torch.float64, device=dev)))

    def step(b):
        if sharded:
            _lib.check(_lib.lib.ebic_count_matches_device(
                ev.handle, b["off"].data_ptr(), b["cols"].data_ptr(), b["P"], b["L"], t.eps, t.sigma,
                b["counts"].data_ptr(), None, stream.cuda_stream))
            dist.all_reduce(b["counts"], op=dist.ReduceOp.SUM)
            _lib.check(_lib.lib.ebic_fitness_device(
                ev.handle, b["counts"].data_ptr(), b["off"].data_ptr(), b["P"], t.sigma,
                b["fit"].data_ptr(), stream.cuda_stream))
        else:
            _lib.check(_lib.lib.ebic_count_matches_device(
                ev.handle, b["off"].data_ptr(), b["cols"].data_ptr(), b["P"], b["L"], t.eps, t.sigma,
                b["counts"].data_ptr(), b["fit"].data_ptr(), stream.cuda_stream))

    for k in range(4):
        step(bs[k % len(bs)])
    torch.cuda.synchronize()
    for b, (_, _, _, want_fit) in zip(bs, t.batches):
        step(b)
        torch.cuda.synchronize()
        assert (b["counts"].cpu().numpy().astype(np.uint64) == b["want"]).all(), "C5 count mismatch"
        assert (b["fit"].cpu().numpy().view(np.uint64) == want_fit.view(np.uint64)).all(), "C5 fitness mismatch"
    layout = ev.info().layout

    # row-sharded sweep measurement (every N)
    n_sh = max(20, min(args.steps // 10, 100))
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_sh)]
    if sharded:
        dist.barrier()
    torch.cuda.synchronize()
    series_sh = 0
    for k in range(n_sh):
        b = bs[k % len(bs)]
        evict()
        torch.cuda._sleep(100_000)
        evs[k][0].record(stream)
        step(b)
        evs[k][1].record(stream)
        series_sh += b["P"]
    torch.cuda.synchronize()
    sh_ms = float(sum(e0.elapsed_time(e1) for e0, e1 in evs))
    if sharded:
        tt = torch.tensor([sh_ms], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        sh_ms = float(tt.item())
    row_sharded = {"value": series_sh / (sh_ms / 1e3), "unit": UNIT, "n_gpus": world,
                   "us_per_step": sh_ms * 1e3 / n_sh, "steps": n_sh, "rows_per_gpu": hi - lo,
                   "reduce": (f"{backend} all-reduce of the counts + Eq. 1 kernel" if sharded
                              else "none (1 GPU)"),
                   "timing": "per-step CUDA events, L2 evicted before each step, max over ranks",
                   "parity": "counts and fitness bit-exact vs the reference trace on every batch"}
    if sharded:
        ev.close()
        return {"workload": C5_DESC, "row_sharded": row_sharded}

    nbytes = 0
    steps = max(20, min(args.steps // 20, 200))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for k in range(steps):
        b = bs[k % len(bs)]
        step(b)
        nbytes += algorithmic_bytes(R, b["off_np"], b["cols_np"], LAYOUT_CELL_BYTES[layout])
    e1.record(stream)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / steps
    series = sum(bs[k % len(bs)]["P"] for k in range(steps))
    achieved = nbytes / steps / (us / 1e6) / 1e9
    # Bytes the kernel stages per launch: K1v2 at this size copies only the
    # launch's referenced columns (= the algorithmic matrix bytes); the v1
    # kernel (EBIC_KERNEL=1) stages whole row tiles.
    staged = (nbytes / steps if os.environ.get("EBIC_KERNEL", "2") != "1"
              else R * ev.n_cols * LAYOUT_CELL_BYTES[layout])
    ev.close()
    return {"workload": C5_DESC, "bound": "hbm", "achieved": achieved, "peak": peak,
            "unit": "GB/s", "frac": achieved / peak, "avg_launch_us": us,
            "algorithmic_bytes_per_launch": nbytes / steps, "layout": LAYOUT_NAMES[layout],
            "staged_bytes_per_launch": staged,
            "staged_GBps": staged / (us / 1e6) / 1e9, "staged_frac": staged / (us / 1e6) / 1e9 / peak,
            "biclusters_per_s": series / (us * steps / 1e6), "steps": steps,
            "timing": "back-to-back launches between one CUDA event pair (inputs > L2)",
            "row_sharded": row_sharded}


C5_DESC = ("c5: synthetic 200000x1000 (5 planted 6000x30 trend blocks, seed 2027), reference GA "
           "batches of generations 100..1000 (every 100th) of a 1000-generation run")


def run_e2e_driver(t, args):
    """Runs paper_1801_03039_b200/ebic_e2e_driver on the workload's batches."""
    import tempfile
    exe = ROOT / "paper_1801_03039_b200" / "ebic_e2e_driver"
    if not exe.exists():
        return None
    with tempfile.TemporaryDirectory() as td:
        path = Path(td) / "batches.bin"
        with open(path, "wb") as f:
            for off, cols, counts, fit in t.batches:
                f.write(np.uint64(len(off) - 1).tobytes())
                f.write(off.astype(np.uint64).tobytes())
                f.write(cols.astype(np.uint16).tobytes())
                f.write(counts.astype(np.uint64).tobytes())
                f.write(fit.astype(np.float64).tobytes())
        s = t.spec
        cmd = [str(exe), str(path), str(s["rows"]), str(s["cols"]), str(len(s["blocks"])),
               str(s["blocks"][0][0]), str(s["blocks"][0][1]), str(s["pattern"]), str(s["overlap"]),
               repr(float(s["noise"])), str(s["seed"]), repr(float(t.eps)), str(t.sigma),
               str(args.steps), str(max(args.warmup, 3))]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    if r.returncode != 0:
        raise RuntimeError(f"e2e driver failed ({r.returncode}): {r.stderr.strip()[-400:]}")
    return json.loads(r.stdout.strip().splitlines()[-1])


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_1801_03039_b200 as eb
    from paper_1801_03039_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    n_visible = torch.cuda.device_count()
    if world != args.gpus:
        # a line whose rank count differs from --gpus would mislabel the run
        print(f"[bench] refusing to run: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.backend == "nccl" and world > n_visible:
        print(f"[bench] refusing to run: {world} NCCL ranks need {world} GPUs, {n_visible} visible "
              f"(--backend gloo lets ranks share a GPU)", file=sys.stderr)
        sys.exit(2)
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, n_visible)
    n_devices = min(world, max(1, n_visible))
    sharded = world > 1 or args.force_sharded
    if sharded:
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        # communicator size and transport (NVLink / NVLS) in the log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if args.backend == "nccl":
            dist.init_process_group("nccl", rank=rank, world_size=world,
                                    device_id=torch.device("cuda", local))
        else:  # several ranks on one GPU (tests of the kernel-side reduction)
            dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    t = load_workload(args.workload)
    values = t.matrix()
    R = values.shape[0]
    lo, hi = eb.shard_range(R, world, rank)
    if sharded:
        ev = eb.Evaluator(values[lo:hi], devices=[local], shard=(lo, R))
    else:
        ev = eb.Evaluator(values, devices=[local])

    # A dedicated stream: the kernels, the collectives and the timing events
    # all run on it (events only see the stream they are recorded on).
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    st = stream.cuda_stream
    # Device-resident inputs: every batch's CBF in HBM.
    dev_batches = []
    for off, cols, counts, fit in t.batches:
        dev_batches.append(dict(
            P=len(off) - 1, L=int(off[-1]),
            off=torch.from_numpy(off.astype(np.int64)).to(dev),
            cols=torch.from_numpy(cols.view(np.int16)).to(dev),
            counts=torch.zeros(len(off) - 1, dtype=torch.int64, device=dev),
            fit=torch.zeros(len(off) - 1, dtype=torch.float64, device=dev),
            h_counts=np.zeros(len(off) - 1, dtype=np.uint64),
            h_fit=np.zeros(len(off) - 1, dtype=np.float64),
            want=(counts, fit)))
    # L2 eviction between timed steps by READING 512 MB (4x L2): leaves L2 full
    # of clean lines, so the timed kernel does not pay for write-backs that a
    # write-based flush would leave behind.
    flush = torch.zeros(128 << 20, dtype=torch.float32, device=dev)
    flush_sink = torch.zeros(1, dtype=torch.float32, device=dev)

    def evict_l2():
        torch.sum(flush, dim=0, keepdim=True, out=flush_sink)

    # Cross-rank reduction inside the count kernels (ebic_xgroup_*): set up
    # once, torch.distributed only broadcasts the IPC handle.  The host path
    # (e2e) always uses it; the device-resident path (`value`) uses it with
    # --reduce kernel, else an NCCL all-reduce that pipelines without host syncs.
    import ctypes as C
    xgroup = None
    if sharded:
        import uuid
        handle = (C.c_ubyte * 64)()
        name = f"/ebic_bench_{os.getpid()}_{uuid.uuid4().hex[:8]}"
        ok = 1
        if rank == 0:
            ok = int(_lib.lib.ebic_xgroup_create(ev.handle, 2048, name.encode(), handle) == 0)
        obj = [bytes(handle), name, ok]
        dist.broadcast_object_list(obj, src=0)
        xgroup = _lib.vp()
        if obj[2]:
            ok = int(_lib.lib.ebic_xgroup_join(ev.handle, (C.c_ubyte * 64).from_buffer_copy(obj[0]),
                                               obj[1].encode(), world, 2048, C.byref(xgroup)) == 0)
        else:
            ok = 0
        # every rank must agree (IPC may be unavailable in a container)
        agree = torch.tensor([ok], dtype=torch.int32, device=dev if args.backend == "nccl" else "cpu")
        dist.all_reduce(agree, op=dist.ReduceOp.MIN)
        if not int(agree.item()):
            if ok:
                _lib.check(_lib.lib.ebic_xgroup_destroy(xgroup))
            print(f"[bench] rank {rank}: in-kernel cross-rank sum unavailable "
                  f"({_lib.lib.ebic_last_error().decode()}); e2e not measured", file=sys.stderr)
            xgroup = None
            if args.reduce == "kernel":
                args.reduce = "collective"
        dist.barrier()
    xg = xgroup if args.reduce == "kernel" else None
    xseq = [0]

    def step(b):
        if xg is not None:
            xseq[0] += 1
            _lib.check(_lib.lib.ebic_xgroup_count(
                xg, b["off"].data_ptr(), b["cols"].data_ptr(), b["P"], b["L"], t.eps, t.sigma, 1,
                xseq[0], st))
            _lib.check(_lib.lib.ebic_xgroup_wait(
                xg, xseq[0], b["P"], b["h_counts"].ctypes.data_as(_lib.u64p),
                b["h_fit"].ctypes.data_as(_lib.f64p)))
        elif sharded:
            _lib.check(_lib.lib.ebic_count_matches_device(
                ev.handle, b["off"].data_ptr(), b["cols"].data_ptr(), b["P"], b["L"], t.eps,
                t.sigma, b["counts"].data_ptr(), None, st))
            dist.all_reduce(b["counts"], op=dist.ReduceOp.SUM)
            _lib.check(_lib.lib.ebic_fitness_device(
                ev.handle, b["counts"].data_ptr(), b["off"].data_ptr(), b["P"], t.sigma,
                b["fit"].data_ptr(), st))
        else:
            _lib.check(_lib.lib.ebic_count_matches_device(
                ev.handle, b["off"].data_ptr(), b["cols"].data_ptr(), b["P"], b["L"], t.eps,
                t.sigma, b["counts"].data_ptr(), b["fit"].data_ptr(), st))

    launches_per_step = 2 if (sharded and xg is None) else 1

    # warm-up + correctness gate on every batch (bit-exact vs the reference trace)
    for k in range(max(args.warmup, len(dev_batches))):
        step(dev_batches[k % len(dev_batches)])
    torch.cuda.synchronize()
    layout = ev.info().layout
    for b, (off, cols, _, _) in zip(dev_batches, t.batches):
        b["bytes"] = algorithmic_bytes(hi - lo, off, cols, LAYOUT_CELL_BYTES[layout])
    for b in dev_batches:
        step(b)
        torch.cuda.synchronize()
        if xg is not None:
            c, f = b["h_counts"].copy(), b["h_fit"].copy()
        else:
            c = b["counts"].cpu().numpy().astype(np.uint64)
            f = b["fit"].cpu().numpy()
        assert (c == b["want"][0]).all(), "count mismatch vs reference"
        assert (f.view(np.uint64) == b["want"][1].view(np.uint64)).all(), "fitness mismatch"

    # ---- timed: device-resident inputs ----
    clocks = ClockSampler(local)
    if rank == 0:
        clocks.start()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if sharded:
        dist.barrier()
    torch.cuda.synchronize()
    series = 0
    nbytes = 0
    for k in range(args.steps):
        b = dev_batches[k % len(dev_batches)]
        evict_l2()                          # evict L2 (outside the events)
        torch.cuda._sleep(100_000)          # keep the queue ahead of the host launch path
        starts[k].record(stream)
        step(b)
        ends[k].record(stream)
        series += b["P"]
        nbytes += b["bytes"]
    torch.cuda.synchronize()
    if sharded:
        dist.barrier()
    times = [s.elapsed_time(e) for s, e in zip(starts, ends)]  # ms
    total_ms = float(sum(times))
    clk = clocks.stop() if rank == 0 else None
    if sharded:
        tt = torch.tensor([total_ms], dtype=torch.float64,
                          device=dev if args.backend == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    value = series / (total_ms / 1e3)

    # Diagnostic: the same launches back to back between one event pair (no
    # eviction between them; the 40 MB rank tile stays L2-resident): launch
    # gaps + L2-warm kernel time.  Not the reported value.
    b2b_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    evict_l2()
    torch.cuda._sleep(100_000)
    b2b_ev[0].record(stream)
    for k in range(50):
        step(dev_batches[k % len(dev_batches)])
    b2b_ev[1].record(stream)
    torch.cuda.synchronize()
    b2b_us = b2b_ev[0].elapsed_time(b2b_ev[1]) * 1e3 / 50

    phases = None
    if os.environ.get("EBIC_PHASE_TIMING"):
        import ctypes as C
        stamps = np.zeros((4096, 8), dtype=np.uint64)
        nc = C.c_size_t(0)
        _lib.check(_lib.lib.ebic_ctx_phase_times(ev.handle, stamps.ctypes.data_as(_lib.u64p), 4096,
                                                 C.byref(nc)))
        st_ = stamps[:nc.value].astype(np.int64)
        t0 = st_[:, 0].min()
        rel = lambda k: (st_[:, k] - t0) / 1e3  # noqa: E731
        phases = {"prologue_us": float(np.median(st_[:, 1] - st_[:, 0]) / 1e3),
                  "start_spread_us": float(rel(0).max()),
                  "tiles_done_us_min": float(rel(2).min()),
                  "tiles_done_us_max": float(rel(2).max()),
                  "partials_flushed_us_max": float(rel(4).max()),
                  "arrived_us_max": float(rel(5).max()),
                  "group_reduced_us_max": float(rel(6)[st_[:, 6] > 0].max()) if (st_[:, 6] > 0).any() else None,
                  "final_start_us": float(rel(7)[st_[:, 7] > 0].max()) if (st_[:, 7] > 0).any() else None,
                  "epilogue_end_us_max": float(rel(3).max())}

    # kernel-only timing for the roofline (single launch per step when unsharded)
    avg_launch_ms = total_ms / args.steps if not sharded else None
    peak, peak_src = hbm_peak()
    info = ev.info()

    # ---- BASELINE config 5: kernel roofline (1 GPU) and the row-sharded sweep
    # (every N).  Measured before the cross-rank e2e below. ----
    big = None
    if not args.no_large:
        big = large_roofline(args, peak, evict_l2, sharded=sharded, world=world, rank=rank,
                             backend=args.backend)

    # ---- e2e (headline): the public C ABI from a C++ caller -- the view of the
    # reference's GA loop through include/ebic/fitness.hpp -- host buffers,
    # pinned H2D of the CBF, the kernel, results back in host memory, L2
    # evicted between steps (paper_1801_03039_b200/csrc/e2e_driver.cu) ----
    e2e_cpp = None
    if not sharded:
        e2e_cpp = run_e2e_driver(t, args)
    # ---- e2e through the Python mirror (same C ABI call + ctypes marshalling) ----
    pops = [eb.CbfPopulation(off, cols) for off, cols, _, _ in t.batches]
    e2e_val = None
    h2d = d2h = 0
    if not sharded:
        params = eb.FitnessParams(t.sigma)
        for k in range(max(3, args.warmup)):
            ev.evaluate_population(pops[k % len(pops)], params, t.eps)
        el = 0.0
        n_e2e = 0
        for k in range(args.steps):
            pop = pops[k % len(pops)]
            evict_l2()
            torch.cuda.synchronize()
            a = time.perf_counter()
            ev.evaluate_population(pop, params, t.eps)  # returns host fitness (synchronous)
            el += time.perf_counter() - a
            n_e2e += pop.size()
            h2d += (pop.size() + 1) * 8 + len(pop.col_indices) * 2
            d2h += pop.size() * 16
        e2e_val = n_e2e / el
        h2d //= args.steps
        d2h //= args.steps

    # ---- e2e at N ranks: the host path through the in-kernel cross-rank sum
    # (ebic_xgroup_evaluate: host CBF staged in-kernel, every rank's count,
    # the last rank's kernel writes counts + fitness to shared host memory) ----
    def sharded_e2e():
        n_sh = 0
        el = 0.0
        host_pops = [(np.ascontiguousarray(off, dtype=np.uint64), np.ascontiguousarray(cols, dtype=np.uint16))
                     for off, cols, _, _ in t.batches]
        hc = np.zeros(2048, dtype=np.uint64)
        hf = np.zeros(2048, dtype=np.float64)

        def call(off, cols):
            xseq[0] += 1
            _lib.check(_lib.lib.ebic_xgroup_evaluate(
                xgroup, off.ctypes.data_as(_lib.szp), cols.ctypes.data_as(_lib.u16p), len(off) - 1,
                t.sigma, t.eps, xseq[0], hc.ctypes.data_as(_lib.u64p), hf.ctypes.data_as(_lib.f64p)))
        for k in range(max(3, args.warmup)):
            call(*host_pops[k % len(host_pops)])
        for k in range(args.steps):
            off, cols = host_pops[k % len(host_pops)]
            evict_l2()
            torch.cuda.synchronize()
            dist.barrier()  # every rank enters the call together (outside the timing)
            a = time.perf_counter()
            call(off, cols)
            el += time.perf_counter() - a
            n_sh += len(off) - 1
            want = t.batches[k % len(t.batches)]
            assert (hf[:len(off) - 1].view(np.uint64) == want[3].view(np.uint64)).all(), "e2e fitness mismatch"
        tt = torch.tensor([el], dtype=torch.float64, device=dev if args.backend == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        el = float(tt.item())
        pb = [len(off) - 1 for off, _ in host_pops]
        lb = [int(off[-1]) for off, _ in host_pops]
        nb = len(host_pops)
        return {"value": n_sh / el, "unit": UNIT,
                "h2d_bytes_per_step": int(sum((p + 1) * 8 + l * 2 for p, l in zip(pb, lb)) / nb),
                "d2h_bytes_per_step": int(sum(16 * p for p in pb) / nb),
                "us_per_step": el / args.steps * 1e6,
                "caller": "ebic_xgroup_evaluate (C ABI) on every rank, host buffers; "
                          "cross-rank sum inside the count kernels"}

    e2e_sh = None
    if sharded and xgroup is not None:
        try:
            e2e_sh = sharded_e2e()
        except (RuntimeError, AssertionError) as exc:  # symmetric on every rank (shared results)
            e2e_sh = {"error": f"in-kernel cross-rank path failed: {exc}"[:300]}

    if xgroup is not None:  # the group refers to this context: release it first
        if rank != 0:
            _lib.check(_lib.lib.ebic_xgroup_destroy(xgroup))
        dist.barrier()
        if rank == 0:
            _lib.check(_lib.lib.ebic_xgroup_destroy(xgroup))
        xgroup = None
    cb = None
    if rank == 0 and not args.no_cpu_baseline:
        cb = cpu_reference(t, values, t.batches, steps=min(args.steps, 40), warmup=2,
                           budget_s=args.cpu_budget, single_budget_s=min(10.0, args.cpu_budget))

    if rank == 0:
        avg_bytes = nbytes / args.steps
        roof = None
        if avg_launch_ms:
            achieved = avg_bytes / (avg_launch_ms / 1e3) / 1e9
            traffic = None
            tp = ROOT / "profiles" / f"traffic_{args.workload}.json"
            if tp.exists():
                traffic = json.loads(tp.read_text()).get("dram_bytes_per_launch")
            roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": traffic,
                    "algorithmic_bytes_per_launch": avg_bytes,
                    "layout": LAYOUT_NAMES[layout], "cell_bytes": LAYOUT_CELL_BYTES[layout],
                    "peak_source": peak_src,
                    "kernel": ("count_tma_kernel (v1, fused Eq. 1 epilogue)" if os.environ.get("EBIC_KERNEL") == "1"
                               else "count_v2_kernel (K1v2, fused Eq. 1 epilogue)"),
                    "avg_launch_us": avg_launch_ms * 1e3}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator, bit-identical) + reference GA batches",
            "config": workload_config(t, args, world, n_devices),
            "roofline": roof, "cpu_baseline": cb, "clocks": clk,
            "e2e": e2e_sh if sharded else ({"value": e2e_cpp["e2e_biclusters_per_s"], "unit": UNIT,
                     "h2d_bytes_per_step": e2e_cpp["h2d_bytes_per_step"],
                     "d2h_bytes_per_step": e2e_cpp["d2h_bytes_per_step"],
                     "us_per_step": e2e_cpp["us_per_step"],
                     "caller": "C++ -> ebic_evaluate_population (C ABI), host buffers",
                     "parity_mismatched_steps": e2e_cpp["mismatched_steps"],
                     "host_us_breakdown": e2e_cpp.get("host_us")} if e2e_cpp else None),
            "e2e_python_api": ({"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d,
                                "d2h_bytes_per_step": d2h,
                                "caller": "Python Evaluator.evaluate_population (ctypes)"}
                               if e2e_val else None),
            "roofline_c5": big,
            "gpu_launches": args.steps * launches_per_step,
            "kernel_config": {"rows_per_tile": info.rows_per_tile, "stages": info.stages,
                              "grid": info.grid, "sm_count": info.sm_count,
                              "layout": LAYOUT_NAMES[info.layout],
                              "consumer_warps": info.consumer_warps},
            "parity": "counts and fitness bit-exact vs reference trace on every batch",
            **({"phases": phases} if phases else {}),
            "diag_back_to_back_us_per_step": b2b_us,
        }
        print(json.dumps(line), flush=True)
    ev.close()
    if sharded:
        dist.destroy_process_group()


def relaunch(n: int) -> int:
    """`bench.py --gpus N` started without torchrun: re-executes itself as N
    ranks (one process per GPU) under torch.distributed.run on 127.0.0.1 and
    returns the launcher's exit code.  Rank 0 prints the JSON line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c4",
                    help="c4: BASELINE config 4, steady-state GA batches (default); c5: config 5")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-large", action="store_true",
                    help="skip the config-5 (200,000 x 1000) roofline run")
    ap.add_argument("--backend", choices=["nccl", "gloo"], default="nccl",
                    help="torch.distributed backend (gloo: several ranks sharing one GPU, "
                         "kernel-side reduction only)")
    ap.add_argument("--reduce", choices=["kernel", "collective"], default="kernel",
                    help="device-resident multi-process path (`value`): cross-rank sum in the count "
                         "kernels (default; one launch per step, host wait per step), or an NCCL "
                         "all-reduce + Eq. 1 kernel; the e2e host path always sums inside the kernels")
    ap.add_argument("--force-sharded", action="store_true",
                    help="use the multi-process shard path (all-reduce + fitness kernel) even at N=1")
    ap.add_argument("--cpu-budget", type=float, default=15.0,
                    help="seconds of timed CPU reference work for cpu_baseline")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus))
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
