"""Multi-process row shards with the reduction inside the count kernels
(ebic_xgroup_*, paper_1801_03039_b200/distributed.py reduce="kernel").

2 and 3 processes share the one GPU of the test box: every rank's kernel adds
its shard's totals into rank 0's accumulator through CUDA IPC and the last one
writes the result into a shared-memory block; no kernel waits for another, so
sharing a GPU is safe.  torch.distributed (gloo) only carries the handle.
Counts and fitness must equal the reference's trace values bit for bit.
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, reduce, q):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import paper_1801_03039_b200 as eb
    from paper_1801_03039_b200.distributed import RowShardedEvaluator
    from golden_io import trace
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        t = trace(name)
        v = t.matrix()
        ev = RowShardedEvaluator(v, device=0, reduce=reduce)
        bad = 0
        for rep in range(2):
            for off, cols, counts, fit in t.batches:
                pop = eb.CbfPopulation(off, cols)
                f = ev.evaluate_population(pop, eb.FitnessParams(t.sigma), t.eps)
                c = ev.count_matches(pop, t.eps)
                bad += int(not (c == counts).all()) + int(not (f.view(np.uint64) == fit.view(np.uint64)).all())
        q.put((rank, ev.reduce, bad))
        ev.close()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced through the queue
        q.put((rank, "error", repr(e)))


def _run(world, name, reduce):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, reduce, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    return sorted(out)


@pytest.mark.gpu
@pytest.mark.parametrize("world,name", [(2, "c4"), (3, "c3"), (2, "c1e")])
def test_in_kernel_cross_process_reduction(world, name):
    out = _run(world, name, "kernel")
    assert all(r[1] == "kernel" for r in out), out
    assert all(r[2] == 0 for r in out), out


@pytest.mark.gpu
def test_collective_reduction_on_gpu_shards():
    out = _run(2, "c3", "collective")
    assert all(r[1] == "collective" and r[2] == 0 for r in out), out


def _nccl_worker(port, q):
    """World size 1 over NCCL: the collective path must all-reduce a CUDA
    tensor (an NCCL group rejects host tensors).  reduce="kernel" with a
    population above the in-kernel limit (2048 series) takes the same path."""
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    import oracle
    import paper_1801_03039_b200 as eb
    from paper_1801_03039_b200.distributed import RowShardedEvaluator
    from golden_io import trace
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        t = trace("c3")
        v = t.matrix()
        bad = 0
        ev = RowShardedEvaluator(v, device=0, reduce="collective")
        for off, cols, counts, fit in t.batches:
            pop = eb.CbfPopulation(off, cols)
            f = ev.evaluate_population(pop, eb.FitnessParams(t.sigma), t.eps)
            bad += int(not (ev.count_matches(pop, t.eps) == counts).all())
            bad += int(not (f.view(np.uint64) == fit.view(np.uint64)).all())
        mode1 = ev.reduce
        ev.close()
        # > 2048 series: outside the in-kernel reduction's limit
        rng = np.random.default_rng(5)
        series = [list(map(int, rng.choice(v.shape[1], size=int(rng.integers(2, 6)), replace=False)))
                  for _ in range(2500)]
        pop = eb.encode_population(series)
        ev = RowShardedEvaluator(v, device=0, reduce="kernel")
        got = ev.count_matches(pop, t.eps)
        want = oracle.Port().count_matches(v, pop.offsets, pop.col_indices, t.eps)
        bad += int(not (got == want).all())
        ev.close()
        q.put((mode1, bad))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced through the queue
        q.put(("error", repr(e)))


@pytest.mark.gpu
def test_nccl_collective_path_world_one():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    p.start()
    out = q.get(timeout=600)
    p.join(timeout=120)
    assert out == ("collective", 0), out


@pytest.mark.gpu
def test_bench_launches_two_ranks_itself():
    """`bench.py --gpus 2` (no torchrun) re-executes itself as two ranks; with
    gloo both share the one GPU.  The line must say n_gpus 2; the bench asserts
    counts/fitness parity on every batch before timing."""
    import json
    import subprocess
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--backend", "gloo",
                        "--steps", "5", "--warmup", "3", "--no-large", "--no-cpu-baseline",
                        "--workload", "c4"], capture_output=True, text=True, timeout=900, env=env,
                       cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2
    assert "2 rank(s)" in line["config"]["parallelism"]
    assert line["e2e"] and "error" not in line["e2e"], line["e2e"]
