"""World-size-2 (and 3) gloo tests of the one-process-per-GPU path on CPU.

Each rank holds the rows shard_range(total, world, rank) of the matrix and
counts them; the per-series partial counts are all-reduced (int64 SUM) and Eq. 1
is applied to the reduced counts (paper_1801_03039_b200.distributed).  The
per-shard count here is the CPU oracle (no GPU in this container); the GPU run
uses the sm_100a kernel through the same class.  Expected values: the reference
GA traces (tests/golden).
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import oracle
    import paper_1801_03039_b200 as eb
    from paper_1801_03039_b200.distributed import RowShardedEvaluator
    from golden_io import trace
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = trace(name)
        v = t.matrix()
        port_ = oracle.Port()
        lo, hi = eb.shard_range(v.shape[0], world, rank)

        def local(pop, eps):
            return port_.count_matches(v[lo:hi], pop.offsets, pop.col_indices, eps)

        ev = RowShardedEvaluator(v, local_counter=local)
        ok = True
        for off, cols, counts, fit in t.batches[:3]:
            pop = eb.CbfPopulation(off, cols)
            got_c = ev.count_matches(pop, t.eps)
            got_f = ev.evaluate_population(pop, eb.FitnessParams(t.sigma), t.eps)
            ok &= bool((got_c == counts).all())
            ok &= bool((got_f.view(np.uint64) == fit.view(np.uint64)).all())
        q.put((rank, ok, (lo, hi)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,name", [(2, "c1e"), (2, "c2_scale"), (3, "c3")])
def test_row_sharded_allreduce_matches_reference(world, name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(ok for _, ok, _ in res)
    # shards tile the rows contiguously, 64-row aligned
    bounds = [b for _, _, b in res]
    assert bounds[0][0] == 0
    for (a0, a1), (b0, b1) in zip(bounds, bounds[1:]):
        assert a1 == b0 and a1 % 64 == 0


def test_shard_range_partitions():
    import paper_1801_03039_b200 as eb
    for total in (1, 63, 64, 65, 1000, 20000, 200000):
        for world in (1, 2, 3, 4, 8):
            lo_prev = 0
            for r in range(world):
                lo, hi = eb.shard_range(total, world, r)
                assert lo == lo_prev and hi >= lo
                lo_prev = hi
            assert lo_prev == total


def _bad_reduce_worker(port, q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_1801_03039_b200.distributed import RowShardedEvaluator
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        RowShardedEvaluator(np.zeros((4, 3)), reduce="kernal")
        q.put("accepted")
    except ValueError as e:
        q.put(str(e))
    finally:
        dist.destroy_process_group()


def test_invalid_reduce_rejected_before_any_device_work():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_bad_reduce_worker, args=(_free_port(), q))
    p.start()
    out = q.get(timeout=120)
    p.join(timeout=60)
    assert "reduce must be" in out


def test_bench_refuses_mismatched_world_size():
    """A line whose rank count differs from --gpus would mislabel a scaling
    run: bench.py refuses it (here WORLD_SIZE=2 but --gpus 3), and a
    self-launched `--gpus 2` on a box without 2 GPUs refuses in every rank."""
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "3", "--steps", "3",
                        "--warmup", "3"], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 2 and "refusing" in r.stderr
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--steps", "3",
                        "--warmup", "3"], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode != 0 and "refusing" in r.stderr
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
