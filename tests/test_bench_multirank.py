"""The N > 1 path of bench.py (replicas, max over ranks) under world_size 2 with gloo on CPU."""
import os
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import bench

    w, r, _ = bench.dist_setup("gloo")
    ms_local = 10.0 + 5.0 * r           # rank 1 is the slow one
    ms_max, value = bench.aggregate(ms_local, steps=20, world=w, device="cpu")
    q.put((r, ms_max, value))
    import torch.distributed as dist

    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_max_over_ranks_and_whole_job_throughput():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=100) for _ in procs)
    for p in procs:
        p.join(timeout=30)
    assert all(p.exitcode == 0 for p in procs)
    for _, ms_max, value in out:
        assert ms_max == 15.0
        assert abs(value - 2 * 20 / 0.015) < 1e-6


@pytest.mark.timeout(300)
def test_bench_gpus_2_runs_end_to_end_on_cpu_ranks():
    """`python bench.py --gpus 2` relaunches itself under torch.distributed.run, runs the
    direction-sharded path on two gloo ranks (BENCH_PLUMBING=1: stand-in halves, no GPU) and
    rank 0 prints ONE JSON line with the contract's keys."""
    import json
    import subprocess

    env = dict(os.environ, BENCH_PLUMBING="1", CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
                          "--warmup", "3"], capture_output=True, text=True, env=env, timeout=280, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "config", "e2e", "clocks", "gpu_launches"):
        assert key in rec, key
    assert rec["n_gpus"] == 2 and rec["scaling"] == "strong" and rec["steps"] == 3
    assert "PLUMBING" in rec["data"]
    assert "parallelism" not in rec["config"]
