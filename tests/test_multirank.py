"""CPU tier: the N>1 host logic of bench.py on gloo, world_size 2.

The path has no data-path collective (independent per-GPU drains); the only
exchange is the host barrier and the max-over-ranks timing, tested here.
"""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, q) -> None:
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import bench
    g = bench.HostGroup(world, rank)
    g.barrier()
    m = g.max(float(10 + rank * 5))
    # per-rank device pinning: each rank sees only its LOCAL_RANK device
    os.environ.pop("CUDA_VISIBLE_DEVICES", None)
    bench.pin_device(rank, world)
    q.put((rank, m, os.environ["CUDA_VISIBLE_DEVICES"]))
    g.close()


def test_host_barrier_and_max_over_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    got = sorted(q.get(timeout=5) for _ in range(2))
    assert got == [(0, 15.0, "0"), (1, 15.0, "1")]


def test_reference_arm_nonzero_ranks_exit_without_work(capsys):
    import bench

    class A:
        impl = "reference"
        steps = 1
        warmup = 0
        region_mib = 64
        cpu_sample_gib = 0.0625

    bench.run_reference(A, world=2, rank=1)
    assert capsys.readouterr().out == ""


def test_bench_gpus_2_spawns_two_ranks_on_distinct_devices():
    """`bench.py --gpus 2` outside torchrun launches the two ranks itself,
    each pinned to its own device, joined by gloo and by the product's
    shared-memory checkpoint barrier (dry run: no GPU work)."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "LOCAL_WORLD_SIZE", "MASTER_PORT",
                        "CUDA_VISIBLE_DEVICES")}
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--dry-run"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert sorted(d["rank"] for d in lines) == [0, 1]
    assert all(d["world"] == 2 and d["dry_run"] for d in lines)
    devs = {d["rank"]: d["cuda_visible_devices"] for d in lines}
    assert devs == {0: "0", 1: "1"}
    assert all(d["barrier_generation"] == 1 for d in lines)
