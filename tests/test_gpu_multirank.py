"""GPU tier: the N-rank bench path end to end on this box's one GPU.

`bench.py --gpus 2 --share-gpu` launches two ranks (one process each, as on
an 8-GPU node, but both on cuda:0): gloo group, the product's shared-memory
global-checkpoint barrier installed on every session (every drain of the
timed loop meets the other rank at quiesce-complete and image-complete),
per-step max over ranks, and rank 0's single JSON line.  A small footprint
per rank keeps both states and images within one GPU / host.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def test_two_rank_bench_on_one_gpu():
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "LOCAL_WORLD_SIZE", "MASTER_PORT")}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--share-gpu",
                        "--footprint-gib", "2", "--steps", "2", "--warmup", "1",
                        "--no-cpu-baseline", "--no-stall"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    d = lines[0]
    assert d["n_gpus"] == 2 and d["steps"] == 2
    assert d["config"]["global_barrier"]
    assert d["verified"]["ok"]
    live = d["config"]["live_bytes_per_gpu"]
    assert live == 2 << 30
    # whole-box value: both ranks' bytes over the per-step max
    assert d["value"] == pytest.approx(2 * live * 2 * 2 / (d["ms_per_step"] * 2 * 1e-3) / 1e9,
                                       rel=1e-3)
