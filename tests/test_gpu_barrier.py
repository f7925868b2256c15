"""GPU tier: the global-checkpoint hook inside the checkpoint entry points.

SURVEY §8(e): one process per GPU, independent drains, a host barrier at
quiesce-complete and at image-complete marks the consistent global checkpoint.
The reference is single-process (ckpt_engine.cpp:29-61), so the contract here
is crac_engine.h's: every entry point calls the hook with PHASE_QUIESCED inside
the quiesce and PHASE_IMAGE_COMPLETE once its image is complete; a failing hook
fails the checkpoint with QuiesceTimeout and leaves the application running.
"""
import os
import time

import pytest
import torch.multiprocessing as mp

import workloads

pytestmark = pytest.mark.gpu

Q, IC, PE = 0, 1, 2


@pytest.fixture
def engine():
    from paper_2008_10596_b200 import engine as e
    return e


def _device_session(engine, seed=5):
    s = engine.Session(seed=seed, arena_bytes=64 << 20)
    workloads.build_regions(s, 6, lambda r: (1 << 20) + 4096 * r + 48, seed)
    return s


def test_hook_phases_of_every_entry_point(engine, tmp_path):
    s = _device_session(engine)
    plain, _ = s.checkpoint()
    seen = []
    s.set_barrier_hook(lambda ph: seen.append(ph))
    img = engine.Image()
    st = s.checkpoint_into(img)
    assert seen == [Q, IC] and img.tobytes() == plain
    assert st["barrier_ms"] >= 0
    seen.clear()
    s.checkpoint_into(img, incremental=True)
    assert seen == [Q, IC] and img.tobytes() == plain
    seen.clear()
    s.reserve_shadow(8 << 20)
    s.checkpoint_begin(img)
    assert seen == [Q]  # the image completes in finish
    s.checkpoint_finish()
    assert seen == [Q, IC] and img.tobytes() == plain
    seen.clear()
    s.checkpoint_begin(img)
    s.checkpoint_into(img)  # completes the pending one first: its IC, then its own pair
    assert seen == [Q, IC, Q, IC]
    s.reserve_shadow(0)
    seen.clear()
    s.checkpoint_precopy_begin(img)
    assert seen == []  # the application keeps running: not the checkpoint instant
    s.checkpoint_precopy_finish()
    assert seen == [Q, IC] and img.tobytes() == plain
    seen.clear()
    s.checkpoint_to_file(tmp_path / "a.img", img)
    assert seen == [Q, IC, PE]
    assert (tmp_path / "a.img").read_bytes() == plain
    s.set_barrier_hook(None)
    seen.clear()
    s.checkpoint_into(img)
    assert seen == []
    s.close()


def test_failing_hook_fails_the_checkpoint_and_resumes_the_app(engine):
    s = _device_session(engine)
    plain, _ = s.checkpoint()
    s.set_barrier_hook(lambda ph: 1 if ph == Q else 0)
    img = engine.Image()
    with pytest.raises(engine.CracError) as e:
        s.checkpoint_into(img)
    assert e.value.errc == "QuiesceTimeout"
    # the gate was released: the application can run and checkpoint again
    i, _ = s.alloc(engine.DEVICE, 4096)
    s.fill_synthetic(i, 9)
    s.free(i)
    s.set_barrier_hook(lambda ph: 1 if ph == IC else 0)
    with pytest.raises(engine.CracError):
        s.checkpoint_into(img)
    s.set_barrier_hook(None)
    again, _ = s.checkpoint()
    r, _ = engine.restart(again)
    assert r.checkpoint()[0] == again
    assert plain != again  # the alloc/free went into the log
    s.close()
    r.close()


def _rank(name, rank, delay, q):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import workloads as w
    from paper_2008_10596_b200 import engine as e
    s = e.Session(seed=11 + rank, arena_bytes=64 << 20)
    w.build_regions(s, 4, lambda r: (2 << 20) + 512 * r, 11 + rank)
    plain, _ = s.checkpoint()
    b = e.Barrier(name, 2, rank, timeout_ms=60000)
    s.set_barrier(b)
    img = e.Image()
    rows = []
    for k in range(3):
        time.sleep(delay)
        t0 = time.monotonic()
        st = s.checkpoint_into(img)
        rows.append((t0, time.monotonic(), st["barrier_ms"], img.tobytes() == plain))
    s.set_barrier(None)
    q.put((rank, rows))
    s.close()
    b.close(unlink=rank == 0)


def test_two_ranks_commit_one_global_checkpoint(engine):
    """Two processes (two ranks sharing this box's one GPU) checkpoint through
    the shared-memory barrier: the early rank's checkpoint cannot complete
    before the late rank started its own (so no rank resumes before every rank
    quiesced), its barrier wait shows the delay, and both images stay exact."""
    name = f"/crac_gpu_bar_{os.getpid()}"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(name, r, 0.0 if r == 0 else 0.5, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for k in range(3):
        early, late = res[0][k], res[1][k]
        assert early[3] and late[3]
        assert early[1] >= late[0], (k, early, late)
    assert max(r[2] for r in res[0]) > 300  # rank 0 waited for rank 1 in the hook
