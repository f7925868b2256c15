"""CPU tier: the global-checkpoint barrier of the C-ABI (crac_barrier_*), world_size 2.

The B200 box runs one process per GPU; each drains its own state and the only
cross-rank step is this host barrier (north_star "only a
host-side barrier marks a consistent global checkpoint").  These tests run the
barrier primitive itself in separate processes (no GPU needed); the hook's
placement inside the checkpoint entry points is covered by
tests/test_gpu_barrier.py.
"""
import os
import time

import pytest
import torch.multiprocessing as mp


def _name(tag: str) -> str:
    return f"/crac_test_{tag}_{os.getpid()}_{time.monotonic_ns() % 10**9}"


def _arrive(name, world, rank, delay, rounds, q):
    from paper_2008_10596_b200 import engine
    b = engine.Barrier(name, world, rank, timeout_ms=20000)
    out = []
    for k in range(rounds):
        time.sleep(delay * (k + 1))
        t_arrive = time.monotonic()
        b.wait()
        out.append((t_arrive, time.monotonic(), b.generation()))
    q.put((rank, out))
    b.close(unlink=(rank == 0))


def test_no_rank_leaves_before_every_rank_arrived():
    """'Neither rank may resume before both have quiesced': the early rank's
    wait returns only after the late rank arrived, for several consecutive
    checkpoints on the same segment (generation advances once per episode)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    name = _name("order")
    procs = [ctx.Process(target=_arrive, args=(name, 2, r, 0.0 if r == 0 else 0.3, 3, q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for k in range(3):
        early_leave = res[0][k][1]
        late_arrive = res[1][k][0]
        assert early_leave >= late_arrive, (k, res)
        # CLOCK_MONOTONIC is system-wide: both ranks compare on one clock
        assert res[0][k][2] == res[1][k][2]
    gens = [g for _, _, g in res[0]]
    assert gens == sorted(gens) and len(set(gens)) == 3


def test_timeout_withdraws_the_arrival_and_the_barrier_stays_usable():
    from paper_2008_10596_b200 import engine
    name = _name("timeout")
    b0 = engine.Barrier(name, 2, 0, timeout_ms=200)
    t0 = time.monotonic()
    with pytest.raises(engine.CracError) as e:
        b0.wait()  # rank 1 never comes
    assert e.value.rc == 12  # 1 + Errc::QuiesceTimeout
    assert time.monotonic() - t0 >= 0.19
    assert b0.generation() == 0
    # the withdrawn arrival leaves no phantom: a full episode still needs both
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_arrive, args=(name, 2, 1, 0.2, 1, q))
    p.start()
    t_before = time.monotonic()
    b0_long = engine.Barrier(name, 2, 0, timeout_ms=20000)
    b0_long.wait()
    rank, out = q.get(timeout=60)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert out[0][0] >= t_before  # rank 1 arrived after rank 0 started waiting
    assert b0_long.generation() == 1
    b0_long.close()
    b0.close(unlink=True)


def test_world_mismatch_and_bad_arguments_are_rejected():
    from paper_2008_10596_b200 import engine
    name = _name("world")
    b = engine.Barrier(name, 2, 0)
    with pytest.raises(engine.CracError) as e:
        engine.Barrier(name, 3, 1)
    assert e.value.rc == 1  # InvalidArgument
    with pytest.raises(engine.CracError):
        engine.Barrier("no_slash", 2, 0)
    with pytest.raises(engine.CracError):
        engine.Barrier(_name("rank"), 2, 2)
    b.close(unlink=True)


def test_single_rank_barrier_is_immediate():
    from paper_2008_10596_b200 import engine
    b = engine.Barrier(_name("one"), 1, 0, timeout_ms=10)
    for k in range(5):
        b.wait()
    assert b.generation() == 5
    b.close(unlink=True)
