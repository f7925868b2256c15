"""Deterministic call sequences run identically against the B200 engine
(paper_2008_10596_b200.engine.Session) and the reference (oracle.ref.RefSession).

Shapes follow the reference's own drivers: tests/support/sequence_gen.hpp
(SequenceDriver), test_ckpt_engine.cpp:32-68 (drive_ops) and the alloc_churn /
uvm_tasks workloads (src/harness.cpp:345-389, 443-519).
"""
from __future__ import annotations

import random

DEVICE, PINNED, MANAGED = 1, 2, 3
HOST_SIDE, DEVICE_SIDE = 0, 1
STD_KERNELS = [("fill8", 1, 2), ("add8", 1, 2), ("affine8", 1, 3), ("dot_f32", 3, 1),
               ("gemv_f32", 3, 2), ("gemm_f32", 3, 3)]


def patterned(n: int, salt: int) -> bytes:
    rnd = random.Random(salt)
    return bytes(rnd.getrandbits(8) for _ in range(n))


def drive_small(api, seed: int = 1) -> None:
    """Every section populated: all kinds, odd sizes, frees, streams, binaries,
    managed pages touched from both sides, queued launches, app state."""
    api.register_fat_binary(STD_KERNELS)
    h2 = api.register_fat_binary([("ephemeral", 1, 1)])
    s1 = api.stream_create()
    s2 = api.stream_create()
    s3 = api.stream_create()
    api.stream_destroy(s2)
    ids = []
    for k, size in enumerate([1000, 4096, 77, 65536 + 13, 100000, 256, 1]):
        i, _ = api.alloc(DEVICE, size)
        api.copy_h2d(i, 0, patterned(size, seed * 100 + k))
        ids.append(i)
    p1, _ = api.alloc(PINNED, 5000)
    api.copy_h2d(p1, 0, patterned(5000, seed + 7))
    m1, _ = api.alloc(MANAGED, 3 * 4096 + 100)
    api.page_write(m1, 0, patterned(3 * 4096 + 100, seed + 8), HOST_SIDE)
    m2, _ = api.alloc(MANAGED, 2 * 4096)
    api.page_write(m2, 4096, patterned(4096, seed + 9), DEVICE_SIDE)
    api.free(ids[2])
    g, _ = api.alloc(DEVICE, 64)  # reuses the freed hole
    api.copy_h2d(g, 0, patterned(64, seed + 10))
    api.unregister_fat_binary(h2)
    api.launch(s1, "fill8", [(ids[1], 0)], [0x5A, 4096])
    api.launch(s1, "add8", [(ids[1], 0)], [3, 2048])
    api.launch(s3, "affine8", [(ids[3], 0)], [7, 1, 65536])
    api.launch(s1, "add8", [(m1, 4096)], [1, 100])  # page 1 of m1 migrates to device
    api.synchronize()
    api.set_app_state(patterned(99, seed + 11))


def drive_random(api, seed: int, ops: int, arena: int, stamp: bool = True) -> None:
    """SequenceDriver (sequence_gen.hpp:13-122) restated: legal random calls."""
    rng = random.Random(seed)
    allocs, streams, binaries = [], [], []
    counter = 0
    for _ in range(ops):
        pick = rng.randrange(100)
        if pick < 45:
            kind = 1 + rng.randrange(3)
            size = 1 + rng.randrange(8192)
            try:
                i, _ = api.alloc(kind, size)
            except Exception as e:  # OutOfArena is a no-op in the driver
                if getattr(e, "errc", "") != "OutOfArena":
                    raise
                continue
            allocs.append(i)
            if stamp:
                b = patterned(min(size, 64), rng.randrange(1 << 30))
                if kind == MANAGED:
                    api.page_write(i, 0, b, HOST_SIDE)
                else:
                    api.copy_h2d(i, 0, b)
        elif pick < 75:
            if allocs:
                api.free(allocs.pop(rng.randrange(len(allocs))))
        elif pick < 85:
            if len(streams) < 100:
                streams.append(api.stream_create())
        elif pick < 92:
            if streams:
                api.stream_destroy(streams.pop(rng.randrange(len(streams))))
        elif pick < 97:
            n = 1 + rng.randrange(3)
            ks = []
            for _ in range(n):
                ks.append((f"gen_k{counter}", 1, 1))
                counter += 1
            binaries.append(api.register_fat_binary(ks))
        else:
            if binaries:
                api.unregister_fat_binary(binaries.pop(rng.randrange(len(binaries))))


def build_regions(api, n: int, size_fn, seed: int) -> list[int]:
    """C1 shape: n Device allocations with synthetic content."""
    ids = []
    for r in range(n):
        i, _ = api.alloc(DEVICE, size_fn(r))
        api.fill_synthetic(i, seed)
        ids.append(i)
    return ids


def build_churn(api, calls: int, seed: int, streams: int = 4, max_size: int = 65536) -> None:
    """C2 shape (alloc_churn, harness.cpp:476-499): 70 % alloc / 30 % free of
    256-byte-multiple Device sizes, one fill8 per allocation on 4 streams."""
    rng = random.Random(seed)
    api.register_fat_binary(STD_KERNELS)
    sids = [api.stream_create() for _ in range(streams)]
    live = []
    for c in range(calls):
        if live and rng.random() < 0.3:
            api.synchronize()  # queued launches may reference the victim
            api.free(live.pop(rng.randrange(len(live))))
        else:
            size = 256 * (1 + rng.randrange(max_size // 256))
            i, _ = api.alloc(DEVICE, size)
            api.launch(sids[c % streams], "fill8", [(i, 0)], [c & 0xFF, size])
            live.append(i)
        if c % 256 == 255:
            api.synchronize()
    api.synchronize()
