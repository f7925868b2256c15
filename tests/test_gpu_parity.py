"""GPU tier: the B200 drain/refill against the oracle, through the C-ABI.

Bar: bit-exact.  Every image the GPU path emits must equal, byte for byte,
the image the unmodified reference library emits for the same call sequence
(live, via oracle/_ref, and frozen in tests/golden); every restart must
reproduce the state; every corruption must be refused with ImageCorrupt.
"""
import os
import random
import struct
import zlib

import pytest

import workloads
from oracle import image_oracle as io
from oracle import ref

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------------------
# K1 (chunk CRC) against the restated zlib CRC
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n", [1, 15, 16, 17, 511, 512, 513, 4095, 4096, 4097, 65535, 65536,
                               65537, 65536 * 3 + 1234, 1 << 20])
@pytest.mark.parametrize("chunk", [512, 4096, 65536])
def test_k1_chunk_crc_matches_oracle(eng, n, chunk):
    data = os.urandom(n)
    got = eng.hash_chunks(data, chunk)
    want = ref.chunk_crc32(data, chunk)
    assert got == want
    assert want == [zlib.crc32(data[i:i + chunk]) for i in range(0, n, chunk)]


def test_k1_known_answer(eng):
    assert eng.hash_chunks(b"123456789", 512) == [0xCBF43926]
    zeros = bytes(65536)
    assert eng.hash_chunks(zeros) == [zlib.crc32(zeros)]


# ---------------------------------------------------------------------------
# drain parity: GPU image == reference image
# ---------------------------------------------------------------------------
def test_arena_sits_at_the_reference_base(eng):
    s = eng.Session(seed=0, arena_bytes=1 << 20)
    assert s.fixed_va  # logged addresses are the device pointers
    i, addr = s.alloc(workloads.DEVICE, 100)
    assert addr == 0x0D00_0000_0000 == s.backing_ptr(i)


def test_empty_session_is_188_bytes(eng, golden):
    _, images = golden
    s = eng.Session(seed=0, arena_bytes=1 << 24)
    img, stats = s.checkpoint()
    assert img == images["empty"]
    assert stats["image_bytes"] == 188


def test_small_session_matches_golden_and_live_reference(eng, golden):
    _, images = golden
    s = eng.Session(seed=3, arena_bytes=1 << 22)
    workloads.drive_small(s, seed=1)
    img, stats = s.checkpoint()
    assert img == images["small_session"]
    r = ref.RefSession(seed=3, arena_bytes=1 << 22)
    workloads.drive_small(r, seed=1)
    assert img == r.checkpoint()[0]
    assert stats["hash_launches"] >= 1 and stats["pack_launches"] >= 1
    # the value-type adapter (checkpoint -> Snapshot -> encode_image) agrees
    assert s.checkpoint_value() == img


def test_c1_mini_matches_golden(eng, golden):
    _, images = golden
    s = eng.Session(seed=1, arena_bytes=1 << 24)
    workloads.build_regions(s, 8, lambda r: 100 * 1024 - r % 3 * 17, seed=1)
    assert s.checkpoint()[0] == images["c1_mini"]


def test_random_sequence_matches_golden(eng, golden):
    _, images = golden
    s = eng.Session(seed=7, arena_bytes=1 << 20)
    workloads.drive_random(s, seed=42, ops=300, arena=1 << 20)
    assert s.checkpoint()[0] == images["random_300"]


@pytest.mark.parametrize("seed", range(6))
def test_random_sessions_match_reference(eng, seed):
    s = eng.Session(seed=seed, arena_bytes=1 << 21)
    r = ref.RefSession(seed=seed, arena_bytes=1 << 21)
    for api in (s, r):
        workloads.drive_random(api, seed=1000 + seed, ops=400, arena=1 << 21)
        api.set_app_state(bytes([seed]) * (seed * 7))
    assert s.checkpoint()[0] == r.checkpoint()[0]


def test_checkpoint_is_non_destructive_and_repeatable(eng):
    s = eng.Session(seed=2, arena_bytes=1 << 22)
    workloads.drive_small(s, seed=5)
    a = s.checkpoint()[0]
    b = s.checkpoint()[0]
    assert a == b
    # the session keeps working and the log continues
    i, addr = s.alloc(workloads.DEVICE, 2048)
    r = ref.RefSession(seed=2, arena_bytes=1 << 22)
    workloads.drive_small(r, seed=5)
    r.checkpoint()
    assert (i, addr) == r.alloc(workloads.DEVICE, 2048)


def test_c1_shape_odd_sizes_matches_reference(eng):
    # odd region sizes (4 MiB - r%3) stress the misaligned framing
    n, size = 24, lambda r: (1 << 20) - r % 3
    s = eng.Session(seed=1, arena_bytes=32 << 20)
    r = ref.RefSession(seed=1, arena_bytes=32 << 20)
    for api in (s, r):
        workloads.build_regions(api, n, size, seed=1)
    img, stats = s.checkpoint()
    assert img == r.checkpoint()[0]
    assert stats["d2h_bytes"] == sum(16 + size(k) for k in range(n)) + 20


def test_queued_work_is_drained_before_capture(eng):
    # test_ckpt_engine.cpp:332-349
    s = eng.Session(seed=0, arena_bytes=1 << 20)
    s.register_fat_binary(workloads.STD_KERNELS)
    st = s.stream_create()
    i, _ = s.alloc(workloads.DEVICE, 1024)
    s.launch(st, "fill8", [(i, 0)], [9, 1024])
    s.launch(st, "add8", [(i, 0)], [1, 1024])
    img = s.checkpoint()[0]
    snap = io.decode_image(img)
    assert snap.payloads == [(i, bytes([10]) * 1024)]


# ---------------------------------------------------------------------------
# refill
# ---------------------------------------------------------------------------
def _state(api):
    recs = api.live_records()
    out = []
    for rec in recs:
        rid, kind, size, addr = (rec.id, rec.kind, rec.size, rec.address) if hasattr(rec, "id") else rec
        entry = [rid, kind, size, addr, api.read_raw(addr, size)]
        if kind == workloads.MANAGED:
            entry.append(api.managed_pages(rid))
        out.append(entry)
    return out


def test_restart_round_trip_is_lossless(eng):
    s = eng.Session(seed=4, arena_bytes=1 << 22)
    workloads.drive_small(s, seed=2)
    first, _ = s.checkpoint()
    r, stats = eng.restart(first)
    assert _state(r) == _state(s)
    second, _ = r.checkpoint()
    assert second == first  # test_ckpt_engine.cpp:212-224
    assert stats["h2d_bytes"] > 0 and stats["hash_launches"] >= 1
    # ids / stream ids continue past the old ceiling
    assert r.stream_create() == s.stream_create()
    assert r.alloc(workloads.DEVICE, 64) == s.alloc(workloads.DEVICE, 64)


def test_restart_from_reference_images(eng, golden):
    _, images = golden
    for name in ("small_session", "c1_mini", "empty"):
        r, _ = eng.restart(images[name])
        assert r.checkpoint()[0] == images[name]
        live = ref.ref_restart(images[name])[0]
        assert _state(r) == _state(live)


def test_reference_restarts_from_gpu_images(eng):
    s = eng.Session(seed=9, arena_bytes=1 << 22)
    workloads.drive_small(s, seed=3)
    img, _ = s.checkpoint()
    rs, _ = ref.ref_restart(img)
    assert rs.checkpoint()[0] == img


def test_restart_of_restart_is_lossless(eng, golden):
    _, images = golden
    img = images["small_session"]
    for _ in range(3):
        r, _ = eng.restart(img)
        img2 = r.checkpoint()[0]
        assert img2 == img
        img = img2


def test_bulk_corruption_is_caught_by_the_gpu_verify(eng, golden):
    _, images = golden
    img = bytearray(images["c1_mini"])
    summ = ref.ref_summarize(bytes(img))
    s3 = 16 + (20 + 24) + (20 + summ["lengths"][1]) + 16
    rnd = random.Random(1)
    for _ in range(24):
        # flip a payload (not frame) bit deep inside ALLOC_PAYLOADS
        pos = s3 + 16 + rnd.randrange(100 * 1024 - 64)
        bit = 1 << rnd.randrange(8)
        img[pos] ^= bit
        with pytest.raises(eng.CracError) as e:
            eng.restart(bytes(img))
        assert e.value.errc == "ImageCorrupt"
        img[pos] ^= bit
    eng.restart(bytes(img))  # restored image is accepted


def test_every_bit_flip_of_small_image_refused_by_restart(eng, golden):
    _, images = golden
    img = bytearray(images["small_session"])
    rnd = random.Random(3)
    for _ in range(64):
        bit = rnd.randrange(len(img) * 8)
        img[bit // 8] ^= 1 << (bit % 8)
        with pytest.raises(eng.CracError) as e:
            eng.restart(bytes(img))
        assert e.value.errc == "ImageCorrupt"
        img[bit // 8] ^= 1 << (bit % 8)


def test_tampered_log_address_is_replay_divergence(eng, golden):
    _, images = golden
    snap = io.decode_image(images["small_session"])
    # second Alloc record: shift its address by one alignment unit (test_ckpt_engine.cpp:132-141)
    k = [i for i, e in enumerate(snap.log) if e[1] == 1][1]
    seq, op, kind, size, ident, addr = snap.log[k]
    snap.log[k] = (seq, op, kind, size, ident, addr + 256)
    bad = io.encode_image(snap)
    with pytest.raises(eng.CracError) as e:
        eng.restart(bad)
    assert e.value.errc in ("ReplayDivergence", "ImageCorrupt")
    with pytest.raises(ref.RefError) as e2:
        ref.ref_restart(bad)
    assert e.value.errc == e2.value.errc


@pytest.mark.parametrize("which", ["live_last", "live_first", "freed"])
def test_tampered_device_only_log_while_data_path_runs(eng, which):
    """Device-only images at the fixed VA refill before the replay has run
    (the destinations are the logged addresses); a log whose replay diverges
    must still be refused with the reference's error, with the engine
    streams drained before the session unwinds, and the next restart works."""
    s = eng.Session(seed=5, arena_bytes=1 << 30)
    ids = workloads.build_regions(s, 12, lambda k: (3 << 20) + 4096 * k + 5 * k, seed=5)
    s.free(ids[3])
    s.free(ids[7])
    i, _ = s.alloc(workloads.DEVICE, 5000)
    s.fill_synthetic(i, 5)
    good, _ = s.checkpoint()
    snap = io.decode_image(good)
    allocs = [k for k, e in enumerate(snap.log) if e[1] == 1]
    freed = {e[4] for e in snap.log if e[1] == 2}
    live = [k for k in allocs if snap.log[k][4] not in freed]
    k = {"live_last": live[-1], "live_first": live[0],
         "freed": [a for a in allocs if snap.log[a][4] in freed][0]}[which]
    seq, op, kind, size, ident, addr = snap.log[k]
    snap.log[k] = (seq, op, kind, size, ident, addr + 256)
    bad = io.encode_image(snap)
    with pytest.raises(eng.CracError) as e:
        eng.restart(bad)
    with pytest.raises(ref.RefError) as e2:
        ref.ref_restart(bad)
    assert e.value.errc in ("ReplayDivergence", "ImageCorrupt")
    assert e.value.errc == e2.value.errc
    r, _ = eng.restart(good)
    assert r.checkpoint()[0] == good


def test_unknown_kernel_body_refused(eng, golden):
    _, images = golden
    # "scale"/"probe" and the random gen_k* kernels are not in the standard catalog
    for name in ("rich", "random_300"):
        with pytest.raises(eng.CracError) as e:
            eng.restart(images[name])
        assert e.value.errc == "UnknownKernelBody"
        with pytest.raises(ref.RefError) as e2:
            ref.ref_restart(images[name])
        assert e2.value.errc == "UnknownKernelBody"


def test_managed_residence_restored(eng):
    s = eng.Session(seed=1, arena_bytes=1 << 22)
    m, _ = s.alloc(workloads.MANAGED, 6 * 4096 + 10)
    s.page_write(m, 0, workloads.patterned(6 * 4096 + 10, 1), workloads.HOST_SIDE)
    s.page_read(m, 2 * 4096, 3 * 4096, workloads.DEVICE_SIDE)
    flags = s.managed_pages(m)
    assert flags == [2, 2, 3, 3, 3, 2, 2]
    img, _ = s.checkpoint()
    r, _ = eng.restart(img)
    assert r.managed_pages(m) == flags
    assert r.page_read(m, 0, 6 * 4096 + 10, workloads.HOST_SIDE) == workloads.patterned(6 * 4096 + 10, 1)


# ---------------------------------------------------------------------------
# incremental drain (new behaviour: must emit exactly the full image)
# ---------------------------------------------------------------------------
def _mutate_reference(r, sizes, ids, seed, epoch, threshold, chunk=65536):
    """The C5 epoch mutation restated on the reference session (crac_gpu.h:
    chunk c changes iff mix64(seed ^ (epoch << 40) ^ c) < threshold, new content
    = synth(seed + epoch) of that chunk's words)."""
    c = 0
    for size, i in zip(sizes, ids):
        for off in range(0, size, chunk):
            if ref.mix64(seed ^ (epoch << 40) ^ c) < threshold:
                n = min(chunk, size - off)
                r.copy_h2d(i, off, ref.synth_bytes(seed + epoch, i, n, off // 8))
            c += 1


@pytest.mark.parametrize("pct", [0, 1, 25, 100])
def test_incremental_equals_full(eng, pct):
    sizes = [(4 << 20) - k * 4096 - (k % 2) * 100 for k in range(12)]
    s = eng.Session(seed=1, arena_bytes=64 << 20)
    r = ref.RefSession(seed=1, arena_bytes=64 << 20)
    ids = workloads.build_regions(s, 12, lambda k: sizes[k], seed=3)
    assert workloads.build_regions(r, 12, lambda k: sizes[k], seed=3) == ids
    image = eng.Image()
    st0 = s.checkpoint_into(image)
    assert not st0["incremental"]
    assert image.tobytes() == r.checkpoint()[0]
    threshold = (2**64 - 1) * pct // 100
    for epoch in range(1, 3):
        mutated = s.mutate(seed=3, epoch=epoch, threshold=threshold)
        _mutate_reference(r, sizes, ids, 3, epoch, threshold)
        st = s.checkpoint_into(image, incremental=True)
        assert st["incremental"]
        assert st["dirty_chunks"] == mutated
        assert image.tobytes() == r.checkpoint()[0]  # exactly the full image


def test_incremental_falls_back_when_layout_changes(eng):
    s = eng.Session(seed=1, arena_bytes=16 << 20)
    workloads.build_regions(s, 4, lambda r: 1 << 20, seed=1)
    image = eng.Image()
    s.checkpoint_into(image)
    i, _ = s.alloc(workloads.DEVICE, 12345)
    s.fill_synthetic(i, 5)
    st = s.checkpoint_into(image, incremental=True)
    assert not st["incremental"]
    assert image.tobytes() == s.checkpoint()[0]


# ---------------------------------------------------------------------------
# config shapes: C2 churn, C3 managed with mixed residence
# ---------------------------------------------------------------------------
def test_c2_churn_matches_reference(eng):
    s = eng.Session(seed=2, arena_bytes=256 << 20)
    r = ref.RefSession(seed=2, arena_bytes=256 << 20)
    for api in (s, r):
        workloads.build_churn(api, 3000, seed=5, max_size=16384)
    img, st = s.checkpoint()
    assert img == r.checkpoint()[0]
    rs, _ = eng.restart(img)
    assert rs.checkpoint()[0] == img
    assert _state(rs) == _state(s)


def test_c3_managed_mixed_residence_matches_reference(eng):
    s = eng.Session(seed=3, arena_bytes=64 << 20)
    r = ref.RefSession(seed=3, arena_bytes=64 << 20)
    for api in (s, r):
        for k in range(6):
            i, _ = api.alloc(workloads.MANAGED, (1 << 20) + 4096 * k + 123 * (k % 2))
            api.fill_synthetic(i, 7, workloads.DEVICE_SIDE)
            for off in range(64 << 10, 1 << 20, 128 << 10):
                api.page_read(i, off, 64 << 10, workloads.HOST_SIDE)
        d, _ = api.alloc(workloads.DEVICE, 100000)
        api.fill_synthetic(d, 7)
    img, _ = s.checkpoint()
    assert img == r.checkpoint()[0]
    rs, _ = eng.restart(img)
    assert _state(rs) == _state(s)
    assert rs.checkpoint()[0] == img


def test_direct_runs_edges_match_reference(eng):
    """Device payloads around the direct-run threshold (6 stream tiles plus
    the 64-byte margins), payloads that straddle 64 MiB window boundaries,
    odd sizes on every word phase, a big Pinned payload (never direct) and a
    managed one between them: the image equals the reference's, and the
    refill (direct H2D + edge scatter) restores every byte."""
    MIB, T = 1 << 20, 65536
    sizes = [6 * T + 127, 6 * T + 128, 6 * T + 129, 7 * T, 7 * T + 15, 64 * MIB + 1,
             30 * MIB + 3, 30 * MIB + 5, 30 * MIB + 7, 5 * T - 1]
    s = eng.Session(seed=11, arena_bytes=512 * MIB)
    r = ref.RefSession(seed=11, arena_bytes=512 * MIB)
    for api in (s, r):
        for k, size in enumerate(sizes):
            i, _ = api.alloc(workloads.DEVICE, size)
            api.fill_synthetic(i, 40 + k)
            if k == 4:
                p_, _ = api.alloc(workloads.PINNED, 2 * MIB + 9)
                api.fill_synthetic(p_, 3)
                m, _ = api.alloc(workloads.MANAGED, MIB + 77)
                api.fill_synthetic(m, 4, workloads.DEVICE_SIDE)
    img, st = s.checkpoint()
    assert img == r.checkpoint()[0]
    rs, _ = eng.restart(img)
    assert _state(rs) == _state(s)
    assert rs.checkpoint()[0] == img


def test_refill_skips_ring_windows_no_scatter_reads(eng):
    """Big Device payloads only (the C4 shape at 10 x 64 MiB, plus one odd
    size): past the early windows, a window holds only frames between exact
    direct runs, so the refill skips its ring H2D (CRAC_RING_SKIP) -- fewer
    H2D bytes than the stream -- and still restores every byte, cold and
    warm."""
    MIB = 1 << 20
    sizes = [64 * MIB] * 9 + [64 * MIB + 4097]
    s = eng.Session(seed=21, arena_bytes=704 * MIB)
    r = ref.RefSession(seed=21, arena_bytes=704 * MIB)
    for api in (s, r):
        for k, size in enumerate(sizes):
            i, _ = api.alloc(workloads.DEVICE, size)
            api.fill_synthetic(i, 60 + k)
    img, st = s.checkpoint()
    assert img == r.checkpoint()[0]
    want = _state(s)
    s.close()
    eng.drop_arena_cache()
    rs, rst = eng.restart(img)  # cold
    assert rst["h2d_bytes"] < st["d2h_bytes"], (rst["h2d_bytes"], st["d2h_bytes"])
    assert _state(rs) == want
    assert rs.checkpoint()[0] == img
    rs.close()
    rw, _ = eng.restart(img)  # warm (the arena of the closed session adopted)
    assert _state(rw) == want and rw.checkpoint()[0] == img


def test_c3_host_runs_skip_the_link_and_match_reference(eng):
    """Host-resident runs >= 256 KiB never cross PCIe (the window copies skip
    them; host threads write their frames and content).  Runs straddle the
    64 MiB window boundaries, one ends at a partial last page, short runs
    (< 256 KiB) ride along as zeros and are overwritten after landing."""
    MIB = 1 << 20
    s = eng.Session(seed=4, arena_bytes=256 * MIB)
    r = ref.RefSession(seed=4, arena_bytes=256 * MIB)
    sizes = [40 * MIB + 4096 * k + 77 * k for k in range(3)]
    for api in (s, r):
        for k, size in enumerate(sizes):
            i, _ = api.alloc(workloads.MANAGED, size)
            api.fill_synthetic(i, 9 + k, workloads.DEVICE_SIDE)
            for off in range(MIB // 2, size - MIB, 2 * MIB):       # 1 MiB runs
                api.page_read(i, off, MIB, workloads.HOST_SIDE)
            for off in range(MIB // 4, 8 * MIB, 4 * MIB):          # 64 KiB runs
                api.page_read(i, off, 64 << 10, workloads.HOST_SIDE)
            api.page_read(i, size - 300 * 1024, 300 * 1024, workloads.HOST_SIDE)  # to the end
        d, _ = api.alloc(workloads.DEVICE, 3 * MIB + 5)
        api.fill_synthetic(d, 7)
    img, st = s.checkpoint()
    assert img == r.checkpoint()[0]
    assert st["d2h_bytes"] < len(img) * 0.7  # the big host runs stayed off the link
    rs, rst = eng.restart(img)
    assert rst["h2d_bytes"] == st["d2h_bytes"]
    assert _state(rs) == _state(s)
    assert rs.checkpoint()[0] == img


@pytest.mark.parametrize("shadow", [0, 1, 64], ids=["sync", "ring+shadow", "all-shadow"])
def test_pinned_payloads_move_on_the_host_and_match_reference(eng, shadow):
    """Pinned-host payloads of >= 256 KiB are moved by host threads between
    the allocation and the image (their bytes never cross PCIe for the move:
    d2h / h2d exclude them); small ones ride the windows.  Byte-equal to the
    reference for the synchronous and the stall-reduced drains, and through
    the restart."""
    MIB = 1 << 20
    s = eng.Session(seed=6, arena_bytes=512 * MIB)
    r = ref.RefSession(seed=6, arena_bytes=512 * MIB)
    big = [5 * MIB + 3, 70 * MIB + 4096 + 5, 256 * 1024, 3 * MIB]
    small = [1000, 255 * 1024]
    for api in (s, r):
        for k, size in enumerate(big + small):
            i, _ = api.alloc(workloads.PINNED, size)
            api.fill_synthetic(i, 20 + k)
            d, _ = api.alloc(workloads.DEVICE, MIB + 17 * k)
            api.fill_synthetic(d, 40 + k)
    want = r.checkpoint()[0]
    if shadow:
        s.reserve_shadow(shadow * MIB)
        img = eng.Image()
        s.checkpoint_begin(img)
        st = s.checkpoint_finish()
        got = img.tobytes()
        s.reserve_shadow(0)
    else:
        img = eng.Image()
        st = s.checkpoint_into(img)
        got = img.tobytes()
        # the host-computed chunk CRCs and dirty keys of the pinned runs equal
        # the GPU's: an incremental drain of the unchanged state finds nothing
        inc = s.checkpoint_into(img, incremental=True)
        assert inc["incremental"] and inc["dirty_chunks"] == 0
        assert img.tobytes() == want
    assert got == want
    assert st["d2h_bytes"] <= len(got) - sum(big)
    rs, rst = eng.restart(got)
    assert rst["h2d_bytes"] <= len(got) - sum(big)
    assert _state(rs) == _state(s)
    assert rs.checkpoint()[0] == want
    rs.close()
    s.close()
    r.close()


# ---------------------------------------------------------------------------
# edge shapes and error parity (test_device_core.cpp / test_shim.cpp cases)
# ---------------------------------------------------------------------------
def _shape_tiny(api):
    for kind in (workloads.DEVICE, workloads.PINNED, workloads.MANAGED):
        i, _ = api.alloc(kind, 1)
        if kind == workloads.MANAGED:
            api.page_write(i, 0, b"\x7f", workloads.HOST_SIDE)
        else:
            api.copy_h2d(i, 0, b"\x7f")


def _shape_chunk_edges(api):
    for k, size in enumerate([65535, 65536, 65537, 131073, 4096 * 3, 255, 257]):
        i, _ = api.alloc(workloads.DEVICE, size)
        api.fill_synthetic(i, 11 + k)
    for size in (4096, 8192, 4097):
        i, _ = api.alloc(workloads.MANAGED, size)
        api.fill_synthetic(i, 5, workloads.DEVICE_SIDE)


def _shape_streams_and_binaries(api):
    ids = [api.stream_create() for _ in range(128)]
    for s in ids[::3]:
        api.stream_destroy(s)
    hs = [api.register_fat_binary([(f"k{b}_{j}", 1 + j, j) for j in range(3)]) for b in range(40)]
    for h in hs[::3]:
        api.unregister_fat_binary(h)
    api.set_app_state(bytes(range(256)) * 4096)  # 1 MiB of app state


@pytest.mark.parametrize("shape", [_shape_tiny, _shape_chunk_edges, _shape_streams_and_binaries])
def test_edge_shapes_match_reference(eng, shape):
    s = eng.Session(seed=8, arena_bytes=4 << 20)
    r = ref.RefSession(seed=8, arena_bytes=4 << 20)
    shape(s)
    shape(r)
    img = s.checkpoint()[0]
    assert img == r.checkpoint()[0]
    if shape is not _shape_streams_and_binaries:  # generated kernels have no bodies
        rs, _ = eng.restart(img)
        assert rs.checkpoint()[0] == img


def _errc(fn):
    try:
        fn()
    except (ref.RefError, Exception) as e:  # noqa: B014
        return getattr(e, "errc", type(e).__name__)
    return None


def test_error_codes_match_reference(eng):
    cases = []
    for api in (eng.Session(seed=1, arena_bytes=1 << 20), ref.RefSession(seed=1, arena_bytes=1 << 20)):
        a, _ = api.alloc(workloads.DEVICE, 1024)
        m, _ = api.alloc(workloads.MANAGED, 8192)
        api.register_fat_binary(workloads.STD_KERNELS)
        st = api.stream_create()
        api.free(a)
        out = [
            _errc(lambda: api.free(a)),                                   # DoubleFree
            _errc(lambda: api.free(999)),                                 # UnknownId
            _errc(lambda: api.alloc(workloads.DEVICE, 0)),                # InvalidArgument
            _errc(lambda: api.alloc(workloads.DEVICE, 2 << 20)),          # OutOfArena
            _errc(lambda: api.launch(st, "nope", [(m, 0)], [1, 2])),      # UnregisteredKernel
            _errc(lambda: api.launch(st, "fill8", [(m, 0)], [1])),        # arity: InvalidArgument
            _errc(lambda: api.launch(st, "fill8", [(m, 9000)], [1, 1])),  # OutOfRange
            _errc(lambda: api.copy_h2d(m, 8190, b"1234")),                # OutOfRange
            _errc(lambda: api.stream_destroy(77)),                        # UnknownId
            _errc(lambda: api.register_fat_binary([("fill8", 1, 2)])),    # DuplicateKernelId
        ]
        api.launch(st, "fill8", [(m, 0)], [3, 8192])
        out.append(_errc(lambda: api.stream_destroy(st)))                 # BusyStream
        api.synchronize()
        out.append(_errc(lambda: api.stream_destroy(st)))                 # None
        d2, _ = api.alloc(workloads.DEVICE, 64)
        out.append(_errc(lambda: api.page_read(d2, 0, 8, workloads.HOST_SIDE)))  # NotManaged
        cases.append(out)
    assert cases[0] == cases[1]
    assert cases[0][0] == "DoubleFree" and cases[0][10] == "BusyStream"


# ---------------------------------------------------------------------------
# stall-reduced drain (checkpoint_begin / checkpoint_finish)
# ---------------------------------------------------------------------------
MIB = 1 << 20


def _big_state(api):
    """3 x 40 MiB device regions, an 80 MiB managed allocation with 1 MiB
    alternating residence, plus every small section populated."""
    workloads.drive_small(api, seed=4)
    for k in range(3):
        i, _ = api.alloc(workloads.DEVICE, 40 * MIB - 17 * k)
        api.fill_synthetic(i, 20 + k)
    m, _ = api.alloc(workloads.MANAGED, 80 * MIB + 333)
    api.fill_synthetic(m, 9, workloads.DEVICE_SIDE)
    for off in range(MIB, 80 * MIB, 2 * MIB):
        api.page_read(m, off, MIB, workloads.HOST_SIDE)
    for off in range(MIB // 2, 80 * MIB, 8 * MIB):  # short (64 KiB) host runs
        api.page_read(m, off, 64 << 10, workloads.HOST_SIDE)
    return m


@pytest.mark.parametrize("shadow_mib", [0, 64, 128, 512])
def test_async_drain_is_the_image_at_begin(eng, shadow_mib):
    s = eng.Session(seed=6, arena_bytes=512 * MIB)
    m = _big_state(s)
    want = s.checkpoint()[0]
    s.reserve_shadow(shadow_mib * MIB)
    img = eng.Image()
    st = s.checkpoint_begin(img)
    stream = len(want) - 1000  # roughly the bulk stream
    if shadow_mib >= 512:
        assert st["shadow_bytes"] > stream - 64 * MIB
    elif shadow_mib == 0:
        assert st["shadow_bytes"] == 0
    else:
        assert 0 < st["shadow_bytes"] <= shadow_mib * MIB
    # the app runs while the D2H drains: none of this may reach the image
    s.mutate(seed=1, epoch=1, threshold=(1 << 64) - 1)
    s.page_write(m, 5 * MIB, b"\xEE" * 8192, workloads.HOST_SIDE)
    s.page_write(m, 6 * MIB, b"\xDD" * 8192, workloads.DEVICE_SIDE)
    x, _ = s.alloc(workloads.DEVICE, 4096)
    s.free(x)
    done = s.checkpoint_finish()
    assert img.tobytes() == want
    assert done["stall_ms"] <= done["total_ms"]
    assert done["d2h_bytes"] > 0
    rs, _ = eng.restart(img.tobytes())
    assert rs.checkpoint()[0] == want
    assert s.checkpoint()[0] != want  # the mutations are live


@pytest.mark.parametrize("shadow_mib", [64, 512])
def test_async_drain_with_managed_runs_matches_reference(eng, shadow_mib):
    """The stall-reduced drain over long and short host-resident runs equals
    the reference's image; host pages change right after begin."""
    s = eng.Session(seed=6, arena_bytes=512 * MIB)
    r = ref.RefSession(seed=6, arena_bytes=512 * MIB)
    m = _big_state(s)
    _big_state(r)
    want = r.checkpoint()[0]
    s.reserve_shadow(shadow_mib * MIB)
    img = eng.Image()
    s.checkpoint_begin(img)
    s.page_write(m, MIB // 2, b"\x11" * 4096, workloads.HOST_SIDE)   # a short-run page
    s.page_write(m, 3 * MIB, b"\x22" * 8192, workloads.HOST_SIDE)    # a long-run page
    s.checkpoint_finish()
    assert img.tobytes() == want
    s.reserve_shadow(0)


def test_buddy_shadow_placement(eng):
    """reserve_shadow on a device: this GPU's own ordinal is
    the ordinary shadow; an ordinal with no peer route is refused with
    InvalidArgument and leaves the session able to drain."""
    import torch
    s = eng.Session(seed=2, arena_bytes=1 << 22)
    r = ref.RefSession(seed=2, arena_bytes=1 << 22)
    for api in (s, r):
        workloads.drive_small(api, seed=6)
    want = r.checkpoint()[0]
    s.reserve_shadow(64 * MIB, device=0)
    img = eng.Image()
    s.checkpoint_begin(img)
    s.checkpoint_finish()
    assert img.tobytes() == want
    n = torch.cuda.device_count()
    with pytest.raises(eng.CracError) as e:
        s.reserve_shadow(64 * MIB, device=n + 3)
    assert e.value.errc == "InvalidArgument"
    assert s.checkpoint()[0] == want
    if n > 1:  # a real buddy: the snapshot crosses NVLink
        s.reserve_shadow(64 * MIB, device=1)
        s.checkpoint_begin(img)
        s.checkpoint_finish()
        assert img.tobytes() == want
    s.reserve_shadow(0)


def test_precopy_drain_is_the_image_at_finish(eng):
    """Pre-copy: the state changes while phase 1 copies it (a
    device kernel rewriting ~10 % of the chunks, a host copy); the image is the
    state at finish, and only the changed chunks were sent again."""
    s = eng.Session(seed=9, arena_bytes=1 << 30)
    workloads.build_regions(s, 6, lambda k: 24 * MIB + 4096 * k + 3 * k, seed=9)
    img = eng.Image()
    s.checkpoint_precopy_begin(img)
    mutated = s.mutate(seed=2, epoch=1, threshold=(1 << 64) // 10)
    first = s.live_records()[0].id
    s.copy_h2d(first, 1000, b"\x42" * 5000)
    st = s.checkpoint_precopy_finish()
    assert st["incremental"] == 1
    assert 0 < st["dirty_chunks"] < st["total_chunks"]
    assert st["dirty_chunks"] <= mutated + 2
    assert st["stall_ms"] <= st["total_ms"]
    want = s.checkpoint()[0]
    assert img.tobytes() == want
    rs, _ = eng.restart(want)
    assert rs.checkpoint()[0] == want


def test_precopy_layout_change_and_ineligible_sessions(eng):
    # an allocation during phase 1: finish falls back to a full drain
    s = eng.Session(seed=3, arena_bytes=1 << 28)
    workloads.build_regions(s, 3, lambda k: 8 * MIB + k, seed=3)
    img = eng.Image()
    s.checkpoint_precopy_begin(img)
    i, _ = s.alloc(workloads.DEVICE, 3 * MIB)
    s.fill_synthetic(i, 4)
    st = s.checkpoint_precopy_finish()
    assert st["incremental"] == 0
    assert img.tobytes() == s.checkpoint()[0]
    # pinned / managed allocations: begin drains synchronously, like the reference
    s2 = eng.Session(seed=2, arena_bytes=1 << 22)
    r2 = ref.RefSession(seed=2, arena_bytes=1 << 22)
    for api in (s2, r2):
        workloads.drive_small(api, seed=8)
    img2 = eng.Image()
    s2.checkpoint_precopy_begin(img2)
    s2.checkpoint_precopy_finish()
    assert img2.tobytes() == r2.checkpoint()[0]


def test_async_drain_matches_reference_small(eng):
    s = eng.Session(seed=2, arena_bytes=1 << 22)
    r = ref.RefSession(seed=2, arena_bytes=1 << 22)
    for api in (s, r):
        workloads.drive_small(api, seed=3)
    s.reserve_shadow(64 * MIB)
    img = eng.Image()
    s.checkpoint_begin(img)
    s.copy_h2d(s.live_records()[0].id, 0, b"\x01" * 16)
    s.checkpoint_finish()
    assert img.tobytes() == r.checkpoint()[0]


def test_async_then_incremental_and_implicit_finish(eng):
    s = eng.Session(seed=1, arena_bytes=256 * MIB)
    workloads.build_regions(s, 5, lambda k: 20 * MIB + k, seed=3)
    s.reserve_shadow(256 * MIB)
    img = eng.Image()
    s.checkpoint_begin(img)
    # any other drain finishes the pending one first
    s.mutate(seed=5, epoch=1, threshold=1 << 61)  # new content = synth(6)
    st = s.checkpoint_into(img, incremental=True)
    assert st["incremental"] == 1 and 0 < st["dirty_chunks"] < st["total_chunks"]
    assert img.tobytes() == s.checkpoint()[0]
    s.reserve_shadow(0)
    assert s.checkpoint_finish()["total_ms"] == 0  # nothing pending


def test_early_refill_with_address_gaps(eng):
    """The refill's data path runs before the replay when the arena sits at
    its logged VA: every live extent must be mapped up front even when id
    order is not address order (first fit reuses low holes) and extents are
    more than 2 MiB apart."""
    import gc
    gc.collect()  # sessions of earlier tests give the logged VA back
    s = eng.Session(seed=4, arena_bytes=1 << 30)
    at_base = s.fixed_va
    a = [s.alloc(workloads.DEVICE, 40 * MIB)[0] for _ in range(4)]
    for i in a:
        s.fill_synthetic(i, 1)
    s.free(a[0])
    s.free(a[2])
    b, _ = s.alloc(workloads.DEVICE, 3 * MIB)  # lands in the low hole
    s.fill_synthetic(b, 2)
    c, _ = s.alloc(workloads.DEVICE, MIB + 7)
    s.fill_synthetic(c, 3)
    img, _ = s.checkpoint()
    want = _state(s)
    s.close()  # the restart takes the logged VA: Device-only, so the early path
    rs, _ = eng.restart(img)
    assert rs.fixed_va == at_base  # the VA s held comes back: the early path ran
    assert _state(rs) == want
    assert rs.checkpoint()[0] == img


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_mixed_paths_agree(eng, seed):
    """Random Device layouts (sizes from 1 B to 40 MiB, so direct runs, edge
    tiles and small payloads mix), random frees and mutations, then every
    drain flavour on the same state: synchronous (== the reference's bytes),
    incremental, shadow at a random size, pre-copy; each restart reproduces
    the state."""
    rnd = random.Random(seed)
    s = eng.Session(seed=seed, arena_bytes=1 << 30)
    r = ref.RefSession(seed=seed, arena_bytes=1 << 30)
    ids = []
    for k in range(40):
        size = rnd.choice([1, 17, 4096, 65536 * 6 + rnd.randrange(1000), 3 * MIB + rnd.randrange(9999),
                           rnd.randrange(1, 40 * MIB)])
        pair = []
        for api in (s, r):
            i, _ = api.alloc(workloads.DEVICE, size)
            api.fill_synthetic(i, seed * 100 + k)
            pair.append(i)
        ids.append(pair[0])
        if k % 7 == 3:
            victim = ids.pop(rnd.randrange(len(ids)))
            s.free(victim)
            r.free(victim)
    want = r.checkpoint()[0]
    img, _ = s.checkpoint()
    assert img == want
    rs, _ = eng.restart(img)
    assert _state(rs) == _state(s)
    # incremental after a mutation equals a fresh synchronous drain
    image = eng.Image()
    s.checkpoint_into(image)
    s.mutate(seed=seed, epoch=1, threshold=(1 << 64) // 5)
    st = s.checkpoint_into(image, incremental=True)
    assert st["incremental"] == 1
    sync = s.checkpoint()[0]
    assert image.tobytes() == sync
    # shadow drain of a random size, then a pre-copy racing a mutation
    s.reserve_shadow(rnd.choice([0, 64, 128, 512]) * MIB)
    s.checkpoint_begin(image)
    s.checkpoint_finish()
    assert image.tobytes() == sync
    s.reserve_shadow(0)
    s.checkpoint_precopy_begin(image)
    s.mutate(seed=seed, epoch=2, threshold=(1 << 64) // 50)
    s.checkpoint_precopy_finish()
    final = s.checkpoint()[0]
    assert image.tobytes() == final
    rs2, _ = eng.restart(final)
    assert rs2.checkpoint()[0] == final


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_random_managed_and_pinned_paths_agree(eng, seed, tmp_path):
    """Random managed allocations (residence set by random host / device
    touches, long and short host runs, partial last pages), pinned and Device
    payloads between them: synchronous drain == the reference's bytes; the
    restart restores bytes and page flags; a shadow drain at a random size
    with host and device page writes right after begin, and a file round
    trip, agree with the synchronous image."""
    rnd = random.Random(seed)
    s = eng.Session(seed=seed, arena_bytes=512 * MIB)
    r = ref.RefSession(seed=seed, arena_bytes=512 * MIB)
    managed = []
    for k in range(8):
        kind = rnd.choice([workloads.MANAGED, workloads.MANAGED, workloads.PINNED, workloads.DEVICE])
        size = rnd.choice([4096 * rnd.randrange(1, 64) + rnd.randrange(4096), rnd.randrange(1, 24 * MIB)])
        ops = []
        if kind == workloads.MANAGED:
            for _ in range(rnd.randrange(1, 12)):
                off = rnd.randrange(0, size)
                n = min(size - off, rnd.choice([4096, 64 << 10, MIB, 3 * MIB]))
                ops.append((off, n, rnd.choice([workloads.HOST_SIDE, workloads.DEVICE_SIDE])))
        for api in (s, r):
            i, _ = api.alloc(kind, size)
            api.fill_synthetic(i, seed + k, rnd.choice([workloads.DEVICE_SIDE]) if kind == workloads.MANAGED
                               else workloads.DEVICE_SIDE)
            for off, n, side in ops:
                if n > 0:
                    api.page_read(i, off, n, side)
        if kind == workloads.MANAGED:
            managed.append(i)
    want = r.checkpoint()[0]
    img, _ = s.checkpoint()
    assert img == want
    rs, _ = eng.restart(img)
    assert _state(rs) == _state(s)
    assert rs.checkpoint()[0] == img
    # shadow drain with writes racing the shadow D2H
    image = eng.Image()
    s.reserve_shadow(rnd.choice([64, 128, 512]) * MIB)
    s.checkpoint_begin(image)
    if managed:
        m = managed[0]
        s.page_write(m, 0, b"\x33" * 4096, workloads.HOST_SIDE)
        s.page_write(m, 0, b"\x44" * 100, workloads.DEVICE_SIDE)
    s.checkpoint_finish()
    assert image.tobytes() == want
    s.reserve_shadow(0)
    # file round trip of the current state
    now = s.checkpoint()[0]
    p = tmp_path / "m.img"
    s.checkpoint_to_file(p)
    assert p.read_bytes() == now
    back, _, _ = eng.restart_from_file(p)
    assert back.checkpoint()[0] == now


@pytest.mark.parametrize("seed", [21, 22])
def test_random_churn_paths_agree(eng, seed):
    """C2-shaped churn (random 256 B-64 KiB allocations and frees, fill8
    launches on 4 streams): the image equals the reference's; a restart
    (early data path when the VA is free) reproduces it; incremental and
    pre-copy drains after more launches equal the synchronous drain."""
    calls = 1500 + 500 * (seed % 3)
    s = eng.Session(seed=seed, arena_bytes=64 * MIB)
    r = ref.RefSession(seed=seed, arena_bytes=64 * MIB)
    for api in (s, r):
        workloads.build_churn(api, calls, seed)
    img, _ = s.checkpoint()
    assert img == r.checkpoint()[0]
    rs, _ = eng.restart(img)
    assert rs.checkpoint()[0] == img
    image = eng.Image()
    s.checkpoint_into(image)
    s.mutate(seed=seed, epoch=3, threshold=(1 << 64) // 3)
    st = s.checkpoint_into(image, incremental=True)
    assert st["incremental"] == 1
    assert image.tobytes() == s.checkpoint()[0]
    s.checkpoint_precopy_begin(image)
    s.mutate(seed=seed, epoch=4, threshold=(1 << 64) // 7)
    s.checkpoint_precopy_finish()
    assert image.tobytes() == s.checkpoint()[0]


def test_cold_restart_after_dropping_the_arena_cache(eng):
    """A restart after crac_drop_arena_cache maps its physical memory afresh
    (as in a new process) and reproduces the state and the image; so does a
    warm restart that adopts the cached arena."""
    import gc
    gc.collect()
    s = eng.Session(seed=8, arena_bytes=1 << 30)
    ids = [s.alloc(workloads.DEVICE, sz)[0] for sz in (5 * MIB + 3, 64 * 1024, 17, 9 * MIB)]
    for k, i in enumerate(ids):
        s.fill_synthetic(i, 40 + k)
    s.free(ids[1])
    img, _ = s.checkpoint()
    want = _state(s)
    s.close()
    eng.drop_arena_cache()
    cold, _ = eng.restart(img)
    assert _state(cold) == want
    assert cold.checkpoint()[0] == img
    cold.close()  # its arena is cached again: the next restart adopts it
    warm, _ = eng.restart(img)
    assert _state(warm) == want
    assert warm.checkpoint()[0] == img
    warm.close()
    eng.drop_arena_cache()
    eng.drop_arena_cache()  # nothing cached: a no-op


def test_incremental_resends_a_crc_preserving_change(eng):
    """SURVEY §7 hard part 5: the dirty key is (CRC-32, chunk key).  A chunk
    rewritten so its CRC-32 is unchanged is still re-sent; the incremental
    image equals the reference's full image (and the GPU's own full drain)."""
    from dirtykey import forge_crc
    sizes = [(3 << 20) + 4096 * k + 13 * k for k in range(6)]
    s = eng.Session(seed=1, arena_bytes=64 << 20)
    r = ref.RefSession(seed=1, arena_bytes=64 << 20)
    ids = workloads.build_regions(s, 6, lambda k: sizes[k], seed=5)
    assert workloads.build_regions(r, 6, lambda k: sizes[k], seed=5) == ids
    image = eng.Image()
    s.checkpoint_into(image)
    for k, off in ((2, 65536 * 7), (4, 65536 * 48)):  # chunk 48 of region 4 is its ragged last one
        cur = bytearray(s.copy_d2h(ids[k], off, min(65536, sizes[k] - off)))
        target = zlib.crc32(cur)
        cur[10] ^= 0x01
        forge_crc(cur, len(cur) - 9, target)
        for api in (s, r):
            api.copy_h2d(ids[k], off, bytes(cur))
    st = s.checkpoint_into(image, incremental=True)
    assert st["incremental"]
    assert st["dirty_chunks"] == 2
    assert image.tobytes() == r.checkpoint()[0] == s.checkpoint()[0]


def test_split_drain_first_in_a_fresh_process():
    """A split drain begun without stats (checkpoint_begin) and finished with
    them, as the first drain of a process: drain_finish once timed the ring
    windows from events that only a drain with stats creates, so on a fresh
    engine it read handles that were never made (segfault).  Run in its own
    process so no earlier drain has sized the engine's event tables."""
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    for node in ("test_pinned_payloads_move_on_the_host_and_match_reference[all-shadow]",
                 "test_async_drain_with_managed_runs_matches_reference[64]"):
        out = subprocess.run([sys.executable, "-X", "faulthandler", "-m", "pytest", "-x", "-q", "-p",
                              "no:cacheprovider", f"tests/test_gpu_parity.py::{node}"],
                             cwd=root, capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
