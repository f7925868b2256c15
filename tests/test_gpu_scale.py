"""GPU tier, BASELINE sizes: parity pinned at the configs the bench runs.

* C1 exactly as BASELINE.json configs[0] states it: 256 x 4 MiB Device
  regions (1 GiB), full checkpoint -> restart round trip, the GPU image
  compared byte for byte with the unmodified reference's `encode_image`
  (oracle/_ref) for the same call sequence, plus the odd-size variant
  (4 MiB - r%3) of SURVEY Appendix A.
* C2 at the bench's 40 k calls (alloc_churn shape, 4 streams) against the
  reference.
* Images the reference's own arena check lets through but whose payloads
  cannot exist are refused by the restart before anything is indexed by
  them (drain.cu premap).
"""
import struct
import zlib

import pytest

import workloads
from oracle import ref
from oracle.image_oracle import K_ARENA_BASE, MAGIC

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

MIB = 1 << 20


def _sections(img: bytes) -> list[tuple[int, int, int]]:
    """(payload offset, length, stored crc) of the 7 sections."""
    out, at = [], 16
    for _ in range(7):
        n = struct.unpack_from("<Q", img, at + 8)[0]
        out.append((at + 16, n, struct.unpack_from("<I", img, at + 16 + n)[0]))
        at += 20 + n
    return out


@pytest.mark.parametrize("odd", [False, True], ids=["4MiB", "4MiB-r%3"])
def test_c1_full_size_matches_reference(eng, odd):
    n = 256
    size = (lambda r: 4 * MIB - r % 3) if odd else (lambda r: 4 * MIB)
    arena = n * 4 * MIB + MIB
    s = eng.Session(seed=1, arena_bytes=arena)
    r = ref.RefSession(seed=1, arena_bytes=arena)
    for api in (s, r):
        workloads.build_regions(api, n, size, seed=1)
    img, st = s.checkpoint()
    want, _ = r.checkpoint()
    assert len(img) == len(want)
    assert img == want
    secs = _sections(img)
    # ALLOC_PAYLOADS at 96 + 36 * n_log, Σ(16 + size) long
    assert secs[2][0] == 96 + 36 * n
    assert secs[2][1] == sum(16 + size(k) for k in range(n))
    if odd:
        assert secs[2][1] == 1_073_745_665
    else:
        assert len(img) == 1_073_755_324  # SURVEY Appendix A, C1 probe image size
    assert secs[2][2] == zlib.crc32(memoryview(img)[secs[2][0]:secs[2][0] + secs[2][1]])
    assert st["d2h_bytes"] == secs[2][1] + 20
    # round trip: restart from the GPU image, checkpoint again, same bytes;
    # the reference restarts from the GPU image too
    s.close()
    rs, rst = eng.restart(img)
    assert rs.checkpoint()[0] == img
    rs.close()
    rr, _ = ref.ref_restart(img)
    assert rr.checkpoint()[0] == img
    rr.close()
    r.close()


def test_c2_at_bench_size_matches_reference(eng):
    """The bench's C2 shape (40 k calls, 4 streams, 256 B..64 KiB) against
    the reference, then restart(checkpoint) == checkpoint."""
    s = eng.Session(seed=1, arena_bytes=2 << 30)
    r = ref.RefSession(seed=1, arena_bytes=2 << 30)
    for api in (s, r):
        workloads.build_churn(api, 40000, seed=1)
    img, st = s.checkpoint()
    want, _ = r.checkpoint()
    assert img == want
    assert len(s.live_records()) > 15000
    s.close()
    rs, _ = eng.restart(img)
    assert rs.checkpoint()[0] == img
    rs.close()
    r.close()


def _image(kind: int, size: int, pay: bytes, uvm: bytes, free: bool = False) -> bytes:
    log = struct.pack("<QBBHQQQ", 1, 1, kind, 0, size, 1, K_ARENA_BASE)
    if free:
        log += struct.pack("<QBBHQQQ", 2, 2, 0, 0, 0, 1, 0)
    secs = [struct.pack("<QQII", 0, 1 << 24, 1, 0), log, pay, uvm, b"", b"",
            struct.pack("<Q", 0)]
    img = bytearray(MAGIC + struct.pack("<II", 1, 7))
    for tag, p in enumerate(secs, start=1):
        img += struct.pack("<IIQ", tag, 0, len(p)) + p + struct.pack("<I", zlib.crc32(p))
    return bytes(img)


@pytest.mark.parametrize("kind,size,pay,uvm", [
    (1, (1 << 64) - 1, b"\0" * 15, b""),
    (1, (1 << 64) - 17, b"\0" * 32, b""),
    (3, (1 << 64) - 1, b"", b"\0" * 40),
])
def test_restart_refuses_wrapping_sizes(eng, kind, size, pay, uvm):
    img = _image(kind, size, pay, uvm)
    with pytest.raises(ref.RefError) as r:
        ref.ref_decode_check(img)
    assert r.value.errc == "ImageCorrupt"
    with pytest.raises(eng.CracError) as e:
        eng.restart(img)
    assert e.value.errc == "ImageCorrupt"


def test_restart_checked_against_regenerated_content(eng):
    """The bench's independent checks (crac_image_verify on the host image,
    verify_synthetic on the restarted device state) agree with a clean round
    trip, and catch a payload change whose section CRC was re-stamped (the
    image is self-consistent, so the refill's K1 verify accepts it)."""
    n, size = 24, 4 * MIB + 48
    s = eng.Session(seed=1, arena_bytes=n * (size + 256) // MIB * MIB + 2 * MIB)
    workloads.build_regions(s, n, lambda r: size, seed=1)
    img, _ = s.checkpoint()
    s.close()
    eng.drop_arena_cache()  # cold: the restart maps fresh physical memory
    rep = eng.verify_image(img, synth_seed=1)
    assert rep["ok"] and rep["payloads_compared"] == n
    rs, _ = eng.restart(img)
    v = rs.verify_synthetic(1)
    assert v == {"bad_allocations": 0, "bytes_checked": n * size}
    rs.close()
    bad = bytearray(img)
    off3, n3, _ = _sections(img)[2]
    bad[off3 + 16 + (n // 2) * (16 + size) + 12345] ^= 0x10
    struct.pack_into("<I", bad, off3 + n3, zlib.crc32(memoryview(bad)[off3:off3 + n3]))
    rep = eng.verify_image(bytes(bad), synth_seed=1)
    assert rep["bad_sections"] == 0 and rep["mismatched_payloads"] == 1
    eng.drop_arena_cache()
    rs, _ = eng.restart(bytes(bad))
    assert rs.verify_synthetic(1)["bad_allocations"] == 1
    rs.close()


def test_cold_restart_two_handle_map_after_async_release(eng):
    """A cold restart of an arena bigger than half the GPU right after
    drop_arena_cache(release_later=True): the refill maps its head before the
    copies and the tail on a thread that must wait for the old arena's
    release (the two cannot coexist in HBM).  The restarted state equals the
    regenerated content, twice over, and a synchronous drop still works."""
    import torch
    free, total = torch.cuda.mem_get_info()
    n = int(total * 0.55) >> 30  # 1 GiB regions: arena > half of HBM
    s = eng.Session(seed=5, arena_bytes=(n << 30) + n * (4 << 20))
    workloads.build_regions(s, n, lambda r: (1 << 30) - 4096 * (r % 3), seed=5)
    image = eng.Image()
    try:
        for rep in range(2):
            s.checkpoint_into(image)
            s.close()
            eng.drop_arena_cache(release_later=True)
            addr, size = image.address()
            s, st = eng.restart_from_address(addr, size)
            v = s.verify_synthetic(5)
            assert v["bad_allocations"] == 0 and v["bytes_checked"] > (n - 1) << 30, (rep, v)
        s.close()
        eng.drop_arena_cache()  # waits for nothing in flight; frees the cached arena
    finally:
        image.close()
