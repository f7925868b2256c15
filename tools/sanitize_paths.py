"""Every kernel path of the engine at small sizes, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

  full drain        K1 (paired chains, key lane) + K2a pack + K4 fold
  incremental       K1 split drain (hashers + writer CTAs, inter-CTA queue),
                    then the fused form (CRAC_FORCE_FUSED=1 in a 2nd process)
  stall-reduced     K1 hash+copy (mode 2/3) into the shadow, shadow D2H
  pre-copy          K1 hash+copy into the pinned image, incremental finish
  restart           H2D + k_scatter_records + K1 verify (CRC only, paired),
                    cold: early windows, exact-end direct runs, verify_synth
  deflate           K5 segments + gather
  managed / pinned  UVM page hashing, host-resident pages, pinned payloads

Exits nonzero on any mismatch against a plain full drain.
    compute-sanitizer --tool memcheck python tools/sanitize_paths.py
"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from paper_2008_10596_b200 import engine  # noqa: E402
import workloads  # noqa: E402

MIB = 1 << 20


def device_session(seed):
    s = engine.Session(seed=seed, arena_bytes=64 * MIB)
    # odd sizes: tails, partial chunks, unpaired last chunk, misaligned frames
    workloads.build_regions(s, 7, lambda r: (1 + r) * 300_000 + 17 * r, seed)
    return s


def main():
    s = device_session(1)
    img = engine.Image()
    full = s.checkpoint_into(img)
    ref = img.tobytes()
    # incremental: mutate ~10 % of the chunks on the device, re-drain
    s.mutate(seed=3, epoch=1, threshold=(2**64 - 1) // 10)
    inc = s.checkpoint_into(img, incremental=True)
    want, _ = s.checkpoint()
    assert inc["incremental"] and img.tobytes() == want, "incremental != full"
    # stall-reduced (shadow smaller than the stream: ring + shadow parts)
    s.reserve_shadow(2 * MIB)
    s.checkpoint_begin(img)
    s.checkpoint_finish()
    assert img.tobytes() == want, "begin/finish != full"
    s.reserve_shadow(0)
    # pre-copy
    s.checkpoint_precopy_begin(img)
    s.mutate(seed=4, epoch=2, threshold=(2**64 - 1) // 20)
    s.checkpoint_precopy_finish()
    want2, _ = s.checkpoint()
    assert img.tobytes() == want2, "pre-copy != full"
    # restart: scatter + verify; then the same cold, alone (fixed VA: the
    # early ring windows, exact-end direct runs, threaded map and replay)
    r, _ = engine.restart(want2)
    assert r.checkpoint()[0] == want2, "restart round trip"
    r.close()
    s.close()
    engine.drop_arena_cache()
    big = engine.Session(seed=8, arena_bytes=256 * MIB)
    workloads.build_regions(big, 5, lambda r: (1 + r) * 8 * MIB, 8)
    bimg, _ = big.checkpoint()
    big.close()
    engine.drop_arena_cache()
    r, _ = engine.restart(bimg)
    assert r.checkpoint()[0] == bimg, "cold restart round trip"
    assert r.verify_synthetic(8)["bad_allocations"] == 0, "verify kernel"
    r.close()
    # K5: the GPU deflate (compressible and incompressible segments)
    z, _ = engine.compress_image_gpu(bimg[: 3 * MIB] + bytes(2 * MIB))
    import zlib
    assert zlib.decompress(z[16:]) == bimg[: 3 * MIB] + bytes(2 * MIB), "deflate"
    # managed (split residence) + pinned payloads + a random session
    m = engine.Session(seed=2, arena_bytes=16 * MIB)
    i, _ = m.alloc(engine.MANAGED, 3 * MIB + 123)
    m.fill_synthetic(i, 2)
    m.page_read(i, MIB, MIB, engine.HOST_SIDE)
    j, _ = m.alloc(engine.PINNED, 700_000)  # >= 256 KiB: moved by host threads
    m.fill_synthetic(j, 2)
    st = m.stream_create()
    for k in range(12):  # small payloads of every kind beside them, some freed
        a, _ = m.alloc(1 + k % 3, 1 + 997 * k)
        if k % 4 == 3:
            m.free(a)
    m.stream_destroy(st)
    mi, _ = m.checkpoint()
    r, _ = engine.restart(mi)
    assert r.checkpoint()[0] == mi, "managed round trip"
    r.close()
    m.close()
    print("sanitize paths ok", len(ref), full["hash_launches"], inc["dirty_chunks"])


if __name__ == "__main__":
    main()
