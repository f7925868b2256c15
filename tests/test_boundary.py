"""CPU tier: the drop-in boundary.

* libcrac_b200.so loads and exports exactly what include/*.h declares;
* with no GPU the engine refuses loudly (DeviceFault), never a CPU fallback;
* the host-side codec behind the C-ABI (strict decode, summarize) agrees with
  the reference on every golden image and rejects corrupted ones.
"""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared(header: str) -> set[str]:
    text = (ROOT / "include" / header).read_text()
    return set(re.findall(r"^\s*(?:int|void|uint32_t|uint64_t|const char\*)\s+(crac_\w+)\s*\(", text, re.M))


@pytest.fixture(scope="module")
def so():
    from paper_2008_10596_b200 import engine
    if not engine.LIB_PATH.exists():
        from paper_2008_10596_b200 import build
        build.build()
    return engine


def test_library_exports_every_declared_symbol(so):
    lib = ctypes.CDLL(str(so.LIB_PATH))
    names = declared("crac_engine.h") | declared("crac_gpu.h")
    assert len(names) >= 40
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    # the Python mirror binds every declared entry point with a signature
    assert names == set(so.exported_symbols())


def test_no_cpu_fallback_without_gpu(so):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(so.CracError) as e:
        so.Session(seed=1, arena_bytes=1 << 20)
    assert e.value.errc == "DeviceFault"


@pytest.mark.parametrize("name", ["empty", "rich", "small_session", "c1_mini", "random_300"])
def test_host_codec_accepts_reference_images(so, golden, name):
    manifest, images = golden
    so.decode_check(images[name])
    summ = so.summarize_image(images[name])
    assert summ["lengths"] == manifest[name]["lengths"]
    assert [f"{c:08x}" for c in summ["crcs"]] == manifest[name]["crcs"]
    assert summ["file_bytes"] == len(images[name])


def test_host_codec_rejects_every_bit_flip(so, golden):
    _, images = golden
    img = bytearray(images["rich"])
    for bit in range(len(img) * 8):
        img[bit // 8] ^= 1 << (bit % 8)
        with pytest.raises(so.CracError) as e:
            so.decode_check(bytes(img))
        assert e.value.errc == "ImageCorrupt"
        img[bit // 8] ^= 1 << (bit % 8)


def test_host_codec_rejects_truncation_and_trailing(so, golden):
    _, images = golden
    b = images["small_session"]
    for keep in (0, 7, 15, 16, 50, len(b) - 1):
        with pytest.raises(so.CracError):
            so.decode_check(b[:keep])
    with pytest.raises(so.CracError):
        so.decode_check(b + b"\0")


def test_preload_exports_its_api_and_interposers(so):
    """libcrac_preload.so exports every crac_preload.h entry
    point and the cudart calls it interposes; it links the engine library."""
    import subprocess
    pre = so.LIB_PATH.parent / "libcrac_preload.so"
    if not pre.exists():
        from paper_2008_10596_b200 import build
        build.build()
    text = (ROOT / "include" / "crac_preload.h").read_text()
    api = set(re.findall(r"^\s*(?:int|void\*)\s+(crac_preload_\w+)\s*\(", text, re.M))
    assert len(api) == 6
    out = subprocess.run(["nm", "-D", "--defined-only", str(pre)], capture_output=True,
                         text=True, check=True).stdout
    syms = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    interposed = {"cudaMalloc", "cudaMallocManaged", "cudaMallocHost", "cudaHostAlloc",
                  "cudaFree", "cudaFreeHost", "cudaStreamCreate", "cudaStreamCreateWithFlags",
                  "cudaStreamCreateWithPriority", "cudaStreamDestroy", "cudaLaunchKernel",
                  "cudaMemcpy", "cudaMemcpyAsync", "cudaMemset", "cudaMemsetAsync",
                  "cudaLaunchKernelExC", "cudaLaunchCooperativeKernel", "cudaGraphLaunch",
                  "cudaMemcpy2D", "cudaMemcpy2DAsync", "cudaMemcpy3D", "cudaMemcpy3DAsync",
                  "cudaMemcpyPeer", "cudaMemcpyPeerAsync", "cudaMemcpyToSymbol",
                  "cudaMemcpyToSymbolAsync", "cudaMemcpyFromSymbol", "cudaMemcpyFromSymbolAsync",
                  "cudaMemset2D", "cudaMemset2DAsync", "cudaMemset3D", "cudaMemset3DAsync"}
    assert api | interposed <= syms, sorted((api | interposed) - syms)
    # the engine library itself must not export cuda* (its static runtime
    # would otherwise be interposed by the preload)
    eng = subprocess.run(["nm", "-D", "--defined-only", str(so.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    assert not [ln for ln in eng.splitlines() if " T cuda" in ln]
    needed = subprocess.run(["readelf", "-d", str(pre)], capture_output=True, text=True).stdout
    assert "libcrac_b200.so" in needed


def test_host_codec_payload_frames_match_reference(so):
    """ALLOC_PAYLOADS frames are validated at offsets computed from the log
    (parse_payload_frames' fast path).  Frames tampered so that only the frame
    check can catch them (the section CRC re-sealed) are rejected exactly when
    the reference's sequential walk rejects them (ref: image.cpp:175-197)."""
    import random
    import struct
    import sys
    import zlib
    sys.path.insert(0, str(ROOT))
    from oracle import ref
    s = ref.RefSession(seed=3, arena_bytes=1 << 26)
    rng = random.Random(5)
    ids = []
    for k in range(60):
        if ids and rng.random() < 0.3:
            s.free(ids.pop(rng.randrange(len(ids))))
        else:
            i, _ = s.alloc(1, 256 * (1 + rng.randrange(16)))
            ids.append(i)
    img, _ = s.checkpoint()
    so.decode_check(img)
    ref.ref_decode_check(img)
    # section 3 (ALLOC_PAYLOADS): walk to it, then list its frames
    at = 16
    for _ in range(2):
        at += 20 + struct.unpack_from("<Q", img, at + 8)[0]
    s3, l3 = at + 16, struct.unpack_from("<Q", img, at + 8)[0]
    frames, p = [], s3
    while p < s3 + l3:
        frames.append(p)
        p += 16 + struct.unpack_from("<Q", img, p + 8)[0]
    assert len(frames) >= 20

    def seal(b):
        struct.pack_into("<I", b, s3 + l3, zlib.crc32(bytes(b[s3:s3 + l3])))
        return bytes(b)

    cases = []
    for f in (frames[0], frames[len(frames) // 2], frames[-1]):
        for field, delta in ((0, 1), (0, -1), (8, 256), (8, -256), (8, 1)):
            b = bytearray(img)
            v = struct.unpack_from("<Q", b, f + field)[0]
            struct.pack_into("<Q", b, f + field, (v + delta) % (1 << 64))
            cases.append(seal(b))
    # two frames swapped (same total length)
    b = bytearray(img)
    a0, a1 = frames[1], frames[2]
    b[a0:a0 + 16], b[a1:a1 + 16] = img[a1:a1 + 16], img[a0:a0 + 16]
    cases.append(seal(b))
    for c in cases:
        try:
            ref.ref_decode_check(c)
            ref_ok = True
        except ref.RefError:
            ref_ok = False
        try:
            so.decode_check(c)
            ours_ok = True
        except so.CracError as e:
            assert e.errc == "ImageCorrupt"
            ours_ok = False
        assert ours_ok == ref_ok
        assert not ours_ok


@pytest.mark.parametrize("kind,size,pay,uvm", [
    # one Device alloc of 2^64-1 at the arena base, a 15-byte ALLOC_PAYLOADS
    # (16 + size wraps to 15): the advisor's reproduction
    (1, (1 << 64) - 1, b"\0" * 15, b""),
    (1, (1 << 64) - 17, b"\0" * 32, b""),
    # the same through the managed prefix sums
    (3, (1 << 64) - 1, b"", b"\0" * 40),
    (3, (1 << 64) - 4096, b"", b"\0" * 64),
])
def test_host_codec_rejects_wrapping_logged_sizes(so, kind, size, pay, uvm):
    """A logged size near 2^64 passes the reference's own arena check
    (round_up_align wraps to 0, ref: image.cpp:133-135) but can never have a
    payload frame: the reference rejects such an image in its bounds-checked
    walk; ours must raise ImageCorrupt too (all CRCs valid), never read past
    the section (image.cpp:185, drain.cu:1506)."""
    import struct
    import sys
    import zlib
    sys.path.insert(0, str(ROOT))
    from oracle import ref
    from oracle.image_oracle import K_ARENA_BASE, MAGIC
    secs = [struct.pack("<QQII", 0, 1 << 24, 1, 0),
            struct.pack("<QBBHQQQ", 1, 1, kind, 0, size, 1, K_ARENA_BASE),
            pay, uvm, b"", b"", struct.pack("<Q", 0)]
    img = bytearray(MAGIC + struct.pack("<II", 1, 7))
    for tag, p in enumerate(secs, start=1):
        img += struct.pack("<IIQ", tag, 0, len(p)) + p + struct.pack("<I", zlib.crc32(p))
    img = bytes(img)
    with pytest.raises(ref.RefError) as r:
        ref.ref_decode_check(img)
    assert r.value.errc == "ImageCorrupt"
    for call in (so.decode_check, so.summarize_image):
        with pytest.raises(so.CracError) as e:
            call(img)
        assert e.value.errc == "ImageCorrupt"
