"""GPU tier: K5, the GPU deflate behind CRACSIMZ.

The reference's compressed bytes are zlib compress2 level 6
(/root/reference/proj/src/image.cpp:419-430); its reader
(maybe_decompress, :347-379) accepts any zlib stream that inflates to exactly
the declared length.  So the bar is: every GPU-compressed wrapper inflates
(stock zlib, and the unmodified reference's restart_from_file) to the exact
image, compresses what is compressible, and never grows more than 5 bytes
per 32 KiB segment.
"""
import os
import struct
import zlib

import pytest

import workloads
from oracle import ref

pytestmark = pytest.mark.gpu

SEG = 32768


def _inflate(z: bytes) -> bytes:
    assert z[:8] == b"CRACSIMZ"
    raw_len = struct.unpack_from("<Q", z, 8)[0]
    out = zlib.decompress(z[16:])  # checks the zlib header and the Adler-32
    assert len(out) == raw_len
    return out


@pytest.mark.parametrize("n", [0, 1, 2, 3, 100, SEG - 1, SEG, SEG + 1, 5 * SEG + 777, 3 << 20])
@pytest.mark.parametrize("kind", ["random", "zeros", "pattern", "text"])
def test_gpu_deflate_inflates_to_the_input(eng, n, kind):
    if kind == "random":
        data = os.urandom(n)
    elif kind == "zeros":
        data = bytes(n)
    elif kind == "pattern":
        data = (bytes(range(251)) * (n // 251 + 1))[:n]
    else:
        words = [b"checkpoint", b"restart", b"drain", b"refill", b"B200", b"CRAC", b" ", b"\n"]
        rnd = os.urandom(n)
        data = b"".join(words[b % 8] for b in rnd)[:n]
    z, ms = eng.compress_image_gpu(data)
    assert _inflate(z) == data
    segs = max(1, (n + SEG - 1) // SEG)
    assert len(z) <= 16 + 2 + n + 5 * segs + 4  # stored fallback bounds the growth
    if kind in ("zeros", "pattern") and n >= SEG:
        assert len(z) < n // 10
    if kind == "text" and n >= SEG:
        assert len(z) < n * 0.8


def test_gpu_deflate_across_batches(eng):
    """An input longer than one 1 GiB device batch: the Adler-32 fold and the
    BFINAL marker cross the batch boundary."""
    n = (1 << 30) + 3 * SEG + 5
    data = bytearray(n)
    data[::4096] = os.urandom(len(data[::4096]))
    data = bytes(data)
    z, _ = eng.compress_image_gpu(data)
    assert zlib.decompress(z[16:]) == data


def test_gpu_compressed_files_restart_on_both_sides(eng, tmp_path):
    s = eng.Session(seed=3, arena_bytes=64 << 20)
    workloads.drive_small(s, seed=4)
    workloads.build_regions(s, 3, lambda r: (1 << 20) + 17 * r, seed=3)
    i, _ = s.alloc(workloads.DEVICE, 3 << 20)  # zeros: compressible
    want, _ = s.checkpoint()
    p = tmp_path / "gpu.img"
    s.checkpoint_to_file(p, compress="gpu")
    z = p.read_bytes()
    assert _inflate(z) == want
    assert len(z) < len(want)
    # the unmodified reference reads the GPU-compressed file
    rr, _ = ref.ref_restart_from_file(p)
    assert rr.checkpoint()[0] == want
    rr.close()
    r, _, _ = eng.restart_from_file(p)
    assert r.checkpoint()[0] == want
    r.close()
    s.close()
