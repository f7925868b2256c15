"""CPU tier: the parallel image-file writer / reader.

It replaces the reference's whole-buffer ofstream / ifstream
(ref: src/image.cpp:432-451), so the bar is: the file holds exactly the
bytes, for every size and alignment O_DIRECT makes awkward (empty, sub-block,
block-exact, ragged last piece, misaligned source / destination buffers), on
any thread count and piece size; I/O failures raise the reference's codes
(write: InvalidArgument "cannot write"; read: ImageCorrupt "cannot read").
No GPU is involved in this layer.
"""
import os

import pytest

from oracle import ref


@pytest.fixture(scope="module")
def eng():
    from paper_2008_10596_b200 import engine
    if not engine.LIB_PATH.exists():
        from paper_2008_10596_b200 import build
        build.build()
    return engine


SIZES = [0, 1, 4095, 4096, 4097, 65536 * 3 + 17, (1 << 20) + 4096, 5 * (1 << 20) + 123]


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("direct", [True, False])
def test_round_trip_bytes(eng, tmp_path, n, direct):
    data = os.urandom(n)
    p = tmp_path / "img.bin"
    w = eng.write_file(p, data, threads=4, chunk_bytes=1 << 20, direct=direct)
    assert w["bytes"] == n
    assert p.stat().st_size == n
    assert p.read_bytes() == data  # what a plain reader (the reference's ifstream) sees
    for off in (0, 1, 4000):
        got, r = eng.read_file(p, threads=3, chunk_bytes=1 << 20, direct=direct, offset=off)
        assert got == data
        assert r["bytes"] == n


def test_piece_geometry(eng, tmp_path):
    """Many threads over tiny pieces and one thread over one piece agree."""
    data = os.urandom(3 * 65536 + 4096 + 1)
    for threads, chunk in [(16, 4096), (1, 0), (7, 8192), (64, 4096)]:
        p = tmp_path / f"g{threads}_{chunk}.bin"
        eng.write_file(p, data, threads=threads, chunk_bytes=chunk)
        assert p.read_bytes() == data
        assert eng.read_file(p, threads=threads, chunk_bytes=chunk)[0] == data


def test_misaligned_source_goes_through_bounce(eng, tmp_path):
    raw = bytearray(os.urandom(2 * (1 << 20) + 4096 + 3))
    view = memoryview(raw)[3:]  # bytearray storage is not 4 KiB aligned anyway
    p = tmp_path / "m.bin"
    w = eng.write_file(p, view, threads=2, chunk_bytes=1 << 20)
    assert p.read_bytes() == bytes(view)
    if w["direct"]:
        assert w["bounced"] == len(view)


def test_truncates_a_longer_existing_file(eng, tmp_path):
    p = tmp_path / "t.bin"
    p.write_bytes(b"x" * 100000)
    eng.write_file(p, b"abc")
    assert p.read_bytes() == b"abc"


def test_golden_images_round_trip(eng, tmp_path, golden):
    _, images = golden
    for name, img in images.items():
        p = tmp_path / f"{name}.img"
        eng.write_file(p, img)
        assert p.read_bytes() == img
        ref.ref_decode_check(eng.read_file(p)[0])  # the reference decoder accepts it


def test_missing_file_is_image_corrupt(eng, tmp_path):
    with pytest.raises(eng.CracError) as e:
        eng.read_file(tmp_path / "nope.img")
    assert e.value.errc == "ImageCorrupt"
    with pytest.raises(eng.CracError) as e:
        eng.read_file(tmp_path)  # a directory is not an image
    assert e.value.errc == "ImageCorrupt"


def test_unwritable_path_is_invalid_argument(eng, tmp_path):
    with pytest.raises(eng.CracError) as e:
        eng.write_file(tmp_path / "no" / "such" / "dir" / "x.img", b"1234")
    assert e.value.errc == "InvalidArgument"
    assert "cannot write" in str(e.value)
