"""CPU tier: pins the oracle before anything is checked against it.

* the C restatement of CRC-32 against its published known answers and against
  Python's zlib (the library the reference links, image.cpp:3);
* the Python image restatement against the golden images the reference
  library produced (tests/golden, oracle/make_golden.py);
* the reference library (oracle/_ref) against the same goldens and against
  the reference's own fixture facts (test_image.cpp:67-124).
"""
import os
import random
import zlib

import pytest

from oracle import image_oracle as io
from oracle import ref


def test_crc_known_answers(golden):
    manifest, _ = golden
    assert ref.crc32(b"123456789") == 0xCBF43926
    assert ref.crc32_bitwise(b"123456789") == 0xCBF43926
    assert ref.crc32(b"") == 0
    assert manifest["crc_known_answers"] == {"123456789": "cbf43926", "": "00000000"}


@pytest.mark.parametrize("n", [0, 1, 3, 7, 8, 9, 15, 16, 17, 255, 511, 512, 513, 4096, 65537])
def test_crc_matches_zlib(n):
    b = os.urandom(n)
    assert ref.crc32(b) == zlib.crc32(b) == ref.crc32_bitwise(b)


def test_crc_combine_matches_concatenation():
    rnd = random.Random(5)
    for _ in range(50):
        a = os.urandom(rnd.randrange(0, 3000))
        b = os.urandom(rnd.randrange(0, 3000))
        assert ref.crc32_combine(zlib.crc32(a), zlib.crc32(b), len(b)) == zlib.crc32(a + b)


def test_chunk_crc_threads_agree():
    b = os.urandom(3 * 65536 + 1234)
    one = ref.chunk_crc32(b, 65536, threads=1)
    many = ref.chunk_crc32(b, 65536, threads=4)
    assert one == many == [zlib.crc32(b[i:i + 65536]) for i in range(0, len(b), 65536)]


def test_python_restatement_encodes_reference_fixtures(golden):
    _, images = golden
    assert io.encode_image(io.empty_snapshot()) == images["empty"]
    assert io.encode_image(io.rich_snapshot()) == images["rich"]
    assert len(images["empty"]) == 188  # test_image.cpp:67-89


def test_fixture_section_facts(golden):
    manifest, _ = golden
    # test_image.cpp:91-113 and SURVEY Appendix A (derived from the oracle)
    assert manifest["rich"]["lengths"] == [24, 324, 1042, 4244, 8, 33, 54]
    assert manifest["rich"]["crcs"] == ["e1fa0daa", "a343fe2c", "9ceee642", "b5ba634e",
                                        "2707d814", "fb4a1fc4", "d1a48f24"]
    assert manifest["empty"]["crcs"] == ["b2fd133b"] + ["00000000"] * 5 + ["6522df69"]


@pytest.mark.parametrize("name", ["empty", "rich", "small_session", "c1_mini", "random_300"])
def test_restatement_round_trips_goldens(golden, name):
    _, images = golden
    snap = io.decode_image(images[name])
    assert io.encode_image(snap) == images[name]
    assert ref.ref_summarize(images[name])["file_bytes"] == len(images[name])


def test_every_bit_flip_is_corrupt_in_both_oracles(golden):
    _, images = golden
    img = bytearray(images["rich"])
    for bit in range(0, len(img) * 8, 7):  # every 7th bit in Python, all bits below in C
        img[bit // 8] ^= 1 << (bit % 8)
        with pytest.raises(io.ImageCorrupt):
            io.decode_image(bytes(img))
        img[bit // 8] ^= 1 << (bit % 8)
    for bit in range(len(img) * 8):  # test_image.cpp:126-142, exhaustively
        img[bit // 8] ^= 1 << (bit % 8)
        with pytest.raises(ref.RefError) as e:
            ref.ref_decode_check(bytes(img))
        assert e.value.errc == "ImageCorrupt"
        img[bit // 8] ^= 1 << (bit % 8)


def test_truncation_and_trailing_bytes(golden):
    _, images = golden
    b = images["rich"]
    for keep in (0, 7, 15, 16, 50, len(b) - 1):  # test_image.cpp:166-175
        with pytest.raises(io.ImageCorrupt):
            io.decode_image(b[:keep])
    with pytest.raises(io.ImageCorrupt):
        io.decode_image(b + b"\0")


def test_reference_library_reproduces_goldens(golden):
    import workloads
    _, images = golden
    s = ref.RefSession(seed=3, arena_bytes=1 << 22)
    workloads.drive_small(s, seed=1)
    assert s.checkpoint()[0] == images["small_session"]
    s = ref.RefSession(seed=7, arena_bytes=1 << 20)
    workloads.drive_random(s, seed=42, ops=300, arena=1 << 20)
    assert s.checkpoint()[0] == images["random_300"]


def test_first_fit_restatement_matches_reference_addresses():
    # test_device_core.cpp:119-152 shape: random alloc/free vs a naive oracle
    rnd = random.Random(11)
    for round_ in range(20):
        s = ref.RefSession(seed=round_, arena_bytes=1 << 20)
        ff = io.FirstFit(1 << 20)
        live = []
        for _ in range(200):
            if live and rnd.random() < 0.4:
                i, addr = live.pop(rnd.randrange(len(live)))
                s.free(i)
                ff.free(addr)
            else:
                size = 1 + rnd.randrange(20000)
                want = ff.alloc(size)
                try:
                    i, addr = s.alloc(1, size)
                except ref.RefError as e:
                    assert e.errc == "OutOfArena" and want is None
                    continue
                assert addr == want
                live.append((i, addr))


def test_synth_content_matches_reference_fill():
    s = ref.RefSession(seed=1, arena_bytes=1 << 20)
    i, _ = s.alloc(1, 1001)
    s.fill_synthetic(i, 9)
    assert s.copy_d2h(i, 0, 1001) == ref.synth_bytes(9, i, 1001)
