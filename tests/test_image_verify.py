"""CPU tier: crac_image_verify, the host-only check the bench runs on its images.

It must agree with the reference on what a valid image is (every golden image
passes), recompute every section CRC itself, and find payload bytes that
differ from the synthetic content f(seed, id, offset) of fill_synthetic even
when the image's own CRCs were recomputed to match (the case a K1-vs-K1 check
cannot see).
"""
import struct
import zlib
from pathlib import Path

import pytest

from oracle import ref

GOLDEN = Path(__file__).resolve().parent / "golden"
MIB = 1 << 20


@pytest.fixture(scope="module")
def eng():
    from paper_2008_10596_b200 import engine
    if not engine.LIB_PATH.exists():
        from paper_2008_10596_b200 import build
        build.build()
    return engine


def _sections(img):
    out, at = [], 16
    for _ in range(7):
        n = struct.unpack_from("<Q", img, at + 8)[0]
        out.append((at + 16, n))
        at += 20 + n
    return out


def _synthetic_image(sizes, seed):
    r = ref.RefSession(seed=seed, arena_bytes=(sum(s + 256 for s in sizes) // MIB + 2) * MIB)
    for sz in sizes:
        i, _ = r.alloc(1, sz)
        r.fill_synthetic(i, seed)
    img, _ = r.checkpoint()
    r.close()
    return img


@pytest.mark.parametrize("name", sorted(p.name for p in GOLDEN.glob("*.bin")))
def test_golden_images_pass(eng, name):
    img = (GOLDEN / name).read_bytes()
    rep = eng.verify_image(img, threads=4)
    assert rep["ok"] and rep["sections_checked"] == 7
    assert rep["crc_bytes"] == sum(n for _, n in _sections(img))


def test_synthetic_payloads_match_and_wrong_seed_does_not(eng):
    sizes = [3 * MIB + 5, 64 * 1024, 17, 2 * MIB, 1]
    img = _synthetic_image(sizes, seed=3)
    rep = eng.verify_image(img, synth_seed=3, threads=3)
    assert rep["ok"], rep
    assert rep["payloads_compared"] == len(sizes)
    assert rep["payload_bytes_compared"] == sum(sizes)
    bad = eng.verify_image(img, synth_seed=4, threads=3)
    assert bad["mismatched_payloads"] == len(sizes) and bad["bad_sections"] == 0


@pytest.mark.parametrize("where", [0, 8, 1 << 20, 3 * MIB + 4])
def test_a_changed_payload_byte_is_found_even_with_recomputed_crcs(eng, where):
    sizes = [3 * MIB + 5, 2 * MIB]
    img = bytearray(_synthetic_image(sizes, seed=7))
    off3, n3 = _sections(img)[2]
    at = off3 + 16 + where  # first payload's data starts after its 16-byte frame
    img[at] ^= 0x40
    rep = eng.verify_image(bytes(img), synth_seed=7)
    assert rep["bad_sections"] == 1 << 2 and rep["mismatched_payloads"] == 1
    assert rep["first_bad_id"] == 1
    # re-stamp the section CRC: the image is self-consistent, the content is not
    struct.pack_into("<I", img, off3 + n3, zlib.crc32(img[off3:off3 + n3]))
    ref.ref_decode_check(bytes(img))  # the reference accepts it
    rep = eng.verify_image(bytes(img), synth_seed=7)
    assert rep["bad_sections"] == 0 and rep["mismatched_payloads"] == 1 and not rep["ok"]


def test_a_stored_crc_flip_is_found(eng):
    img = bytearray((GOLDEN / "rich.bin").read_bytes())
    for s, (off, n) in enumerate(_sections(img)):
        bad = bytearray(img)
        bad[off + n] ^= 1
        with pytest.raises(eng.CracError) as e:  # small sections: the strict parse refuses
            rep = eng.verify_image(bytes(bad))
            assert rep["bad_sections"] == 1 << s  # bulk sections: found by the recompute
            raise eng.CracError(15, "found")
        assert e.value.rc in (14, 15)


def test_framing_errors_are_refused(eng):
    with pytest.raises(eng.CracError) as e:
        eng.verify_image(b"CRACSIM1" + bytes(8))
    assert e.value.errc == "ImageCorrupt"
