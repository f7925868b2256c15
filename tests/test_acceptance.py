"""CPU tier: the reference's acceptance criterion 8 (image robustness),
restated against the B200 build's strict decode.

/root/reference/proj/tests/acceptance/acceptance_main.cpp:379-415: 500 random
sessions (SequenceDriver with stamped contents, 20..79 calls, app state of
0..127 bytes, 1 MiB arena), each image round-trips, and 1000 random single-bit
flips per image all raise ImageCorrupt.  Here the images come from the
unmodified reference (oracle/_ref) and every flip goes through
crac_decode_check, the host half of the restart (its GPU half, the bulk CRC
verify, is exercised by tests/test_gpu_parity.py's restart bit flips).
"""
import random

import pytest

import workloads
from oracle import ref

MIB = 1 << 20


@pytest.fixture(scope="module")
def eng():
    from paper_2008_10596_b200 import engine
    if not engine.LIB_PATH.exists():
        from paper_2008_10596_b200 import build
        build.build()
    return engine


def test_criterion_8_every_single_bit_flip_is_refused(eng):
    rng = random.Random(808)
    snapshots = flips = 0
    for rnd in range(500):
        s = ref.RefSession(seed=rnd, arena_bytes=MIB)
        workloads.drive_random(s, seed=rng.randrange(1 << 62), ops=20 + rng.randrange(60),
                               arena=MIB, stamp=True)
        s.set_app_state(bytes([rnd & 0xFF]) * rng.randrange(128))
        img, _ = s.checkpoint()
        s.close()
        eng.decode_check(img)  # the clean image decodes
        buf = bytearray(img)
        for _ in range(1000):
            bit = rng.randrange(len(buf) * 8)
            buf[bit // 8] ^= 1 << (bit % 8)
            with pytest.raises(eng.CracError) as e:
                eng.decode_check(bytes(buf))
            assert e.value.errc == "ImageCorrupt", (rnd, bit)
            buf[bit // 8] ^= 1 << (bit % 8)
            flips += 1
        snapshots += 1
    assert snapshots == 500 and flips == 500_000
