"""CPU tier: the dirty-key helpers (tests/dirtykey.py) on their own."""
import os
import random
import zlib

from dirtykey import chunk_key, chunk_keys, forge_crc


def test_forged_change_keeps_the_crc_but_not_the_key():
    rng = random.Random(3)
    for n in (64, 4096, 65536, 65536 - 13):
        data = bytearray(os.urandom(n))
        crc, key = zlib.crc32(data), chunk_key(data)
        p = rng.randrange(n)
        data[p] ^= 0x5A
        q = (p + 100) % (n - 4)
        forge_crc(data, q, crc)
        assert zlib.crc32(data) == crc  # a CRC-only dirty check misses this change
        assert chunk_key(data) != key


def test_chunk_key_is_position_and_length_sensitive():
    a = bytes(range(256)) * 256
    b = a[16:32] + a[:16] + a[32:]  # two 16-byte words swapped
    assert chunk_key(a) != chunk_key(b)
    assert chunk_key(a[:100]) != chunk_key(a[:100] + b"\0")  # zero padding vs length
    assert chunk_keys(a, 4096) == [chunk_key(a[i:i + 4096]) for i in range(0, len(a), 4096)]
    assert chunk_key(b"") == chunk_key(bytes(0))
