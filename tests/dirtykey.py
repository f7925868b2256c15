"""Test helpers for the 64-bit dirty key (CRC-32, chunk key) of the
incremental and pre-copy drains.

* ``chunk_key(data)`` restates the second key lane of K1
  (paper_2008_10596_b200/csrc/kernels.cu "Key2", include/crac_gpu.h
  crac_chunk_key_range) in numpy, so the GPU value is pinned independently of
  the kernel's row batching.
* ``forge_crc(data, at)`` rewrites the 4 bytes at ``at`` so that the CRC-32 of
  ``data`` becomes a chosen value: CRC-32 is affine over GF(2), so any change
  can be compensated by 4 bytes (the collision a CRC-only dirty check misses).
"""
from __future__ import annotations

import zlib

import numpy as np

M32 = 0xFFFFFFFF
M64 = (1 << 64) - 1


def chunk_key(data: bytes) -> int:
    n = len(data)
    words = (n + 15) // 16
    buf = bytes(data) + bytes(words * 16 - n)
    a = np.frombuffer(buf, dtype="<u4").reshape(-1, 4).astype(np.uint64)
    j = np.arange(words, dtype=np.uint64)
    k = ((j & np.uint64(31)) + np.uint64(1)) * np.uint64(0x27D4EB2F) + \
        (j >> np.uint64(5)) * np.uint64(0x9E3779B9)
    k &= np.uint64(M32)
    m32 = np.uint64(M32)
    x, y, z, w = a[:, 0], a[:, 1], a[:, 2], a[:, 3]
    with np.errstate(over="ignore"):
        t = ((x + k) & m32) * ((y + np.uint64(0x85EBCA6B)) & m32) + \
            ((z + (k ^ np.uint64(0xC2B2AE35))) & m32) * ((w + np.uint64(0x165667B1)) & m32)
        s = int(t.sum(dtype=np.uint64)) if words else 0
    x = (s ^ (n * 0x9E3779B97F4A7C15)) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    x ^= x >> 31
    return (x ^ (x >> 32)) & M32


def chunk_keys(data: bytes, chunk: int) -> list[int]:
    return [chunk_key(data[i:i + chunk]) for i in range(0, len(data), chunk)]


def forge_crc(data: bytearray, at: int, target: int) -> None:
    """Sets data[at:at+4] so that zlib.crc32(data) == target (in place)."""
    n = len(data)
    assert 0 <= at and at + 4 <= n
    base = bytearray(data)
    base[at:at + 4] = b"\0\0\0\0"
    c0 = zlib.crc32(base)
    zeros = bytes(n)
    z0 = zlib.crc32(zeros)
    # columns: the CRC change caused by bit b of the patch (linear part)
    cols = []
    for b in range(32):
        e = bytearray(zeros)
        e[at + b // 8] = 1 << (b % 8)
        cols.append(zlib.crc32(e) ^ z0)
    # solve sum_b x_b cols[b] = c0 ^ target over GF(2)
    rows = [(cols[b], 1 << b) for b in range(32)]
    want = c0 ^ target
    basis: dict[int, tuple[int, int]] = {}
    for v, tag in rows:
        for bit in range(31, -1, -1):
            if not (v >> bit) & 1:
                continue
            if bit in basis:
                bv, bt = basis[bit]
                v ^= bv
                tag ^= bt
            else:
                basis[bit] = (v, tag)
                break
    x = 0
    for bit in range(31, -1, -1):
        if (want >> bit) & 1:
            bv, bt = basis[bit]  # the 32 columns span GF(2)^32 (x^k is invertible mod P)
            want ^= bv
            x ^= bt
    assert want == 0
    data[at:at + 4] = x.to_bytes(4, "little")
    assert zlib.crc32(data) == target
