"""TEST INFRASTRUCTURE ONLY — plain-Python restatement of the CRACSIM1 image.

Follows the reference encoder/decoder rule by rule:
  encode: /root/reference/proj/src/image.cpp:30-98 (sections), :383-399 (framing)
  decode: /root/reference/proj/src/image.cpp:108-345 (strict validation)
  first-fit placement: /root/reference/proj/src/device_core.cpp:45-103
CRC-32 comes from oracle/crac_oracle.c (restated zlib algorithm) — or from
Python's zlib when the C oracle is not built; the two are pinned equal in
tests/test_oracle.py.  Pinned against the reference itself through the golden
vectors in tests/golden/ (made by oracle/make_golden.py from the reference
library).
"""
from __future__ import annotations

import struct
import zlib
from dataclasses import dataclass, field

K_ARENA_BASE = 0x0D00_0000_0000
K_ALIGN = 256
K_PAGE = 4096
MAGIC = b"CRACSIM1"


class ImageCorrupt(ValueError):
    pass


def crc32(b: bytes) -> int:
    return zlib.crc32(b) & 0xFFFFFFFF


def round_up_align(n: int) -> int:
    return (n + K_ALIGN - 1) & ~(K_ALIGN - 1)


def page_count(n: int) -> int:
    return (n + K_PAGE - 1) // K_PAGE


@dataclass
class Snapshot:
    seed: int = 0
    arena_bytes: int = 1 << 24
    engine_version: int = 1
    log: list = field(default_factory=list)        # (seq, op, kind, size, id, address)
    payloads: list = field(default_factory=list)   # (id, bytes)
    managed: list = field(default_factory=list)    # (id, [(index, dev, dirty, bytes)])
    streams: list = field(default_factory=list)
    app_state: bytes = b""
    binaries: list = field(default_factory=list)   # (handle, [(name, barity, sarity)])


def encode_sections(s: Snapshot) -> list[bytes]:
    meta = struct.pack("<QQII", s.seed, s.arena_bytes, s.engine_version, 0)
    log = b"".join(struct.pack("<QBBHQQQ", seq, op, kind, 0, size, i, addr)
                   for (seq, op, kind, size, i, addr) in s.log)
    pay = b"".join(struct.pack("<QQ", i, len(b)) + b for (i, b) in s.payloads)
    uvm = bytearray()
    for (i, pages) in s.managed:
        uvm += struct.pack("<QQ", i, len(pages))
        for (idx, dev, dirty, b) in pages:
            uvm += struct.pack("<QII", idx, (1 if dev else 0) | (2 if dirty else 0), len(b)) + b
    streams = b"".join(struct.pack("<Q", x) for x in s.streams)
    reg = bytearray(struct.pack("<Q", len(s.binaries)))
    for (h, ks) in s.binaries:
        reg += struct.pack("<QI", h, len(ks))
        for (name, ba, sa) in ks:
            nb = name.encode()
            reg += struct.pack("<I", len(nb)) + nb + struct.pack("<II", ba, sa)
    return [meta, log, pay, bytes(uvm), streams, bytes(s.app_state), bytes(reg)]


def encode_image(s: Snapshot) -> bytes:
    out = bytearray(MAGIC + struct.pack("<II", 1, 7))
    for tag, payload in enumerate(encode_sections(s), start=1):
        out += struct.pack("<IIQ", tag, 0, len(payload)) + payload + struct.pack("<I", crc32(payload))
    return bytes(out)


def _need(b: bytes, pos: int, n: int) -> None:
    if len(b) - pos < n:
        raise ImageCorrupt("truncated input")


def decode_image(b: bytes) -> Snapshot:
    """Strict decode; raises ImageCorrupt exactly where the reference does."""
    _need(b, 0, 16)
    if b[:8] != MAGIC:
        raise ImageCorrupt("bad magic")
    version, count = struct.unpack_from("<II", b, 8)
    if version != 1:
        raise ImageCorrupt("unsupported version")
    if count != 7:
        raise ImageCorrupt("section count")
    pos = 16
    s = Snapshot()
    live, streams, handles = {}, {}, {}
    for i in range(7):
        _need(b, pos, 16)
        tag, reserved, length = struct.unpack_from("<IIQ", b, pos)
        pos += 16
        if tag != i + 1:
            raise ImageCorrupt("tag order")
        if reserved != 0:
            raise ImageCorrupt("reserved")
        _need(b, pos, length)
        payload = b[pos:pos + length]
        pos += length
        _need(b, pos, 4)
        (crc,) = struct.unpack_from("<I", b, pos)
        pos += 4
        if crc != crc32(payload):
            raise ImageCorrupt("crc mismatch")
        if tag == 1:
            if length != 24:
                raise ImageCorrupt("META length")
            s.seed, s.arena_bytes, s.engine_version, r = struct.unpack("<QQII", payload)
            if r != 0 or s.engine_version != 1 or s.arena_bytes == 0 or s.arena_bytes % K_ALIGN:
                raise ImageCorrupt("META")
        elif tag == 2:
            if length % 36:
                raise ImageCorrupt("LOG length")
            nxt = {"a": 1, "s": 1, "h": 1}
            for k in range(length // 36):
                seq, op, kind, pad, size, ident, addr = struct.unpack_from("<QBBHQQQ", payload, 36 * k)
                if seq != k + 1 or pad != 0 or not 1 <= op <= 6:
                    raise ImageCorrupt("LOG record")
                if op == 1:
                    if not 1 <= kind <= 3 or size == 0 or ident != nxt["a"]:
                        raise ImageCorrupt("Alloc")
                    nxt["a"] += 1
                    if (addr < K_ARENA_BASE or addr % K_ALIGN
                            or addr - K_ARENA_BASE + round_up_align(size) > s.arena_bytes):
                        raise ImageCorrupt("Alloc address")
                    live[ident] = (kind, size)
                else:
                    if kind or size or addr:
                        raise ImageCorrupt("non-Alloc payload")
                    if op == 2:
                        if ident not in live:
                            raise ImageCorrupt("Free")
                        del live[ident]
                    elif op == 5:
                        if ident != nxt["s"]:
                            raise ImageCorrupt("stream ids")
                        nxt["s"] += 1
                        streams[ident] = True
                    elif op == 6:
                        if not streams.get(ident):
                            raise ImageCorrupt("destroy")
                        streams[ident] = False
                    elif op == 3:
                        if ident != nxt["h"]:
                            raise ImageCorrupt("handles")
                        nxt["h"] += 1
                        handles[ident] = True
                    elif op == 4:
                        if not handles.get(ident):
                            raise ImageCorrupt("unregister")
                        handles[ident] = False
                s.log.append((seq, op, kind, size, ident, addr))
        elif tag == 3:
            want = [(i_, sz) for i_, (k_, sz) in sorted(live.items()) if k_ != 3]
            p, n = 0, 0
            while p < length:
                if n >= len(want):
                    raise ImageCorrupt("extra payload")
                _need(payload, p, 16)
                ident, ln = struct.unpack_from("<QQ", payload, p)
                p += 16
                if (ident, ln) != want[n]:
                    raise ImageCorrupt("payload frame")
                _need(payload, p, ln)
                s.payloads.append((ident, payload[p:p + ln]))
                p += ln
                n += 1
            if n != len(want):
                raise ImageCorrupt("missing payload")
        elif tag == 4:
            want = [(i_, sz) for i_, (k_, sz) in sorted(live.items()) if k_ == 3]
            p, n = 0, 0
            while p < length:
                if n >= len(want):
                    raise ImageCorrupt("extra uvm")
                _need(payload, p, 16)
                ident, pages = struct.unpack_from("<QQ", payload, p)
                p += 16
                if ident != want[n][0] or pages != page_count(want[n][1]):
                    raise ImageCorrupt("uvm frame")
                plist = []
                for k in range(pages):
                    _need(payload, p, 16)
                    idx, flags, ln = struct.unpack_from("<QII", payload, p)
                    p += 16
                    if idx != k or flags > 3 or ln != min(K_PAGE, want[n][1] - k * K_PAGE):
                        raise ImageCorrupt("page frame")
                    _need(payload, p, ln)
                    plist.append((idx, bool(flags & 1), bool(flags & 2), payload[p:p + ln]))
                    p += ln
                s.managed.append((ident, plist))
                n += 1
            if n != len(want):
                raise ImageCorrupt("missing uvm")
        elif tag == 5:
            if length % 8:
                raise ImageCorrupt("STREAMS length")
            s.streams = list(struct.unpack(f"<{length // 8}Q", payload))
            if s.streams != sorted(k for k, on in streams.items() if on):
                raise ImageCorrupt("STREAMS")
        elif tag == 6:
            s.app_state = payload
        elif tag == 7:
            _need(payload, 0, 8)
            (cnt,) = struct.unpack_from("<Q", payload, 0)
            p, seen = 8, set()
            for _ in range(cnt):
                _need(payload, p, 12)
                h, nk = struct.unpack_from("<QI", payload, p)
                p += 12
                ks = []
                for _ in range(nk):
                    _need(payload, p, 4)
                    (nl,) = struct.unpack_from("<I", payload, p)
                    p += 4
                    _need(payload, p, nl + 8)
                    name = payload[p:p + nl].decode(errors="replace")
                    p += nl
                    ba, sa = struct.unpack_from("<II", payload, p)
                    p += 8
                    if not name or name in seen:
                        raise ImageCorrupt("kernel name")
                    seen.add(name)
                    ks.append((name, ba, sa))
                s.binaries.append((h, ks))
            if p != length:
                raise ImageCorrupt("registry trailing")
            if [h for h, _ in s.binaries] != sorted(k for k, on in handles.items() if on):
                raise ImageCorrupt("registry handles")
    if pos != len(b):
        raise ImageCorrupt("trailing bytes")
    return s


def rich_snapshot() -> Snapshot:
    """The reference's rich_snapshot fixture (test_image.cpp:24-52)."""
    s = Snapshot(seed=5, arena_bytes=1 << 20)
    base = K_ARENA_BASE
    s.log = [(1, 1, 1, 1000, 1, base), (2, 1, 3, 4196, 2, base + 1024), (3, 5, 0, 0, 1, 0),
             (4, 1, 2, 10, 3, base + 1024 + 4352), (5, 3, 0, 0, 1, 0), (6, 5, 0, 0, 2, 0),
             (7, 6, 0, 0, 1, 0), (8, 1, 1, 5, 4, base + 1024 + 4352 + 256), (9, 2, 0, 0, 4, 0)]
    s.payloads = [(1, b"\xA1" * 1000), (3, b"\xA3" * 10)]
    s.managed = [(2, [(0, True, False, b"\xB0" * 4096), (1, False, True, b"\xB1" * 100)])]
    s.streams = [2]
    s.app_state = b"\x5A" * 33
    s.binaries = [(1, [("scale", 2, 1), ("probe", 1, 0)])]
    return s


def empty_snapshot() -> Snapshot:
    """test_image.cpp:14-19."""
    return Snapshot(seed=0, arena_bytes=1 << 24)


class FirstFit:
    """Naive first-fit over live extents (the reference's own test oracle
    shape, tests/support/reference_alloc.hpp:11-38, restated)."""

    def __init__(self, arena_bytes: int, base: int = K_ARENA_BASE):
        self.base, self.limit = base, base + arena_bytes
        self.live: dict[int, int] = {}

    def alloc(self, size: int):
        need = round_up_align(size)
        cursor = self.base
        for addr in sorted(self.live):
            if addr - cursor >= need:
                break
            cursor = addr + self.live[addr]
        if self.limit - cursor < need:
            return None
        self.live[cursor] = need
        return cursor

    def free(self, addr: int) -> None:
        del self.live[addr]
