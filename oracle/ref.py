"""TEST INFRASTRUCTURE ONLY — the CPU checker, never the product.

ctypes bindings for oracle/_ref/libcracsim_ref.so (the unmodified reference
library + oracle/ref_capi.cpp) and oracle/_ref/libcrac_oracle.so (the plain-C
CRC restatement, oracle/crac_oracle.c).  ``RefSession`` mirrors
``paper_2008_10596_b200.engine.Session`` method for method so a test can drive
both with one call sequence.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this module.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path
from typing import Iterable, Optional, Sequence

HERE = Path(__file__).resolve().parent
REF_LIB = HERE / "_ref" / "libcracsim_ref.so"
ORACLE_LIB = HERE / "_ref" / "libcrac_oracle.so"

ERRC = ["InvalidArgument", "OutOfArena", "DoubleFree", "UnknownId", "StreamLimitExceeded",
        "BusyStream", "UnregisteredKernel", "DuplicateKernelId", "OutOfRange", "NotManaged",
        "HalfConflict", "QuiesceTimeout", "ReplayDivergence", "ImageCorrupt",
        "UnknownKernelBody", "DivisionByZero"]


class RefError(RuntimeError):
    def __init__(self, rc: int, message: str):
        self.rc = rc
        self.errc = ERRC[rc - 1] if 1 <= rc <= len(ERRC) else "Unknown"
        super().__init__(f"{self.errc}: {message}")


_U64, _U32, _U8, _I64, _P = C.c_uint64, C.c_uint32, C.c_uint8, C.c_int64, C.c_void_p
_PU64, _PU32, _PU8, _PD = (C.POINTER(C.c_uint64), C.POINTER(C.c_uint32), C.POINTER(C.c_uint8),
                           C.POINTER(C.c_double))
_SIGS = {
    "ref_last_error": (C.c_char_p, []),
    "ref_session_create": (C.c_int, [_U64, _U64, C.c_int, _U32, C.POINTER(_P)]),
    "ref_session_destroy": (None, [_P]),
    "ref_alloc": (C.c_int, [_P, _U8, _U64, _PU64, _PU64]),
    "ref_free": (C.c_int, [_P, _U64]),
    "ref_stream_create": (C.c_int, [_P, _PU64]),
    "ref_stream_destroy": (C.c_int, [_P, _U64]),
    "ref_register_fat_binary": (C.c_int, [_P, _U32, C.POINTER(C.c_char_p), _PU32, _PU32, _PU64]),
    "ref_unregister_fat_binary": (C.c_int, [_P, _U64]),
    "ref_launch": (C.c_int, [_P, _U64, C.c_char_p, _U32, _PU64, _PU64, _U32, _PU64]),
    "ref_copy_h2d": (C.c_int, [_P, _U64, _U64, _P, _U64, _I64]),
    "ref_copy_d2h": (C.c_int, [_P, _P, _U64, _U64, _U64, _I64]),
    "ref_copy_d2d": (C.c_int, [_P, _U64, _U64, _U64, _U64, _U64, _I64]),
    "ref_synchronize": (C.c_int, [_P]),
    "ref_page_read": (C.c_int, [_P, _U64, _U64, _U64, _U8, _P]),
    "ref_page_write": (C.c_int, [_P, _U64, _U64, _P, _U64, _U8]),
    "ref_set_app_state": (C.c_int, [_P, _P, _U64]),
    "ref_fill_synthetic": (C.c_int, [_P, _U64, _U64, _U8]),
    "ref_synth_bytes": (None, [_U64, _U64, _U64, _P]),
    "ref_checkpoint_image": (C.c_int, [_P, C.POINTER(_P), _PU64, _PD, _PD]),
    "ref_buffer_free": (None, [_P]),
    "ref_restart_image": (C.c_int, [_P, _U64, C.c_int, C.POINTER(_P), _PD, _PD]),
    "ref_decode_check": (C.c_int, [_P, _U64]),
    "ref_checkpoint_to_file": (C.c_int, [_P, C.c_char_p, C.c_int, _PD]),
    "ref_restart_from_file": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(_P), _PD]),
    "ref_summarize": (C.c_int, [_P, _U64, _PU64, _PU32, _PU64]),
    "ref_fixture_image": (C.c_int, [C.c_int, C.POINTER(_P), _PU64]),
    "ref_debug_dump": (C.c_int, [_P, C.POINTER(C.c_char_p)]),
    "ref_log_size": (C.c_int, [_P, _PU64]),
    "ref_live_records": (C.c_int, [_P, _U64, _PU64, _PU8, _PU64, _PU64, _PU64]),
    "ref_managed_pages": (C.c_int, [_P, _U64, _U64, _PU8, _PU64]),
    "ref_read_raw": (C.c_int, [_P, _U64, _U64, _P]),
}
_ORACLE_SIGS = {
    "oracle_crc32": (C.c_uint32, [_U32, _P, _U64]),
    "oracle_crc32_bitwise": (C.c_uint32, [_U32, _P, _U64]),
    "oracle_crc32_combine": (C.c_uint32, [_U32, _U32, _U64]),
    "oracle_chunk_crc32": (None, [_P, _U64, _U64, _PU32, C.c_int]),
    "oracle_mix64": (C.c_uint64, [_U64]),
    "oracle_synth_bytes": (None, [_U64, _U64, _U64, _U64, _P]),
}

_REF = None
_ORACLE = None


def ref_lib() -> C.CDLL:
    global _REF
    if _REF is None:
        if not REF_LIB.exists():
            raise RuntimeError(f"{REF_LIB} missing: run `make -C oracle` (needs /root/reference)")
        L = C.CDLL(str(REF_LIB))
        for n, (r, a) in _SIGS.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        _REF = L
    return _REF


def oracle_lib() -> C.CDLL:
    global _ORACLE
    if _ORACLE is None:
        if not ORACLE_LIB.exists():
            raise RuntimeError(f"{ORACLE_LIB} missing: run `make -C oracle`")
        L = C.CDLL(str(ORACLE_LIB))
        for n, (r, a) in _ORACLE_SIGS.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        _ORACLE = L
    return _ORACLE


def _check(rc: int) -> None:
    if rc != 0:
        raise RefError(rc, ref_lib().ref_last_error().decode(errors="replace"))


def _buf(data):
    mv = memoryview(data).cast("B")
    keep = C.create_string_buffer(bytes(mv), max(len(mv), 1))
    return C.cast(keep, C.c_void_p), len(mv), keep


# ---- CRC restatement -------------------------------------------------------------
def crc32(data, crc: int = 0) -> int:
    p, n, keep = _buf(data)
    return oracle_lib().oracle_crc32(crc, p, n)


def crc32_bitwise(data, crc: int = 0) -> int:
    p, n, keep = _buf(data)
    return oracle_lib().oracle_crc32_bitwise(crc, p, n)


def crc32_combine(a: int, b: int, len_b: int) -> int:
    return oracle_lib().oracle_crc32_combine(a, b, len_b)


def chunk_crc32(data, chunk: int = 65536, threads: int = 1) -> list[int]:
    p, n, keep = _buf(data)
    k = (n + chunk - 1) // chunk
    out = (C.c_uint32 * max(k, 1))()
    oracle_lib().oracle_chunk_crc32(p, n, chunk, out, threads)
    return list(out[:k])


def chunk_crc32_ptr(addr: int, n: int, chunk: int, out_addr: int, threads: int) -> None:
    oracle_lib().oracle_chunk_crc32(C.c_void_p(addr), n, chunk, C.cast(C.c_void_p(out_addr), _PU32),
                                    threads)


def synth_bytes(seed: int, alloc_id: int, size: int, word_offset: int = 0) -> bytes:
    out = C.create_string_buffer(max(size, 1))
    oracle_lib().oracle_synth_bytes(seed, alloc_id, word_offset, size, out)
    return out.raw[:size]


def mix64(x: int) -> int:
    return oracle_lib().oracle_mix64(x & (2**64 - 1))


# ---- the reference library --------------------------------------------------------
class RefSession:
    """The unmodified reference Session behind the same methods as engine.Session."""

    def __init__(self, seed: int = 0, arena_bytes: int = 1 << 24, mode: int = 0,
                 quiesce_timeout_ms: int = 30000, _handle=None):
        if _handle is None:
            h = C.c_void_p()
            _check(ref_lib().ref_session_create(seed, arena_bytes, mode, quiesce_timeout_ms,
                                                C.byref(h)))
            _handle = h
        self._h = _handle
        self.last_times = {}

    def alloc(self, kind: int, size: int):
        i, a = C.c_uint64(), C.c_uint64()
        _check(ref_lib().ref_alloc(self._h, kind, size, C.byref(i), C.byref(a)))
        return i.value, a.value

    def free(self, alloc_id: int) -> None:
        _check(ref_lib().ref_free(self._h, alloc_id))

    def stream_create(self) -> int:
        i = C.c_uint64()
        _check(ref_lib().ref_stream_create(self._h, C.byref(i)))
        return i.value

    def stream_destroy(self, stream: int) -> None:
        _check(ref_lib().ref_stream_destroy(self._h, stream))

    def register_fat_binary(self, kernels: Sequence[tuple[str, int, int]]) -> int:
        n = len(kernels)
        names = (C.c_char_p * max(n, 1))(*[k[0].encode() for k in kernels])
        ba = (C.c_uint32 * max(n, 1))(*[k[1] for k in kernels])
        sa = (C.c_uint32 * max(n, 1))(*[k[2] for k in kernels])
        h = C.c_uint64()
        _check(ref_lib().ref_register_fat_binary(self._h, n, names, ba, sa, C.byref(h)))
        return h.value

    def unregister_fat_binary(self, handle: int) -> None:
        _check(ref_lib().ref_unregister_fat_binary(self._h, handle))

    def launch(self, stream: int, kernel: str, buffers: Iterable[tuple[int, int]] = (),
               scalars: Iterable[int] = ()) -> None:
        b, s = list(buffers), list(scalars)
        ids = (C.c_uint64 * max(len(b), 1))(*[x[0] for x in b])
        offs = (C.c_uint64 * max(len(b), 1))(*[x[1] for x in b])
        sc = (C.c_uint64 * max(len(s), 1))(*[x & (2**64 - 1) for x in s])
        _check(ref_lib().ref_launch(self._h, stream, kernel.encode(), len(b), ids, offs, len(s), sc))

    def copy_h2d(self, alloc_id: int, offset: int, data, stream: Optional[int] = None) -> None:
        p, n, keep = _buf(data)
        _check(ref_lib().ref_copy_h2d(self._h, alloc_id, offset, p, n,
                                      -1 if stream is None else stream))

    def copy_d2h(self, alloc_id: int, offset: int, n: int, stream: Optional[int] = None) -> bytes:
        out = C.create_string_buffer(max(n, 1))
        _check(ref_lib().ref_copy_d2h(self._h, out, alloc_id, offset, n,
                                      -1 if stream is None else stream))
        return out.raw[:n]

    def copy_d2d(self, dst, src, n: int, stream: Optional[int] = None) -> None:
        _check(ref_lib().ref_copy_d2d(self._h, dst[0], dst[1], src[0], src[1], n,
                                      -1 if stream is None else stream))

    def synchronize(self) -> None:
        _check(ref_lib().ref_synchronize(self._h))

    def page_read(self, alloc_id: int, offset: int, n: int, side: int) -> bytes:
        out = C.create_string_buffer(max(n, 1))
        _check(ref_lib().ref_page_read(self._h, alloc_id, offset, n, side, out))
        return out.raw[:n]

    def page_write(self, alloc_id: int, offset: int, data, side: int) -> None:
        p, n, keep = _buf(data)
        _check(ref_lib().ref_page_write(self._h, alloc_id, offset, p, n, side))

    def set_app_state(self, data) -> None:
        p, n, keep = _buf(data)
        _check(ref_lib().ref_set_app_state(self._h, p, n))

    def fill_synthetic(self, alloc_id: int, seed: int, side: int = 1) -> None:
        _check(ref_lib().ref_fill_synthetic(self._h, alloc_id, seed, side))

    def checkpoint(self, image=None):
        """checkpoint(session) + encode_image; returns (bytes, times in s)."""
        p, n = C.c_void_p(), C.c_uint64()
        t1, t2 = C.c_double(), C.c_double()
        _check(ref_lib().ref_checkpoint_image(self._h, C.byref(p), C.byref(n), C.byref(t1),
                                              C.byref(t2)))
        try:
            data = C.string_at(p, n.value)
        finally:
            ref_lib().ref_buffer_free(p)
        self.last_times = {"checkpoint_s": t1.value, "encode_s": t2.value}
        return data, self.last_times

    def debug_dump(self) -> str:
        p = C.c_char_p()
        _check(ref_lib().ref_debug_dump(self._h, C.byref(p)))
        s = p.value.decode()
        ref_lib().ref_buffer_free(C.cast(p, C.c_void_p))
        return s

    def log_size(self) -> int:
        n = C.c_uint64()
        _check(ref_lib().ref_log_size(self._h, C.byref(n)))
        return n.value

    def live_records(self):
        n = C.c_uint64()
        _check(ref_lib().ref_live_records(self._h, 0, None, None, None, None, C.byref(n)))
        k = n.value
        ids, kinds = (C.c_uint64 * max(k, 1))(), (C.c_uint8 * max(k, 1))()
        sizes, addrs = (C.c_uint64 * max(k, 1))(), (C.c_uint64 * max(k, 1))()
        _check(ref_lib().ref_live_records(self._h, k, ids, kinds, sizes, addrs, C.byref(n)))
        return [(ids[i], kinds[i], sizes[i], addrs[i]) for i in range(k)]

    def managed_pages(self, alloc_id: int) -> list[int]:
        n = C.c_uint64()
        _check(ref_lib().ref_managed_pages(self._h, alloc_id, 0, None, C.byref(n)))
        flags = (C.c_uint8 * max(n.value, 1))()
        _check(ref_lib().ref_managed_pages(self._h, alloc_id, n.value, flags, C.byref(n)))
        return list(flags[: n.value])

    def read_raw(self, address: int, n: int) -> bytes:
        out = C.create_string_buffer(max(n, 1))
        _check(ref_lib().ref_read_raw(self._h, address, n, out))
        return out.raw[:n]

    def close(self) -> None:
        if getattr(self, "_h", None):
            ref_lib().ref_session_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ref_restart(image, mode: int = 0):
    p, n, keep = _buf(image)
    h = C.c_void_p()
    t1, t2 = C.c_double(), C.c_double()
    _check(ref_lib().ref_restart_image(p, n, mode, C.byref(h), C.byref(t1), C.byref(t2)))
    return RefSession(_handle=h), {"decode_s": t1.value, "restart_s": t2.value}


def ref_checkpoint_to_file(session: "RefSession", path, compress: bool = False) -> float:
    """The reference's checkpoint_to_file; returns its wall time in s."""
    t = C.c_double()
    _check(ref_lib().ref_checkpoint_to_file(session._h, str(path).encode(), int(compress),
                                            C.byref(t)))
    return t.value


def ref_restart_from_file(path, mode: int = 0):
    h, t = C.c_void_p(), C.c_double()
    _check(ref_lib().ref_restart_from_file(str(path).encode(), mode, C.byref(h), C.byref(t)))
    return RefSession(_handle=h), {"total_s": t.value}


def ref_decode_check(image) -> None:
    p, n, keep = _buf(image)
    _check(ref_lib().ref_decode_check(p, n))


def ref_summarize(image) -> dict:
    p, n, keep = _buf(image)
    lengths, crcs, totals = (C.c_uint64 * 7)(), (C.c_uint32 * 7)(), (C.c_uint64 * 5)()
    _check(ref_lib().ref_summarize(p, n, lengths, crcs, totals))
    return {"lengths": list(lengths), "crcs": list(crcs), "log_entries": totals[0],
            "active_allocations": totals[1], "payload_bytes": totals[2],
            "uvm_page_bytes": totals[3], "file_bytes": totals[4]}


def ref_fixture_image(which: int) -> bytes:
    p, n = C.c_void_p(), C.c_uint64()
    _check(ref_lib().ref_fixture_image(which, C.byref(p), C.byref(n)))
    try:
        return C.string_at(p, n.value)
    finally:
        ref_lib().ref_buffer_free(p)
