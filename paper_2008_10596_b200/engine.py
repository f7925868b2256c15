"""Python host mirror of the reference engine API over the C-ABI (crac_engine.h).

Names follow the reference (ref: /root/reference/proj/include/cracsim/
ckpt_engine.hpp, shim.hpp, image.hpp): ``Session`` with the interposed
``RuntimeApi`` calls, ``checkpoint`` / ``restart`` / ``decode_image`` /
``summarize_image``.  Errors surface as ``CracError`` carrying the reference
``Errc`` name.  There is no CPU fallback: if ``libcrac_b200.so`` is missing or
the GPU is unusable every call raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path
from typing import Iterable, Optional, Sequence

LIB_PATH = Path(__file__).resolve().parent / "libcrac_b200.so"

DEVICE, PINNED, MANAGED = 1, 2, 3
HOST_SIDE, DEVICE_SIDE = 0, 1
DIRECT, PROXY = 0, 1

ERRC = ["InvalidArgument", "OutOfArena", "DoubleFree", "UnknownId", "StreamLimitExceeded",
        "BusyStream", "UnregisteredKernel", "DuplicateKernelId", "OutOfRange", "NotManaged",
        "HalfConflict", "QuiesceTimeout", "ReplayDivergence", "ImageCorrupt",
        "UnknownKernelBody", "DivisionByZero", "DeviceFault"]


class CracError(RuntimeError):
    def __init__(self, rc: int, message: str):
        self.rc = rc
        self.errc = ERRC[rc - 1] if 1 <= rc <= len(ERRC) else "Unknown"
        super().__init__(f"{self.errc}: {message}")


class Stats(C.Structure):
    _fields_ = [("total_ms", C.c_double), ("hash_ms", C.c_double), ("pack_ms", C.c_double),
                ("copy_ms", C.c_double), ("hash_bytes", C.c_uint64), ("hash_launches", C.c_uint64),
                ("pack_launches", C.c_uint64), ("pack_bytes", C.c_uint64),
                ("d2h_bytes", C.c_uint64), ("h2d_bytes", C.c_uint64),
                ("image_bytes", C.c_uint64), ("dirty_chunks", C.c_uint64),
                ("total_chunks", C.c_uint64), ("incremental", C.c_int32),
                ("reserved", C.c_int32), ("stall_ms", C.c_double),
                ("shadow_bytes", C.c_uint64), ("barrier_ms", C.c_double),
                ("host_pre_ms", C.c_double)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved"}


class IoStats(C.Structure):
    _fields_ = [("ms", C.c_double), ("bytes", C.c_uint64), ("threads", C.c_uint32),
                ("direct", C.c_int32), ("bounced", C.c_uint64), ("streamed", C.c_uint64)]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["direct"] = bool(d["direct"])
        d["GBps"] = self.bytes / (self.ms * 1e6) if self.ms > 0 else 0.0
        return d


class VerifyReport(C.Structure):
    _fields_ = [("sections_checked", C.c_uint64), ("crc_bytes", C.c_uint64),
                ("payloads_compared", C.c_uint64), ("payload_bytes_compared", C.c_uint64),
                ("mismatched_payloads", C.c_uint64), ("first_bad_id", C.c_uint64),
                ("bad_sections", C.c_uint32), ("threads", C.c_uint32), ("ms", C.c_double)]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["ok"] = self.bad_sections == 0 and self.mismatched_payloads == 0
        if d["first_bad_id"] == 2**64 - 1:
            d["first_bad_id"] = None
        return d


_LIB: Optional[C.CDLL] = None

# name -> (restype, argtypes)
_U64, _U32, _U8, _I64, _P = C.c_uint64, C.c_uint32, C.c_uint8, C.c_int64, C.c_void_p
_PU64, _PU32, _PU8 = C.POINTER(C.c_uint64), C.POINTER(C.c_uint32), C.POINTER(C.c_uint8)
_SIGS = {
    "crac_last_error": (C.c_char_p, []),
    "crac_abi_version": (C.c_int, []),
    "crac_session_create": (C.c_int, [_U64, _U64, C.c_int, _U32, C.POINTER(_P)]),
    "crac_session_destroy": (None, [_P]),
    "crac_session_fixed_va": (C.c_int, [_P]),
    "crac_alloc": (C.c_int, [_P, _U8, _U64, _PU64, _PU64]),
    "crac_free": (C.c_int, [_P, _U64]),
    "crac_stream_create": (C.c_int, [_P, _PU64]),
    "crac_stream_destroy": (C.c_int, [_P, _U64]),
    "crac_register_fat_binary": (C.c_int, [_P, _U32, C.POINTER(C.c_char_p), _PU32, _PU32, _PU64]),
    "crac_unregister_fat_binary": (C.c_int, [_P, _U64]),
    "crac_launch": (C.c_int, [_P, _U64, C.c_char_p, _U32, _PU64, _PU64, _U32, _PU64]),
    "crac_copy_h2d": (C.c_int, [_P, _U64, _U64, _P, _U64, _I64]),
    "crac_copy_d2h": (C.c_int, [_P, _P, _U64, _U64, _U64, _I64]),
    "crac_copy_d2d": (C.c_int, [_P, _U64, _U64, _U64, _U64, _U64, _I64]),
    "crac_synchronize": (C.c_int, [_P]),
    "crac_page_read": (C.c_int, [_P, _U64, _U64, _U64, _U8, _P]),
    "crac_page_write": (C.c_int, [_P, _U64, _U64, _P, _U64, _U8]),
    "crac_set_app_state": (C.c_int, [_P, _P, _U64]),
    "crac_image_create": (C.c_int, [C.POINTER(_P)]),
    "crac_image_destroy": (None, [_P]),
    "crac_image_view": (C.c_int, [_P, C.POINTER(_P), _PU64]),
    "crac_image_pages": (C.c_int, [_P, _PU64, _PU64]),
    "crac_checkpoint": (C.c_int, [_P, _P, C.POINTER(Stats)]),
    "crac_checkpoint_incremental": (C.c_int, [_P, _P, C.POINTER(Stats)]),
    "crac_checkpoint_value": (C.c_int, [_P, C.POINTER(_P), _PU64]),
    "crac_reserve_shadow": (C.c_int, [_P, _U64]),
    "crac_checkpoint_begin": (C.c_int, [_P, _P, C.POINTER(Stats)]),
    "crac_checkpoint_finish": (C.c_int, [_P, C.POINTER(Stats)]),
    "crac_restart": (C.c_int, [_P, _U64, C.c_int, C.POINTER(_P), C.POINTER(Stats)]),
    "crac_decode_check": (C.c_int, [_P, _U64]),
    "crac_checkpoint_precopy_begin": (C.c_int, [_P, _P, C.POINTER(Stats)]),
    "crac_checkpoint_precopy_finish": (C.c_int, [_P, C.POINTER(Stats)]),
    "crac_reserve_shadow_on": (C.c_int, [_P, _U64, C.c_int]),
    "crac_crc32_host": (C.c_uint32, [_P, _U64, _U32]),
    "crac_crc32_copy_host": (C.c_uint32, [_P, _P, _U64, _U32]),
    "crac_session_set_barrier": (C.c_int, [_P, _P, _P]),
    "crac_compress_image_gpu": (C.c_int, [_P, _U64, C.POINTER(_P), _PU64, C.POINTER(C.c_double)]),
    "crac_probe_managed_populate": (C.c_int, [_U64, _U64, _U32, C.POINTER(C.c_double)]),
    "crac_image_verify": (C.c_int, [_P, _U64, _U32, _U64, C.c_int, C.POINTER(VerifyReport)]),
    "crac_session_verify_synthetic": (C.c_int, [_P, _U64, _PU64, _PU64]),
    "crac_barrier_open": (C.c_int, [C.c_char_p, _U32, _U32, _U32, C.POINTER(_P)]),
    "crac_barrier_wait": (C.c_int, [_P]),
    "crac_barrier_hook": (C.c_int, [_P, C.c_int]),
    "crac_barrier_generation": (_U64, [_P]),
    "crac_barrier_close": (None, [_P, C.c_int]),
    "crac_peek_cuda_error": (C.c_int, []),
    "crac_drop_arena_cache": (C.c_int, [C.c_int]),
    "crac_drop_arena_cache_async": (C.c_int, [C.c_int]),
    "crac_stream_handle": (C.c_int, [_P, _U64, C.POINTER(_P)]),
    "crac_live_streams": (C.c_int, [_P, _U64, _PU64, _PU64]),
    "crac_gate_enter": (C.c_int, [_P]),
    "crac_gate_leave": (C.c_int, [_P]),
    "crac_set_device_wide_drain": (C.c_int, [_P, C.c_int]),
    "crac_get_app_state": (C.c_int, [_P, C.POINTER(_P), _PU64]),
    "crac_checkpoint_to_file": (C.c_int, [_P, _P, C.c_char_p, C.c_int, C.POINTER(Stats),
                                          C.POINTER(IoStats)]),
    "crac_restart_from_file": (C.c_int, [C.c_char_p, _P, C.c_int, C.POINTER(_P),
                                         C.POINTER(Stats), C.POINTER(IoStats)]),
    "crac_file_write": (C.c_int, [C.c_char_p, _P, _U64, _U32, _U64, _U32, C.POINTER(IoStats)]),
    "crac_file_size": (C.c_int, [C.c_char_p, _PU64]),
    "crac_file_read": (C.c_int, [C.c_char_p, _P, _U64, _U32, _U64, _U32, _PU64,
                                 C.POINTER(IoStats)]),
    "crac_summarize": (C.c_int, [_P, _U64, _PU64, _PU32, _PU64]),
    "crac_debug_dump": (C.c_int, [_P, C.POINTER(C.c_char_p)]),
    "crac_buffer_free": (None, [_P]),
    "crac_log_size": (C.c_int, [_P, _PU64]),
    "crac_live_records": (C.c_int, [_P, _U64, _PU64, _PU8, _PU64, _PU64, _PU64]),
    "crac_managed_pages": (C.c_int, [_P, _U64, _U64, _PU8, _PU64]),
    "crac_read_raw": (C.c_int, [_P, _U64, _U64, _P]),
    "crac_backing_ptr": (C.c_int, [_P, _U64, _PU64]),
    "crac_fill_synthetic": (C.c_int, [_P, _U64, _U64, _U8]),
    "crac_mutate_device": (C.c_int, [_P, _U64, _U64, _U64, _PU64]),
    "crac_hash_host_buffer": (C.c_int, [_P, _U64, _U32, _PU32]),
    "crac_hash_session": (C.c_int, [_P, C.POINTER(Stats)]),
    # kernel-level C-ABI (crac_gpu.h)
    "crac_gpu_init": (C.c_int, []),
    "crac_chunk_crc32": (C.c_int, [_P, _P, _U32, _U32, _U64, _P, _P]),
    "crac_chunk_crc32_range": (C.c_int, [_P, _P, _U32, _U32, _U64, _U64, _P, _U32, _P]),
    "crac_chunk_key_range": (C.c_int, [_P, _P, _U32, _U32, _U64, _U64, _P, _P, _U32, _P]),
    "crac_gather_chunks_to_host": (C.c_int, [_P, _P, _U32, _U32, _P, _U64, _U64, _P, _P, _P]),
    "crac_write_frames": (C.c_int, [_P, _U32, _P, _P]),
    "crac_hash_copy_range": (C.c_int, [_P, _P, _U32, _U32, _U64, _U64, _P, _P, _P, _P, C.c_int,
                                       _P]),
    "crac_gather_chunks_to_host_dev": (C.c_int, [_P, _P, _U32, _U32, _P, _P, _U64, _U32, _P, _P, _P]),
    "crac_diff_compact_range": (C.c_int, [_P, _P, _U64, _U64, _P, _P, _P, _P]),
    "crac_fold_sections": (C.c_int, [_P, _U32, _P, _P, _U32, _P, _U64, _U64, _P, _P]),
    "crac_hash_drain_range": (C.c_int, [_P, _P, _U32, _U32, _U64, _U64, _P, _P, _P, _P, _P, _P,
                                        _P, _P]),
    "crac_hash_drain_split": (C.c_int, [_P, _P, _U32, _U32, _U64, _U64, _P, _P, _P, _P, _P, _P,
                                        _P, _P, _U32, _P]),
    "crac_pack_records": (C.c_int, [_P, _U32, _P, _U64, _U64, _P, _P]),
    "crac_scatter_records": (C.c_int, [_P, _U32, _P, _P, _U64, _U64, _P]),
    "crac_diff_compact": (C.c_int, [_P, _P, _U64, _P, _P, _P, _P]),
    "crac_gather_chunks": (C.c_int, [_P, _P, _U32, _U32, _P, _U64, _U64, _P, _P]),
    "crac_fill_synth": (C.c_int, [_P, _U64, _U64, _U64, _U64, _P]),
    "crac_deflate_segments": (C.c_int, [_P, _U64, _P, _P, _P, C.c_int, _P]),
    "crac_gather_segments": (C.c_int, [_P, _U64, _P, _P, _P, _P, C.c_int, _P]),
    "crac_touch_even_runs": (C.c_int, [_P, _U64, _U64, _P]),
    "crac_verify_synth": (C.c_int, [_P, _U64, _U64, _U64, _P, _P]),
    "crac_mutate_chunks": (C.c_int, [_P, _P, _P, _U32, _U32, _U64, _U64, _U64, _U64, _P]),
}


def exported_symbols() -> list[str]:
    return sorted(_SIGS)


def lib() -> C.CDLL:
    """Loads the in-tree CUDA library; raises loudly if it is absent."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2008_10596_b200.build` "
                               "(there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def _bytes_at(ptr: int, n: int) -> bytes:
    """Copy of n bytes at ptr (ctypes.string_at takes an int size: wrong past 2 GiB)."""
    if not n:
        return b""
    return bytes(memoryview((C.c_ubyte * n).from_address(ptr)))


def _check(rc: int) -> None:
    if rc != 0:
        raise CracError(rc, lib().crac_last_error().decode(errors="replace"))


def _buf(data) -> tuple[C.c_void_p, int, object]:
    """(pointer, length, keepalive) for bytes / bytearray / memoryview / numpy."""
    mv = memoryview(data).cast("B")
    if mv.readonly:
        keep = C.create_string_buffer(bytes(mv), len(mv)) if len(mv) else C.create_string_buffer(1)
        return C.cast(keep, C.c_void_p), len(mv), keep
    arr = (C.c_char * len(mv)).from_buffer(mv) if len(mv) else C.create_string_buffer(1)
    return C.cast(arr, C.c_void_p), len(mv), arr


def _opt_stream(stream: Optional[int]) -> int:
    return -1 if stream is None else int(stream)


class Image:
    """Page-locked image buffer (cracsim::PinnedImage), reused across checkpoints."""

    def __init__(self):
        h = C.c_void_p()
        _check(lib().crac_image_create(C.byref(h)))
        self._h = h

    def view(self) -> memoryview:
        p, n = C.c_void_p(), C.c_uint64()
        _check(lib().crac_image_view(self._h, C.byref(p), C.byref(n)))
        if n.value == 0:
            return memoryview(b"")
        return memoryview((C.c_char * n.value).from_address(p.value)).cast("B")

    def address(self) -> tuple[int, int]:
        p, n = C.c_void_p(), C.c_uint64()
        _check(lib().crac_image_view(self._h, C.byref(p), C.byref(n)))
        return p.value or 0, n.value

    def tobytes(self) -> bytes:
        return bytes(self.view())

    def pages(self) -> dict:
        """Capacity of the page-locked buffer and its 2 MiB-page backed bytes."""
        cap, huge = C.c_uint64(), C.c_uint64()
        _check(lib().crac_image_pages(self._h, C.byref(cap), C.byref(huge)))
        return {"capacity": cap.value, "huge_page_bytes": huge.value}

    def close(self):
        if getattr(self, "_h", None):
            lib().crac_image_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# CRAC_PHASE_* (crac_engine.h): when a session's global-checkpoint hook runs
PHASE_QUIESCED, PHASE_IMAGE_COMPLETE, PHASE_PERSISTED = 0, 1, 2
BARRIER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int)


class Barrier:
    """The node-local global-checkpoint barrier (crac_barrier_open): every rank
    of the job opens the same name with the same world size."""

    def __init__(self, name: str, world: int, rank: int, timeout_ms: int = 60000):
        h = C.c_void_p()
        _check(lib().crac_barrier_open(name.encode(), world, rank, timeout_ms, C.byref(h)))
        self._h = h
        self.name, self.world, self.rank = name, world, rank

    def wait(self) -> None:
        _check(lib().crac_barrier_wait(self._h))

    def generation(self) -> int:
        return lib().crac_barrier_generation(self._h)

    def close(self, unlink: bool = False) -> None:
        if getattr(self, "_h", None):
            lib().crac_barrier_close(self._h, int(unlink))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class LiveRecord:
    id: int
    kind: int
    size: int
    address: int


class Session:
    """ref: cracsim::Session + RuntimeApi (ckpt_engine.hpp:29-55, shim.hpp:159-184)."""

    def __init__(self, seed: int = 0, arena_bytes: int = 1 << 24, mode: int = DIRECT,
                 quiesce_timeout_ms: int = 30000, _handle: Optional[C.c_void_p] = None):
        if _handle is None:
            h = C.c_void_p()
            _check(lib().crac_session_create(seed, arena_bytes, mode, quiesce_timeout_ms, C.byref(h)))
            _handle = h
        self._h = _handle

    # ---- RuntimeApi ----
    def alloc(self, kind: int, size: int) -> tuple[int, int]:
        i, a = C.c_uint64(), C.c_uint64()
        _check(lib().crac_alloc(self._h, kind, size, C.byref(i), C.byref(a)))
        return i.value, a.value

    def free(self, alloc_id: int) -> None:
        _check(lib().crac_free(self._h, alloc_id))

    def stream_create(self) -> int:
        i = C.c_uint64()
        _check(lib().crac_stream_create(self._h, C.byref(i)))
        return i.value

    def stream_destroy(self, stream: int) -> None:
        _check(lib().crac_stream_destroy(self._h, stream))

    def register_fat_binary(self, kernels: Sequence[tuple[str, int, int]]) -> int:
        n = len(kernels)
        names = (C.c_char_p * max(n, 1))(*[k[0].encode() for k in kernels])
        ba = (C.c_uint32 * max(n, 1))(*[k[1] for k in kernels])
        sa = (C.c_uint32 * max(n, 1))(*[k[2] for k in kernels])
        h = C.c_uint64()
        _check(lib().crac_register_fat_binary(self._h, n, names, ba, sa, C.byref(h)))
        return h.value

    def unregister_fat_binary(self, handle: int) -> None:
        _check(lib().crac_unregister_fat_binary(self._h, handle))

    def launch(self, stream: int, kernel: str, buffers: Iterable[tuple[int, int]] = (),
               scalars: Iterable[int] = ()) -> None:
        b = list(buffers)
        s = list(scalars)
        ids = (C.c_uint64 * max(len(b), 1))(*[x[0] for x in b])
        offs = (C.c_uint64 * max(len(b), 1))(*[x[1] for x in b])
        sc = (C.c_uint64 * max(len(s), 1))(*[x & (2**64 - 1) for x in s])
        _check(lib().crac_launch(self._h, stream, kernel.encode(), len(b), ids, offs, len(s), sc))

    def copy_h2d(self, alloc_id: int, offset: int, data, stream: Optional[int] = None) -> None:
        p, n, keep = _buf(data)
        _check(lib().crac_copy_h2d(self._h, alloc_id, offset, p, n, _opt_stream(stream)))

    def copy_d2h(self, alloc_id: int, offset: int, n: int, stream: Optional[int] = None) -> bytes:
        out = C.create_string_buffer(max(n, 1))
        _check(lib().crac_copy_d2h(self._h, out, alloc_id, offset, n, _opt_stream(stream)))
        return out.raw[:n]

    def copy_d2d(self, dst: tuple[int, int], src: tuple[int, int], n: int,
                 stream: Optional[int] = None) -> None:
        _check(lib().crac_copy_d2d(self._h, dst[0], dst[1], src[0], src[1], n, _opt_stream(stream)))

    def synchronize(self) -> None:
        _check(lib().crac_synchronize(self._h))

    def page_read(self, alloc_id: int, offset: int, n: int, side: int) -> bytes:
        out = C.create_string_buffer(max(n, 1))
        _check(lib().crac_page_read(self._h, alloc_id, offset, n, side, out))
        return out.raw[:n]

    def page_write(self, alloc_id: int, offset: int, data, side: int) -> None:
        p, n, keep = _buf(data)
        _check(lib().crac_page_write(self._h, alloc_id, offset, p, n, side))

    def set_app_state(self, data) -> None:
        p, n, keep = _buf(data)
        _check(lib().crac_set_app_state(self._h, p, n))

    # ---- global checkpoint ----
    def set_barrier(self, barrier: Optional[Barrier]) -> None:
        """Installs the node-local shared-memory barrier as this session's
        global-checkpoint hook (None removes it)."""
        fn = C.cast(lib().crac_barrier_hook, C.c_void_p) if barrier else None
        _check(lib().crac_session_set_barrier(self._h, fn, barrier._h if barrier else None))
        self._barrier_keep = barrier

    def set_barrier_hook(self, hook) -> None:
        """Installs a Python callable hook(phase) -> int as the global-checkpoint
        hook (an MPI/gloo barrier, or a test probe); None removes it."""
        cb = BARRIER_FN(lambda _ctx, phase: int(hook(phase) or 0)) if hook else None
        _check(lib().crac_session_set_barrier(self._h, C.cast(cb, C.c_void_p) if cb else None, None))
        self._barrier_keep = cb

    # ---- engine ----
    def checkpoint(self, image: Optional[Image] = None) -> tuple[bytes, dict]:
        """checkpoint_image: returns (image bytes, device-timed stats)."""
        img = image or Image()
        st = Stats()
        _check(lib().crac_checkpoint(self._h, img._h, C.byref(st)))
        return img.tobytes(), st.as_dict()

    def checkpoint_into(self, image: Image, incremental: bool = False) -> dict:
        st = Stats()
        fn = lib().crac_checkpoint_incremental if incremental else lib().crac_checkpoint
        _check(fn(self._h, image._h, C.byref(st)))
        return st.as_dict()

    def checkpoint_to_file(self, path, image: Optional[Image] = None,
                           compress=False) -> tuple[dict, dict]:
        """checkpoint_to_file: GPU drain into `image`, then the parallel
        (O_DIRECT, fdatasync'd) file write.  compress: False, True (the
        reference's zlib level-6 bytes) or "gpu" (the GPU deflate).  Returns
        (drain stats, io stats)."""
        img = image or Image()
        st, io = Stats(), IoStats()
        mode = 2 if compress == "gpu" else int(bool(compress))
        _check(lib().crac_checkpoint_to_file(self._h, img._h, str(path).encode(), mode,
                                             C.byref(st), C.byref(io)))
        return st.as_dict(), io.as_dict()

    def checkpoint_precopy_begin(self, image: Image) -> dict:
        """Pre-copy the state into `image` while the application keeps running."""
        st = Stats()
        _check(lib().crac_checkpoint_precopy_begin(self._h, image._h, C.byref(st)))
        return st.as_dict()

    def checkpoint_precopy_finish(self) -> dict:
        """Quiesce and re-send the chunks changed since the pre-copy."""
        st = Stats()
        _check(lib().crac_checkpoint_precopy_finish(self._h, C.byref(st)))
        return st.as_dict()

    def reserve_shadow(self, nbytes: int, device: Optional[int] = None) -> None:
        """HBM the stall-reduced drain may stage the stream in (0 releases it);
        `device` puts it on a buddy GPU reachable by peer access (§8f.3)."""
        if device is None:
            _check(lib().crac_reserve_shadow(self._h, nbytes))
        else:
            _check(lib().crac_reserve_shadow_on(self._h, nbytes, device))

    def checkpoint_begin(self, image: Image) -> dict:
        """Quiesce, snapshot into the shadow, resume; the D2H keeps running."""
        st = Stats()
        _check(lib().crac_checkpoint_begin(self._h, image._h, C.byref(st)))
        return st.as_dict()

    def checkpoint_finish(self) -> dict:
        st = Stats()
        _check(lib().crac_checkpoint_finish(self._h, C.byref(st)))
        return st.as_dict()

    def checkpoint_value(self) -> bytes:
        """encode_image(checkpoint(session)) through the value-type adapter."""
        p, n = C.c_void_p(), C.c_uint64()
        _check(lib().crac_checkpoint_value(self._h, C.byref(p), C.byref(n)))
        try:
            return _bytes_at(p.value, n.value)
        finally:
            lib().crac_buffer_free(p)

    # ---- introspection / fixtures ----
    @property
    def fixed_va(self) -> bool:
        return bool(lib().crac_session_fixed_va(self._h))

    def debug_dump(self) -> str:
        p = C.c_char_p()
        _check(lib().crac_debug_dump(self._h, C.byref(p)))
        s = p.value.decode()
        lib().crac_buffer_free(C.cast(p, C.c_void_p))
        return s

    def log_size(self) -> int:
        n = C.c_uint64()
        _check(lib().crac_log_size(self._h, C.byref(n)))
        return n.value

    def live_records(self) -> list[LiveRecord]:
        n = C.c_uint64()
        _check(lib().crac_live_records(self._h, 0, None, None, None, None, C.byref(n)))
        k = n.value
        ids, kinds = (C.c_uint64 * max(k, 1))(), (C.c_uint8 * max(k, 1))()
        sizes, addrs = (C.c_uint64 * max(k, 1))(), (C.c_uint64 * max(k, 1))()
        _check(lib().crac_live_records(self._h, k, ids, kinds, sizes, addrs, C.byref(n)))
        return [LiveRecord(ids[i], kinds[i], sizes[i], addrs[i]) for i in range(k)]

    def managed_pages(self, alloc_id: int) -> list[int]:
        n = C.c_uint64()
        _check(lib().crac_managed_pages(self._h, alloc_id, 0, None, C.byref(n)))
        flags = (C.c_uint8 * max(n.value, 1))()
        _check(lib().crac_managed_pages(self._h, alloc_id, n.value, flags, C.byref(n)))
        return list(flags[: n.value])

    def read_raw(self, address: int, n: int) -> bytes:
        out = C.create_string_buffer(max(n, 1))
        _check(lib().crac_read_raw(self._h, address, n, out))
        return out.raw[:n]

    def backing_ptr(self, alloc_id: int) -> int:
        p = C.c_uint64()
        _check(lib().crac_backing_ptr(self._h, alloc_id, C.byref(p)))
        return p.value

    def fill_synthetic(self, alloc_id: int, seed: int, side: int = DEVICE_SIDE) -> None:
        _check(lib().crac_fill_synthetic(self._h, alloc_id, seed, side))

    def mutate(self, seed: int, epoch: int, threshold: int) -> int:
        n = C.c_uint64()
        _check(lib().crac_mutate_device(self._h, seed, epoch, threshold, C.byref(n)))
        return n.value

    def verify_synthetic(self, seed: int) -> dict:
        """Every live Device allocation compared on the GPU with the synthetic
        content fill_synthetic(id, seed) wrote."""
        bad, nb = C.c_uint64(), C.c_uint64()
        _check(lib().crac_session_verify_synthetic(self._h, seed, C.byref(bad), C.byref(nb)))
        return {"bad_allocations": bad.value, "bytes_checked": nb.value}

    def hash_only(self) -> dict:
        st = Stats()
        _check(lib().crac_hash_session(self._h, C.byref(st)))
        return st.as_dict()

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().crac_session_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def compress_image_gpu(image=None, address: Optional[tuple[int, int]] = None,
                       want_bytes: bool = True):
    """crac_compress_image_gpu: (CRACSIMZ bytes from the GPU deflate, ms);
    `address` = (ptr, size) compresses an image in place (e.g. a pinned one);
    want_bytes=False returns (compressed size, ms) without copying it out."""
    if address is not None:
        p, n, keep = C.c_void_p(address[0]), address[1], None
    else:
        p, n, keep = _buf(image)
    out, on, ms = C.c_void_p(), C.c_uint64(), C.c_double()
    _check(lib().crac_compress_image_gpu(p, n, C.byref(out), C.byref(on), C.byref(ms)))
    try:
        if not want_bytes:
            return on.value, ms.value
        return _bytes_at(out.value, on.value), ms.value
    finally:
        lib().crac_buffer_free(out)


def verify_image(image=None, synth_seed: Optional[int] = None, threads: int = 0,
                 address: Optional[tuple[int, int]] = None) -> dict:
    """crac_image_verify: host-only check of an image (section CRCs recomputed
    on `threads` cores; with synth_seed, Device payloads against regenerated
    synthetic content).  `address` = (ptr, size) checks an image in place."""
    if address is not None:
        p, n, keep = C.c_void_p(address[0]), address[1], None
    else:
        p, n, keep = _buf(image)
    rep = VerifyReport()
    _check(lib().crac_image_verify(p, n, threads, synth_seed or 0, int(synth_seed is not None),
                                   C.byref(rep)))
    return rep.as_dict()


def probe_managed_populate(nbytes: int, run: int = 1 << 20, threads: int = 0) -> float:
    """crac_probe_managed_populate: ms to first-touch fresh managed memory with
    split residence (GPU: even runs, host threads: odd runs), both at once."""
    ms = C.c_double()
    _check(lib().crac_probe_managed_populate(nbytes, run, threads, C.byref(ms)))
    return ms.value


def restart(image, mode: int = DIRECT) -> tuple[Session, dict]:
    """restart_image: strict parse + replay + GPU refill + CRC verify."""
    p, n, keep = _buf(image)
    h, st = C.c_void_p(), Stats()
    _check(lib().crac_restart(p, n, mode, C.byref(h), C.byref(st)))
    return Session(_handle=h), st.as_dict()


def restart_from_address(addr: int, n: int, mode: int = DIRECT) -> tuple[Session, dict]:
    """Zero-copy restart from an image already in (pinned) host memory."""
    h, st = C.c_void_p(), Stats()
    _check(lib().crac_restart(C.c_void_p(addr), n, mode, C.byref(h), C.byref(st)))
    return Session(_handle=h), st.as_dict()


def restart_from_file(path, image: Optional[Image] = None,
                      mode: int = DIRECT) -> tuple[Session, dict, dict]:
    """restart_from_file: parallel read into the pinned `image`, then the GPU
    refill.  Returns (session, refill stats, io stats)."""
    img = image or Image()
    h, st, io = C.c_void_p(), Stats(), IoStats()
    _check(lib().crac_restart_from_file(str(path).encode(), img._h, mode, C.byref(h),
                                        C.byref(st), C.byref(io)))
    return Session(_handle=h), st.as_dict(), io.as_dict()


def write_file(path, data, threads: int = 0, chunk_bytes: int = 0, direct: bool = True,
               sync: bool = True) -> dict:
    """The parallel image-file writer on any host buffer (no GPU involved)."""
    p, n, keep = _buf(data)
    io = IoStats()
    _check(lib().crac_file_write(str(path).encode(), p, n, threads, chunk_bytes,
                                 int(direct) | (int(sync) << 1), C.byref(io)))
    return io.as_dict()


def read_file(path, threads: int = 0, chunk_bytes: int = 0, direct: bool = True,
              offset: int = 0) -> tuple[bytes, dict]:
    """The parallel image-file reader into a host buffer that starts `offset`
    bytes past a 4 KiB boundary (no GPU involved)."""
    n = C.c_uint64()
    _check(lib().crac_file_size(str(path).encode(), C.byref(n)))
    cap = (n.value + 8191) // 4096 * 4096 + offset
    raw = C.create_string_buffer(cap + 4096)
    base = (C.addressof(raw) + 4095) // 4096 * 4096 + offset
    got, io = C.c_uint64(), IoStats()
    _check(lib().crac_file_read(str(path).encode(), C.c_void_p(base), cap - offset, threads,
                                chunk_bytes, int(direct), C.byref(got), C.byref(io)))
    return _bytes_at(base, got.value), io.as_dict()


def drop_arena_cache(device: int = -1, release_later: bool = False) -> None:
    """Frees the arena a closed session left cached on `device`: the next
    restart maps its memory afresh, as a restart in a new process does.
    release_later: only the VA is freed now; the physical memory is released
    on a thread and the next restart's arena map waits for it (the release
    overlaps the restart's first copies)."""
    if release_later:
        _check(lib().crac_drop_arena_cache_async(device))
    else:
        _check(lib().crac_drop_arena_cache(device))


def decode_check(image) -> None:
    p, n, keep = _buf(image)
    _check(lib().crac_decode_check(p, n))


def summarize_image(image) -> dict:
    p, n, keep = _buf(image)
    lengths, crcs, totals = (C.c_uint64 * 7)(), (C.c_uint32 * 7)(), (C.c_uint64 * 5)()
    _check(lib().crac_summarize(p, n, lengths, crcs, totals))
    return {"lengths": list(lengths), "crcs": list(crcs), "log_entries": totals[0],
            "active_allocations": totals[1], "payload_bytes": totals[2],
            "uvm_page_bytes": totals[3], "file_bytes": totals[4]}


def hash_chunks(data, chunk_bytes: int = 65536) -> list[int]:
    """K1 on the GPU over a host buffer: CRC-32 of every chunk."""
    p, n, keep = _buf(data)
    k = (n + chunk_bytes - 1) // chunk_bytes
    out = (C.c_uint32 * max(k, 1))()
    _check(lib().crac_hash_host_buffer(p, n, chunk_bytes, out))
    return list(out[:k])
