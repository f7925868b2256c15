"""CPU tier: host-side C++ logic of the engine, compiled natively here.

* HoleIndex (O(log n) first fit) vs the reference's linear first fit with
  two-sided coalescing (ref: src/device_core.cpp:45-103).
* RegionMap vs the reference's region table (ref: src/shim.cpp:42-88).
"""
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_hole_index_matches_reference_first_fit(tmp_path):
    exe = tmp_path / "hole_index_test"
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "native" / "hole_index_test.cpp"), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe), "60"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.strip() == "ok"


def test_region_map_matches_reference_table(tmp_path):
    """RegionMap (csrc/shim.cpp) vs the reference's region table: its own
    test_shim.cpp cases, then random register/classify sequences against a
    restatement of ref src/shim.cpp:42-88 (same regions, Errc, classes)."""
    from paper_2008_10596_b200 import engine
    if not engine.LIB_PATH.exists():
        from paper_2008_10596_b200 import build
        build.build()
    exe = tmp_path / "region_map_test"
    lib_dir = engine.LIB_PATH.parent
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"),
                    "-I", "/usr/local/cuda/include",
                    str(ROOT / "tests" / "native" / "region_map_test.cpp"), "-o", str(exe),
                    "-L", str(lib_dir), "-lcrac_b200", f"-Wl,-rpath,{lib_dir}"],
                   check=True)
    out = subprocess.run([str(exe), "300"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.strip() == "ok"


def _build_dropin(tmp_path):
    from paper_2008_10596_b200 import engine
    if not engine.LIB_PATH.exists():
        from paper_2008_10596_b200 import build
        build.build()
    exe = tmp_path / "dropin_test"
    lib_dir = engine.LIB_PATH.parent
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"),
                    "-I", "/usr/local/cuda/include",
                    str(ROOT / "tests" / "native" / "dropin_test.cpp"), "-o", str(exe),
                    "-L", str(lib_dir), "-lcrac_b200", f"-Wl,-rpath,{lib_dir}"],
                   check=True)
    return exe


def test_reference_style_client_compiles_against_dropin_headers(tmp_path):
    """A client written against the reference's C++ API (test_ckpt_engine.cpp
    shapes) compiles and links unchanged against include/cracsim + the .so."""
    assert _build_dropin(tmp_path).exists()


import pytest  # noqa: E402


@pytest.mark.gpu
def test_reference_style_client_runs_on_b200(tmp_path):
    exe = _build_dropin(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.strip().endswith("ok")


def test_host_crc_is_zlib():
    """crac_crc32_host (PCLMUL folding, crc_host.cpp) == zlib.crc32 for every
    length around the 16/64-byte fold boundaries, any alignment and seed."""
    import ctypes
    import os
    import zlib

    from paper_2008_10596_b200 import engine
    if not engine.LIB_PATH.exists():
        from paper_2008_10596_b200 import build
        build.build()
    lib = engine.lib()
    buf = os.urandom(1 << 16)
    cbuf = ctypes.create_string_buffer(buf, len(buf))
    base = ctypes.addressof(cbuf)
    for n in list(range(0, 300)) + [4095, 4096, 4097, 65536 - 16]:
        for off in (0, 1, 5, 15):
            for seed in (0, 0xDEADBEEF):
                got = lib.crac_crc32_host(ctypes.c_void_p(base + off), n, seed)
                assert got == zlib.crc32(buf[off:off + n], seed), (n, off, seed)


def test_host_crc_copy_is_zlib_and_memcpy():
    """crac_crc32_copy_host (the drain's host-page move: one read, PCLMUL
    fold + non-temporal stores) returns zlib's CRC of the source and leaves an
    exact copy, for every destination phase (16-byte aligned: streamed; else
    memcpy) and lengths around the fold boundaries."""
    import ctypes
    import os
    import zlib

    from paper_2008_10596_b200 import engine
    if not engine.LIB_PATH.exists():
        from paper_2008_10596_b200 import build
        build.build()
    lib = engine.lib()
    buf = os.urandom(1 << 16)
    src = ctypes.create_string_buffer(buf, len(buf))
    dst = ctypes.create_string_buffer(len(buf) + 64)
    sbase, dbase = ctypes.addressof(src), ctypes.addressof(dst)
    dpad = (-dbase) % 16  # dst + dpad is 16-byte aligned
    for n in list(range(0, 200)) + [4095, 4096, 4097, 65536 - 64]:
        for soff in (0, 3):
            for doff in (dpad, dpad + 16, dpad + 1):
                ctypes.memset(dbase, 0xA5, len(buf) + 64)
                got = lib.crac_crc32_copy_host(ctypes.c_void_p(dbase + doff), ctypes.c_void_p(sbase + soff),
                                               n, 7)
                assert got == zlib.crc32(buf[soff:soff + n], 7), (n, soff, doff)
                out = ctypes.string_at(dbase, len(buf) + 64)
                assert out[doff:doff + n] == buf[soff:soff + n], (n, soff, doff)
                assert out[doff + n:doff + n + 16] == b"\xa5" * len(out[doff + n:doff + n + 16])
                assert out[:doff] == b"\xa5" * doff
