"""GPU tier: cudart interposition — a plain CUDA application
(tests/native/interpose_app.cu, shared cudart, no cracsim code) run under
LD_PRELOAD=libcrac_preload.so.

Bar:
* the application runs unchanged, its kernel launches pass through the
  dispatch gate, and its allocation-family calls become the session's log;
* the image it checkpoints is the reference's image of the same call
  sequence (ref: src/shim.cpp:204-253 fed the same calls, contents stored
  with copy_h2d): META / LOG / ALLOC_PAYLOADS / STREAMS / REGISTRY byte-equal,
  managed page records equal in identity and flags, with the application's
  bytes as content (the reference, having no real device, holds zeros there);
* a second process restarted from the file finds its device buffers at the
  same pointers and every byte intact (verified by its own kernels);
* the reference restarts from the same file.
"""
import os
import struct
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import image_oracle as io
from oracle import ref

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
APP = ROOT / "build" / "interpose_app"
PRELOAD = ROOT / "paper_2008_10596_b200" / "libcrac_preload.so"
ARENA = 1 << 30
KA, KB, KM, KH = 3 * 1024 * 1024 + 12, 1000003, 6 * 4096 + 100, 70000


@pytest.fixture(scope="module")
def built():
    if not (APP.exists() and PRELOAD.exists()):
        from paper_2008_10596_b200 import build
        build.build()
    return APP


def _run(args, **env):
    e = dict(os.environ)
    e.update({k: str(v) for k, v in env.items()})
    return subprocess.run([str(APP), *args], env=e, capture_output=True, text=True, timeout=300)


def expected():
    i = np.arange(KA, dtype=np.uint64)
    a = ((i % 65536).astype(np.float32) * np.float32(0.5) + np.float32(1.0)).tobytes()
    b = ((np.arange(KB, dtype=np.uint64) * 7 + 3) & 0xFF).astype(np.uint8).tobytes()
    j = np.arange(KM, dtype=np.uint64)
    m = np.where(j < KM // 2, (j * 13 + 1) & 0xFF, (j ^ 0xA5) & 0xFF).astype(np.uint8).tobytes()
    h = ((np.arange(KH, dtype=np.uint64) * 3 + 11) & 0xFF).astype(np.uint8).tobytes()
    return a, b, m, h


def test_app_runs_natively(built):
    r = _run(["run", "/nonexistent"])
    assert r.returncode == 0, r.stderr
    assert "no preload" in r.stdout


def test_interposed_checkpoint_matches_reference_and_restarts(built, tmp_path):
    img = tmp_path / "app.img"
    r = _run(["run", img], LD_PRELOAD=PRELOAD, CRAC_ARENA_BYTES=ARENA, CRAC_PRELOAD_VERBOSE=1)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "checkpointed" in r.stdout
    counters = [ln for ln in r.stderr.splitlines() if ln.startswith("crac_preload: allocs")][0]
    allocs, frees, gated = (int(counters.split()[k]) for k in (2, 4, 6))
    assert (allocs, frees) == (5, 1) and gated >= 4, counters  # 4 launches at least
    # device pointers are arena addresses (fixed VA = the reference's kArenaBase)
    ptrs = dict(kv.split("=") for kv in r.stdout.split("\n")[0].split())
    assert int(ptrs["a"], 16) == 0x0D00_0000_0000

    data = img.read_bytes()
    ours = io.decode_image(data)
    a, b, m, h = expected()

    # the reference fed the same calls (cudaStreamCreate x2, cudaMalloc a/tmp/b,
    # cudaFree tmp, cudaMallocManaged m, cudaMallocHost h) and the same bytes
    rs = ref.RefSession(seed=0, arena_bytes=ARENA)
    rs.stream_create()
    rs.stream_create()
    ia, _ = rs.alloc(1, KA * 4)
    it, _ = rs.alloc(1, 1000)
    ib, _ = rs.alloc(1, KB)
    rs.free(it)
    im, _ = rs.alloc(3, KM)
    ih, _ = rs.alloc(2, KH)
    rs.copy_h2d(ia, 0, a)
    rs.copy_h2d(ib, 0, b)
    rs.copy_h2d(ih, 0, h)
    rs.set_app_state(ours.app_state)
    theirs = io.decode_image(rs.checkpoint()[0])

    assert (ours.seed, ours.arena_bytes, ours.engine_version) == \
        (theirs.seed, theirs.arena_bytes, theirs.engine_version)
    assert ours.log == theirs.log
    assert ours.payloads == theirs.payloads
    assert ours.streams == theirs.streams
    assert ours.binaries == theirs.binaries
    assert [(i, [(x, d, y) for (x, d, y, _) in pg]) for (i, pg) in ours.managed] == \
        [(i, [(x, d, y) for (x, d, y, _) in pg]) for (i, pg) in theirs.managed]
    assert b"".join(c for (_, pg) in ours.managed for (_, _, _, c) in pg)[:KM] == m
    ref.ref_decode_check(data)  # the reference accepts the file as is

    # a new process restarts from the file and checks every byte itself
    r2 = _run(["resume"], LD_PRELOAD=PRELOAD, CRAC_RESTART_FROM=img, CRAC_PRELOAD_VERBOSE=1)
    assert r2.returncode == 0, r2.stdout + r2.stderr
    assert "mismatches 0, host-visible mismatches 0" in r2.stdout
    assert "(restarted)" in r2.stderr

    # the reference restarts from it too, and re-encodes it unchanged
    back, _ = ref.ref_restart_from_file(img)
    assert back.checkpoint()[0] == data


def test_sigusr2_checkpoint_of_a_running_app(built, tmp_path):
    """The asynchronous trigger: SIGUSR2 while the application keeps two
    streams busy; the checkpoint thread quiesces it (gate + device-wide
    drain), writes CRAC_CKPT_PATH, and the application carries on.  The image
    restarts into a process that finds every byte."""
    import signal
    import time
    img = tmp_path / "async.img"
    e = dict(os.environ, LD_PRELOAD=str(PRELOAD), CRAC_ARENA_BYTES=str(ARENA),
             CRAC_CKPT_PATH=str(img), CRAC_PRELOAD_VERBOSE="1")
    p = subprocess.Popen([str(APP), "spin", "4000"], env=e, stdout=subprocess.PIPE,
                         stderr=subprocess.PIPE, text=True)
    assert p.stdout.readline().startswith("a=")
    assert p.stdout.readline().strip() == "spinning"
    time.sleep(1.0)
    p.send_signal(signal.SIGUSR2)
    out, err = p.communicate(timeout=300)
    assert p.returncode == 0, out + err
    assert "checkpoints 1" in err, err
    data = img.read_bytes()
    ref.ref_decode_check(data)
    ours = io.decode_image(data)
    a, b, m, h = expected()
    assert [x[1] for x in ours.payloads] == [a, b, h]  # quiesced: no torn kernel output
    r2 = _run(["resume"], LD_PRELOAD=PRELOAD, CRAC_RESTART_FROM=img)
    assert r2.returncode == 0, r2.stdout + r2.stderr


def test_sigusr2_precopy_checkpoint_of_a_device_only_app(built, tmp_path):
    """Device memory only: the preload's checkpoint is a pre-copy (the state
    is copied while the application keeps rewriting it, then only what
    changed is re-sent under the gate).  The image restarts into a process
    that finds every byte, and the reference accepts it."""
    import signal
    import time
    img = tmp_path / "dev.img"
    e = dict(os.environ, LD_PRELOAD=str(PRELOAD), CRAC_ARENA_BYTES=str(ARENA),
             CRAC_CKPT_PATH=str(img), CRAC_PRELOAD_VERBOSE="1")
    p = subprocess.Popen([str(APP), "devspin", "4000"], env=e, stdout=subprocess.PIPE,
                         stderr=subprocess.PIPE, text=True)
    assert p.stdout.readline().startswith("a=")
    assert p.stdout.readline().strip() == "spinning"
    time.sleep(1.0)
    p.send_signal(signal.SIGUSR2)
    out, err = p.communicate(timeout=300)
    assert p.returncode == 0, out + err
    assert "checkpoints 1" in err, err
    data = img.read_bytes()
    ref.ref_decode_check(data)
    a, b, _, _ = expected()
    assert [x[1] for x in io.decode_image(data).payloads] == [a, b]
    r2 = _run(["devresume"], LD_PRELOAD=PRELOAD, CRAC_RESTART_FROM=img)
    assert r2.returncode == 0, r2.stdout + r2.stderr
