"""GPU tier: image persistence — checkpoint_to_file /
restart_from_file through the C-ABI against the reference's own file path
(ref: src/ckpt_engine.cpp:63-65,173-177; src/image.cpp:432-451).

Bar: the file our drain writes is byte-identical to the file the reference
writes for the same call sequence (plain and CRACSIMZ-compressed); each side
restarts from the other's file; a restart from a file reproduces the state;
damaged or missing files are refused with ImageCorrupt.
"""
import os

import pytest

import workloads
from oracle import ref

pytestmark = pytest.mark.gpu


def _pair(eng, seed=1, arena=1 << 22):
    s = eng.Session(seed=seed, arena_bytes=arena)
    r = ref.RefSession(seed=seed, arena_bytes=arena)
    for api in (s, r):
        workloads.drive_small(api, seed=seed + 3)
    return s, r


@pytest.mark.parametrize("compress", [False, True])
def test_file_equals_reference_file(eng, tmp_path, compress):
    s, r = _pair(eng)
    ours, theirs = tmp_path / "ours.img", tmp_path / "theirs.img"
    img = eng.Image()
    drain, io = s.checkpoint_to_file(ours, img, compress=compress)
    ref.ref_checkpoint_to_file(r, theirs, compress=compress)
    assert ours.read_bytes() == theirs.read_bytes()
    assert io["bytes"] == ours.stat().st_size
    if not compress:
        assert ours.read_bytes() == img.tobytes()
        assert drain["image_bytes"] == io["bytes"]
    else:
        assert ours.read_bytes()[:8] == b"CRACSIMZ"


@pytest.mark.parametrize("compress", [False, True])
def test_cross_restart_from_files(eng, tmp_path, compress):
    s, r = _pair(eng, seed=5)
    ours, theirs = tmp_path / "ours.img", tmp_path / "theirs.img"
    s.checkpoint_to_file(ours, compress=compress)
    ref.ref_checkpoint_to_file(r, theirs, compress=compress)
    want = s.checkpoint()[0]
    # ours from the reference's file, the reference from ours
    a, refill, io = eng.restart_from_file(theirs)
    assert a.checkpoint()[0] == want
    assert refill["h2d_bytes"] > 0 and io["bytes"] == theirs.stat().st_size
    b, _ = ref.ref_restart_from_file(ours)
    assert b.checkpoint()[0] == want


def test_multi_piece_file_round_trip(eng, tmp_path):
    """Regions spanning several I/O pieces, odd sizes so the bulk stream sits
    at an unaligned file offset (the O_DIRECT bounce path), 2 restarts deep."""
    s = eng.Session(seed=7, arena_bytes=256 << 20)
    workloads.build_regions(s, 6, lambda k: (24 << 20) + 4096 * k + k * 7 + 1, seed=7)
    p = tmp_path / "big.img"
    img = eng.Image()
    drain, io = s.checkpoint_to_file(p, img)
    want = img.tobytes()
    assert p.read_bytes() == want
    staging = eng.Image()
    r, refill, rio = eng.restart_from_file(p, staging)
    assert rio["bytes"] == len(want) and staging.tobytes() == want
    p2 = tmp_path / "big2.img"
    r.checkpoint_to_file(p2)
    assert p2.read_bytes() == want


def test_restart_from_file_refuses_damage(eng, tmp_path):
    s, _ = _pair(eng, seed=2)
    p = tmp_path / "x.img"
    s.checkpoint_to_file(p)
    data = bytearray(p.read_bytes())
    for pos in (3, len(data) // 2, len(data) - 2):
        bad = bytearray(data)
        bad[pos] ^= 0x10
        q = tmp_path / f"bad{pos}.img"
        q.write_bytes(bytes(bad))
        with pytest.raises(eng.CracError) as e:
            eng.restart_from_file(q)
        assert e.value.errc == "ImageCorrupt"
    q = tmp_path / "short.img"
    q.write_bytes(bytes(data[: len(data) - 5]))
    with pytest.raises(eng.CracError) as e:
        eng.restart_from_file(q)
    assert e.value.errc == "ImageCorrupt"
    with pytest.raises(eng.CracError) as e:
        eng.restart_from_file(tmp_path / "missing.img")
    assert e.value.errc == "ImageCorrupt"


def test_checkpoint_to_unwritable_path(eng, tmp_path):
    s, _ = _pair(eng, seed=3)
    with pytest.raises(eng.CracError) as e:
        s.checkpoint_to_file(tmp_path / "none" / "x.img")
    assert e.value.errc == "InvalidArgument"
    # the session is untouched and still drains
    assert s.checkpoint()[0]


def test_streamed_write_under_the_drain(eng, tmp_path, monkeypatch):
    """CRAC_FILE_STREAM=1: checkpoint_to_file writes the file while the
    drain's windows land (StreamWriter): 1 MiB pieces so most of the file streams under the D2H;
    the leading sections, crc3 and the tail are written again once final.
    Over a longer stale file (in place, cut to size); the same bytes as the
    drain-then-write path, and the reference restarts from it."""
    monkeypatch.setenv("CRAC_IO_CHUNK_MIB", "1")
    monkeypatch.setenv("CRAC_FILE_STREAM", "1")
    s = eng.Session(seed=11, arena_bytes=512 << 20)
    workloads.build_regions(s, 5, lambda k: (64 << 20) + 4096 * k + 3 * k + 5, seed=11)
    p = tmp_path / "streamed.img"
    p.write_bytes(os.urandom(1 << 20) * 400)  # longer than the image, garbage
    img = eng.Image()
    drain, io = s.checkpoint_to_file(p, img)
    want = img.tobytes()
    assert p.read_bytes() == want
    assert io["bytes"] == len(want) and io["streamed"] > 0, io
    monkeypatch.delenv("CRAC_FILE_STREAM")
    q = tmp_path / "plain.img"
    _, io2 = s.checkpoint_to_file(q)
    assert io2["streamed"] == 0 and q.read_bytes() == want
    b, _ = ref.ref_restart_from_file(p)
    assert b.checkpoint()[0] == want
