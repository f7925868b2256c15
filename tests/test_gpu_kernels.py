"""GPU tier: the kernel-level C-ABI (include/crac_gpu.h) on its own, with
device buffers owned by the caller (torch here), checked against host
restatements of what each kernel must produce.
"""
import ctypes as C
import random
import struct
import zlib

import pytest

from oracle import ref

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _p(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


def _spans(buffers):
    """crac_span_t array + chunk_first for a list of device byte tensors."""
    raw = b"".join(struct.pack("<QQ", b.data_ptr(), b.numel()) for b in buffers)
    return torch.frombuffer(bytearray(raw), dtype=torch.uint8).cuda()


def _first(buffers, chunk):
    f = [0]
    for b in buffers:
        f.append(f[-1] + (b.numel() + chunk - 1) // chunk)
    return torch.tensor(f, dtype=torch.int64).cuda(), f


def _rand(n, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.randint(0, 256, (n,), dtype=torch.uint8, generator=g)


def test_chunk_crc32_range_and_multi_span(eng):
    L = eng.lib()
    bufs = [_rand(n, k).cuda() for k, n in enumerate([65536 * 3 + 5, 512, 4096 * 7 + 511, 1])]
    spans = _spans(bufs)
    first_d, first = _first(bufs, 4096)
    out = torch.zeros(first[-1], dtype=torch.int32).cuda()
    # two launches over absolute sub-ranges must equal one launch over all
    mid = first[-1] // 2
    for lo, hi in ((0, mid), (mid, first[-1])):
        assert L.crac_chunk_crc32_range(_p(spans), _p(first_d), len(bufs), 4096, lo, hi, _p(out),
                                        7, None) == 0
    torch.cuda.synchronize()
    want = []
    for b in bufs:
        h = bytes(b.cpu().numpy())
        want += [zlib.crc32(h[i:i + 4096]) for i in range(0, len(h), 4096)]
    assert [x & 0xFFFFFFFF for x in out.cpu().tolist()] == want


@pytest.mark.parametrize("dirty_pct", [0, 3, 50, 100])
def test_diff_compact_is_ordered_and_updates_prev(eng, dirty_pct):
    L = eng.lib()
    n = 10000 + 123
    rnd = random.Random(dirty_pct)
    prev = [rnd.getrandbits(32) for _ in range(n)]
    new = [p if rnd.randrange(100) >= dirty_pct else p ^ 1 for p in prev]
    to32 = lambda v: torch.tensor([x - (1 << 32) if x >= 1 << 31 else x for x in v],
                                  dtype=torch.int32).cuda()
    d_new, d_prev = to32(new), to32(prev)
    counts = torch.zeros(8, dtype=torch.int32).cuda()
    idx = torch.zeros(n, dtype=torch.int64).cuda()
    cnt = torch.zeros(1, dtype=torch.int64).cuda()
    assert L.crac_diff_compact(_p(d_new), _p(d_prev), n, _p(counts), _p(idx), _p(cnt), None) == 0
    torch.cuda.synchronize()
    want = [i for i in range(n) if new[i] != prev[i]]
    assert cnt.item() == len(want)
    assert idx[: len(want)].cpu().tolist() == want
    assert d_prev.cpu().tolist() == d_new.cpu().tolist()
    # the range form writes absolute indices
    d_prev2 = to32(prev)
    assert L.crac_diff_compact_range(_p(d_new), _p(d_prev2), 5000, n, _p(counts), _p(idx),
                                     _p(cnt), None) == 0
    torch.cuda.synchronize()
    want2 = [i for i in want if i >= 5000]
    assert idx[: len(want2)].cpu().tolist() == want2


def test_gather_to_device_and_to_host(eng):
    L = eng.lib()
    chunk = 65536
    bufs = [_rand(chunk * 5 + 77, 1).cuda(), _rand(chunk * 2, 2).cuda()]
    spans = _spans(bufs)
    first_d, first = _first(bufs, chunk)
    dirty = [0, 3, 5, 6]  # chunk 5 is span 0's 77-byte tail, 6 starts span 1
    d_idx = torch.tensor(dirty, dtype=torch.int64).cuda()
    staging = torch.zeros(len(dirty) * chunk, dtype=torch.uint8).cuda()
    assert L.crac_gather_chunks(_p(spans), _p(first_d), 2, chunk, _p(d_idx), 0, len(dirty),
                                _p(staging), None) == 0
    host = [bytes(b.cpu().numpy()) for b in bufs]

    def chunk_bytes(c):
        s = 0 if c < first[1] else 1
        off = (c - first[s]) * chunk
        return host[s][off:off + chunk]

    torch.cuda.synchronize()
    st = bytes(staging.cpu().numpy())
    for k, c in enumerate(dirty):
        cb = chunk_bytes(c)
        assert st[k * chunk:k * chunk + len(cb)] == cb
    # direct-to-host at misaligned image offsets
    image = torch.zeros(len(host[0]) + len(host[1]) + 64, dtype=torch.uint8).pin_memory()
    offs = [3, 3 + len(host[0]) + 16]
    d_off = torch.tensor(offs, dtype=torch.int64).cuda()
    cnt = torch.tensor([len(dirty)], dtype=torch.int64).cuda()
    assert L.crac_gather_chunks_to_host_dev(_p(spans), _p(first_d), 2, chunk, _p(d_idx), _p(cnt),
                                            len(dirty), 0, _p(d_off), _p(image), None) == 0
    torch.cuda.synchronize()
    img = bytes(image.numpy())
    for c in dirty:
        s = 0 if c < first[1] else 1
        off = (c - first[s]) * chunk
        cb = chunk_bytes(c)
        assert img[offs[s] + off:offs[s] + off + len(cb)] == cb


def test_fused_hash_drain_writes_only_changed_chunks(eng):
    L = eng.lib()
    chunk = 65536
    buf = _rand(chunk * 9 + 1000, 3).cuda()
    spans = _spans([buf])
    first_d, first = _first([buf], chunk)
    n = first[-1]
    crc = torch.zeros(n, dtype=torch.int32).cuda()
    prev = torch.zeros(n, dtype=torch.int32).cuda()
    image = torch.zeros(buf.numel() + 32, dtype=torch.uint8).pin_memory()
    d_off = torch.tensor([16], dtype=torch.int64).cuda()
    counters = torch.zeros(2, dtype=torch.int64).cuda()
    args = lambda: (_p(spans), _p(first_d), 1, chunk, 0, n, _p(crc), _p(prev), None, None,
                    _p(d_off), _p(image), _p(counters), None)
    assert L.crac_hash_drain_range(*args()) == 0  # prev all zero: everything is dirty
    torch.cuda.synchronize()
    data = bytes(buf.cpu().numpy())
    assert bytes(image.numpy())[16:16 + len(data)] == data
    assert counters.cpu().tolist() == [n, len(data)]
    assert [x & 0xFFFFFFFF for x in crc.cpu().tolist()] == \
        [zlib.crc32(data[i:i + chunk]) for i in range(0, len(data), chunk)]
    # change two chunks; only they are rewritten
    image.zero_()
    buf[chunk * 2 + 5] ^= 0xFF
    buf[chunk * 9 + 999] ^= 0x01
    counters.zero_()
    assert L.crac_hash_drain_range(*args()) == 0
    torch.cuda.synchronize()
    data = bytes(buf.cpu().numpy())
    img = bytes(image.numpy())
    assert counters.cpu().tolist() == [2, chunk + 1000]
    assert img[16 + 2 * chunk:16 + 3 * chunk] == data[2 * chunk:3 * chunk]
    assert img[16 + 9 * chunk:16 + len(data)] == data[9 * chunk:]
    assert img[16:16 + 2 * chunk] == bytes(2 * chunk)


@pytest.mark.parametrize("writers", [1, 4, 16])
def test_split_hash_drain_writes_only_changed_chunks(eng, writers):
    """crac_hash_drain_split: writer CTAs copy the chunks the hashers hand over
    (more chunks than hashing warps, ragged last chunk, odd offsets)."""
    L = eng.lib()
    chunk = 65536
    bufs = [_rand(chunk * 300 + 1000, 5).cuda(), _rand(chunk * 41 + 3, 6).cuda()]
    spans = _spans(bufs)
    first_d, first = _first(bufs, chunk)
    n = first[-1]
    crc = torch.zeros(n, dtype=torch.int32).cuda()
    prev = torch.zeros(n, dtype=torch.int32).cuda()
    total = sum(b.numel() for b in bufs)
    image = torch.zeros(total + 64, dtype=torch.uint8).pin_memory()
    offs = [16, 16 + bufs[0].numel() + 16]
    d_off = torch.tensor(offs, dtype=torch.int64).cuda()
    counters = torch.zeros(5, dtype=torch.int64).cuda()
    queue = torch.zeros(n + 16 * writers + 1, dtype=torch.int64).cuda()
    args = lambda: (_p(spans), _p(first_d), 2, chunk, 0, n, _p(crc), _p(prev), None, None,
                    _p(d_off), _p(image), _p(counters), _p(queue), writers, None)
    assert L.crac_hash_drain_split(*args()) == 0  # everything dirty
    torch.cuda.synchronize()
    img = bytes(image.numpy())
    for b, o in zip(bufs, offs):
        data = bytes(b.cpu().numpy())
        assert img[o:o + len(data)] == data
    assert counters.cpu().tolist()[:2] == [n, total]
    # a few chunks change, spread over both buffers
    image.zero_()
    counters.zero_()
    for c in (0, 7, 299, 300):
        bufs[0][c * chunk + 11] ^= 0x5A
    bufs[1][41 * chunk + 1] ^= 0x01  # the 3-byte last chunk
    assert L.crac_hash_drain_split(*args()) == 0
    torch.cuda.synchronize()
    img = bytes(image.numpy())
    assert counters.cpu().tolist()[:2] == [5, 3 * chunk + 1000 + 3]
    d0, d1 = bytes(bufs[0].cpu().numpy()), bytes(bufs[1].cpu().numpy())
    for c in (0, 7, 299):
        assert img[16 + c * chunk:16 + (c + 1) * chunk] == d0[c * chunk:(c + 1) * chunk]
    assert img[16 + 300 * chunk:16 + len(d0)] == d0[300 * chunk:]
    assert img[offs[1] + 41 * chunk:offs[1] + len(d1)] == d1[41 * chunk:]
    assert img[offs[1]:offs[1] + 41 * chunk] == bytes(41 * chunk)
    assert img[16 + chunk:16 + 2 * chunk] == bytes(chunk)  # clean chunks untouched
    assert L.crac_hash_drain_split(_p(spans), _p(first_d), 2, chunk, 0, n, _p(crc), _p(prev),
                                   None, None, _p(d_off), _p(image), _p(counters), _p(queue), 0,
                                   None) != 0


def test_pack_scatter_round_trip_random_records(eng):
    """K2a then K3 over a random framed stream, across window boundaries."""
    L = eng.lib()
    rnd = random.Random(9)
    regions, recs, pos = [], [], 0
    for k in range(40):
        size = rnd.choice([1, 15, 16, 17, 100, 4096, 70000, 200000])
        ext = (size + 255) // 256 * 256
        t = _rand(ext + 64, 100 + k).cuda()
        t[size:] = 0
        regions.append((t, size, ext))
        frame = struct.pack("<QQ", k + 1, size)
        recs.append(struct.pack("<QQQQII", pos, t.data_ptr(), size, ext, 16, 0) + frame + bytes(8))
        pos += 16 + size
    stream_len = pos
    d_recs = torch.frombuffer(bytearray(b"".join(recs)), dtype=torch.uint8).cuda()
    tile = 65536
    outs = [r[0:8] for r in recs]
    offs = [struct.unpack("<Q", o)[0] for o in outs]
    tiles = (stream_len + tile - 1) // tile
    tile_rec = []
    r = 0
    for t in range(tiles):
        while r + 1 < len(offs) and offs[r + 1] <= t * tile:
            r += 1
        tile_rec.append(r)
    d_tile = torch.tensor(tile_rec, dtype=torch.int32).cuda()
    win = 3 * tile
    packed = torch.zeros(stream_len + 64, dtype=torch.uint8).cuda()
    for w0 in range(0, stream_len, win):
        wl = min(win, stream_len - w0)
        buf = torch.zeros(win + 64, dtype=torch.uint8).cuda()
        assert L.crac_pack_records(_p(d_recs), len(recs), C.c_void_p(d_tile.data_ptr() + 4 * (w0 // tile)),
                                   w0, wl, _p(buf), None) == 0
        packed[w0:w0 + wl] = buf[:wl]
    torch.cuda.synchronize()
    want = b"".join(struct.pack("<QQ", k + 1, s) + bytes(t[:s].cpu().numpy())
                    for k, (t, s, e) in enumerate(regions))
    assert bytes(packed[:stream_len].cpu().numpy()) == want
    # windows need only 16-byte alignment
    for w0, wl in ((tile + 48, 2 * tile + 5), (16, stream_len - 16),
                   ((stream_len - 40) & ~15, stream_len - ((stream_len - 40) & ~15))):
        buf = torch.zeros(wl + 64, dtype=torch.uint8).cuda()
        assert L.crac_pack_records(_p(d_recs), len(recs), C.c_void_p(d_tile.data_ptr() + 4 * (w0 // tile)),
                                   w0, wl, _p(buf), None) == 0
        torch.cuda.synchronize()
        assert bytes(buf[:wl].cpu().numpy()) == want[w0:w0 + wl]
    # scatter back into scribbled regions
    for t, s, e in regions:
        t.fill_(0xEE)
    for w0 in range(0, stream_len, win):
        wl = min(win, stream_len - w0)
        buf = torch.zeros(win + 64, dtype=torch.uint8).cuda()
        take = min(wl + 16, stream_len - w0)
        buf[:take] = packed[w0:w0 + take]
        assert L.crac_scatter_records(_p(d_recs), len(recs), C.c_void_p(d_tile.data_ptr() + 4 * (w0 // tile)),
                                      _p(buf), w0, wl, None) == 0
    torch.cuda.synchronize()
    for k, (t, s, e) in enumerate(regions):
        got = bytes(t[:e].cpu().numpy())
        assert got[:s] == want[sum(16 + x[1] for x in regions[:k]) + 16:][:s]
        assert got[s:e] == bytes(e - s)  # padding zero-filled


@pytest.mark.parametrize("aligned", [1, 0])
def test_hash_copy_writes_every_chunk_and_hashes(eng, aligned):
    """crac_hash_copy_range: the stall-reduced snapshot's K1 (copy from the
    hashing registers) against zlib and the source bytes, tails and odd
    destination offsets included."""
    L = eng.lib()
    chunk = 65536
    sizes = [chunk * 3, chunk * 2 + 512 * 7 + 33, 511, 512, chunk + 16, 4096 * 5]
    bufs = [_rand(n, 40 + k).cuda() for k, n in enumerate(sizes)]
    spans = _spans(bufs)
    first_d, first = _first(bufs, chunk)
    offs, pos = [], 0
    for n in sizes:
        pos += 16 if aligned else 16 + 7
        offs.append(pos)
        pos += (n + 15) // 16 * 16 if aligned else n
    d_off = torch.tensor(offs, dtype=torch.int64).cuda()
    dst = torch.full((pos + 64,), 0xAB, dtype=torch.uint8).cuda()
    crc = torch.zeros(first[-1], dtype=torch.int32).cuda()
    assert L.crac_hash_copy_range(_p(spans), _p(first_d), len(bufs), chunk, 0, first[-1], _p(crc),
                                  None, _p(d_off), _p(dst), aligned, None) == 0
    torch.cuda.synchronize()
    out = bytes(dst.cpu().numpy())
    want_crc = []
    prev_end = 0
    for b, o in zip(bufs, offs):
        h = bytes(b.cpu().numpy())
        assert out[o:o + len(h)] == h
        assert out[prev_end:o] == b"\xAB" * (o - prev_end)  # nothing outside the payloads
        prev_end = o + len(h)
        want_crc += [zlib.crc32(h[i:i + chunk]) for i in range(0, len(h), chunk)]
    assert [x & 0xFFFFFFFF for x in crc.cpu().tolist()] == want_crc


@pytest.mark.parametrize("chunk", [512, 4096, 65536])
def test_chunk_key_matches_restatement(eng, chunk):
    """crac_chunk_key_range: CRC lane == zlib, key lane == tests/dirtykey.py
    (whatever row batching the chunk size selects), ragged tails included."""
    from dirtykey import chunk_keys
    L = eng.lib()
    sizes = [chunk * 3 + 5, 511, 512, 17, chunk * 2 + 512 * 3 + 33, 1]
    bufs = [_rand(n, 70 + k).cuda() for k, n in enumerate(sizes)]
    spans = _spans(bufs)
    first_d, first = _first(bufs, chunk)
    crc = torch.zeros(first[-1], dtype=torch.int32).cuda()
    key = torch.zeros(first[-1], dtype=torch.int32).cuda()
    assert L.crac_chunk_key_range(_p(spans), _p(first_d), len(bufs), chunk, 0, first[-1], _p(crc),
                                  _p(key), 0, None) == 0
    torch.cuda.synchronize()
    want_crc, want_key = [], []
    for b in bufs:
        h = bytes(b.cpu().numpy())
        want_crc += [zlib.crc32(h[i:i + chunk]) for i in range(0, len(h), chunk)]
        want_key += chunk_keys(h, chunk)
    assert [x & 0xFFFFFFFF for x in crc.cpu().tolist()] == want_crc
    assert [x & 0xFFFFFFFF for x in key.cpu().tolist()] == want_key


@pytest.mark.parametrize("split", [False, True])
def test_forged_crc_collision_is_resent_with_keys(eng, split):
    """A change that keeps a chunk's CRC-32 (4 compensating bytes) is missed
    by a CRC-only dirty check and caught by the 64-bit dirty key."""
    from dirtykey import chunk_key, forge_crc
    L = eng.lib()
    chunk = 65536
    buf = _rand(chunk * 40 + 77, 11).cuda()
    spans = _spans([buf])
    first_d, first = _first([buf], chunk)
    n = first[-1]
    d_off = torch.tensor([16], dtype=torch.int64).cuda()
    image = torch.zeros(buf.numel() + 64, dtype=torch.uint8).pin_memory()
    crc, key = torch.zeros(n, dtype=torch.int32).cuda(), torch.zeros(n, dtype=torch.int32).cuda()
    counters = torch.zeros(5, dtype=torch.int64).cuda()
    queue = torch.zeros(n + 16 * 4 + 1, dtype=torch.int64).cuda()

    def run(prev, prev_key, with_key):
        counters.zero_()
        k = (_p(key), _p(prev_key)) if with_key else (None, None)
        if split:
            rc = L.crac_hash_drain_split(_p(spans), _p(first_d), 1, chunk, 0, n, _p(crc), _p(prev),
                                         *k, _p(d_off), _p(image), _p(counters), _p(queue), 4, None)
        else:
            rc = L.crac_hash_drain_range(_p(spans), _p(first_d), 1, chunk, 0, n, _p(crc), _p(prev),
                                         *k, _p(d_off), _p(image), _p(counters), None)
        assert rc == 0
        torch.cuda.synchronize()
        return counters.cpu().tolist()[0]

    prev, prev_key = torch.zeros(n, dtype=torch.int32).cuda(), torch.zeros(n, dtype=torch.int32).cuda()
    assert run(prev, prev_key, True) == n  # seeds both lanes
    data = bytearray(buf.cpu().numpy().tobytes())
    assert [x & 0xFFFFFFFF for x in prev_key.cpu().tolist()] == \
        [chunk_key(bytes(data[i:i + chunk])) for i in range(0, len(data), chunk)]
    # forge chunk 17: one byte flipped, 4 bytes compensate the CRC
    c = 17
    piece = bytearray(data[c * chunk:(c + 1) * chunk])
    target = zlib.crc32(piece)
    piece[1000] ^= 0x80
    forge_crc(piece, 5000, target)
    buf[c * chunk:(c + 1) * chunk] = torch.frombuffer(bytearray(piece), dtype=torch.uint8).cuda()
    # CRC lane only: the change is invisible
    prev_crc_only = prev.clone()
    image.zero_()
    assert run(prev_crc_only, None, False) == 0
    # the 64-bit key sees it and re-sends exactly that chunk
    assert run(prev, prev_key, True) == 1
    img = bytes(image.numpy())
    assert img[16 + c * chunk:16 + (c + 1) * chunk] == bytes(piece)
    assert img[16:16 + c * chunk] == bytes(c * chunk)


@pytest.mark.parametrize("env", [{"CRAC_FORCE_FUSED": "1"}, {"CRAC_K1_PAIR": "0"},
                                 {"CRAC_K1_PAIR": "8"}, {"CRAC_WRITER_TMA": "0"}],
                         ids=["fused", "one-chain", "pair8-key", "sm-store-writers"])
def test_alternative_kernel_selections_drain_the_same_bytes(env):
    """The fallbacks behind the defaults (the fused incremental drain the
    split one falls back to when its grid cannot be co-resident; the
    one-chain K1; 8-row chains with the key lane) drain the same bytes on
    every path of tools/sanitize_paths.py (each asserts path == full drain)."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    r = subprocess.run([sys.executable, str(root / "tools" / "sanitize_paths.py")],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "sanitize paths ok" in r.stdout
