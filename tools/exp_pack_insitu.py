"""Why is the pack kernel slower inside the drain than alone?  Reproduces the
drain pipeline (pack into a 4 x 64 MiB ring on one stream, 16 MiB D2H pieces
on another, event handshakes) with the kernel-level C-ABI and varies it."""
import ctypes as C
import statistics
import struct
import sys
import torch
sys.path.insert(0, ".")
from paper_2008_10596_b200 import engine

L = engine.lib()
MIB = 1 << 20
W, SLOTS, PIECE = 64 * MIB, 4, 16 * MIB
NWIN = 96
src = torch.empty(W * NWIN + 64, dtype=torch.uint8, device="cuda")
ring = torch.empty(SLOTS * (W + 64), dtype=torch.uint8, device="cuda")
host = torch.empty(W * NWIN, dtype=torch.uint8).pin_memory()
rec = struct.pack("<QQQQII", 0, src.data_ptr(), W * NWIN - 16, W * NWIN, 16, 0) + bytes(24)
d_rec = torch.frombuffer(bytearray(rec), dtype=torch.uint8).cuda()
d_tile = torch.zeros(W * NWIN // 65536 + 1, dtype=torch.int32, device="cuda")
sp, sc = torch.cuda.Stream(priority=-1), torch.cuda.Stream(priority=-1)


other = torch.empty(W, dtype=torch.uint8, device="cuda")
other_h = torch.empty(W, dtype=torch.uint8).pin_memory()


def run(copy=True, wait=True, piece=PIECE, foreign=None):
    ev_ready = [torch.cuda.Event() for _ in range(SLOTS)]
    ev_free = [torch.cuda.Event() for _ in range(SLOTS)]
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(NWIN)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(NWIN)]
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(sp)
    for w in range(NWIN):
        s = w % SLOTS
        buf = ring[s * (W + 64):]
        with torch.cuda.stream(sp):
            if wait and w >= SLOTS:
                sp.wait_event(ev_free[s])
            e0[w].record(sp)
            rc = L.crac_pack_records(C.c_void_p(d_rec.data_ptr()), 1,
                                     C.c_void_p(d_tile.data_ptr() + 4 * (w * W // 65536)),
                                     w * W, W, C.c_void_p(buf.data_ptr()), C.c_void_p(sp.cuda_stream))
            assert rc == 0
            e1[w].record(sp)
            ev_ready[s].record(sp)
        with torch.cuda.stream(sc):
            sc.wait_event(ev_ready[s])
            if foreign == "d2h":  # same traffic, but not from the ring
                for c in range(0, W, piece):
                    other_h[c:c + piece].copy_(other[c:c + piece], non_blocking=True)
            elif foreign == "h2d":
                for c in range(0, W, piece):
                    other[c:c + piece].copy_(other_h[c:c + piece], non_blocking=True)
            elif foreign == "d2d":  # a device-side copy of the same size
                other.copy_(ring[((s + 2) % SLOTS) * (W + 64):][:W], non_blocking=True)
            elif copy:
                for c in range(0, W, piece):
                    host[w * W + c:w * W + c + piece].copy_(buf[c:c + piece], non_blocking=True)
            ev_free[s].record(sc)
    t1.record(sc)
    torch.cuda.synchronize()
    d = [e0[w].elapsed_time(e1[w]) * 1000 for w in range(NWIN)]
    return statistics.median(d), min(d), t0.elapsed_time(t1)


for name, kw in [("pipeline (copy, wait)", {}), ("no copy", {"copy": False}),
                 ("copy, no wait", {"wait": False}), ("copy 64MiB pieces", {"piece": W}),
                 ("foreign d2h", {"foreign": "d2h"}), ("foreign h2d", {"foreign": "h2d"}),
                 ("foreign d2d", {"foreign": "d2d"}), ("no copy, no wait", {"copy": False, "wait": False})]:
    med, mn, tot = run(**kw)
    print(f"{name:24s} pack median {med:7.1f} us  min {mn:7.1f} us  total {tot:8.1f} ms "
          f"({W * NWIN / (tot * 1e-3) / 1e9:5.1f} GB/s)")
