"""Isolated timing of the pack / scatter kernels (64 MiB windows) vs a torch copy."""
import ctypes as C
import struct
import sys
import torch
sys.path.insert(0, ".")
from paper_2008_10596_b200 import engine

L = engine.lib()
W = 64 << 20
src = torch.randint(0, 255, (1 << 30,), dtype=torch.uint8, device="cuda")
out = torch.empty(W + 64, dtype=torch.uint8, device="cuda")
# one record covering the whole source, frame 16 bytes at 0
rec = struct.pack("<QQQQII", 0, src.data_ptr(), src.numel(), src.numel(), 16, 0) + bytes(24)
d_rec = torch.frombuffer(bytearray(rec), dtype=torch.uint8).cuda()
tiles = (src.numel() + 16 + 65535) // 65536
d_tile = torch.zeros(tiles, dtype=torch.int32, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in [
    ("pack", lambda off: L.crac_pack_records(C.c_void_p(d_rec.data_ptr()), 1,
                                             C.c_void_p(d_tile.data_ptr() + 4 * (off // 65536)),
                                             off, W, C.c_void_p(out.data_ptr()), None)),
    ("scatter", lambda off: L.crac_scatter_records(C.c_void_p(d_rec.data_ptr()), 1,
                                                   C.c_void_p(d_tile.data_ptr() + 4 * (off // 65536)),
                                                   C.c_void_p(out.data_ptr()), off, W, None)),
    ("torch copy", lambda off: out[:W].copy_(src[off:off + W]) and 0),
]:
    for _ in range(3):
        fn(0)
    torch.cuda.synchronize()
    e0.record()
    n = 0
    for off in range(65536, (1 << 30) - W, W):
        assert fn(off) in (0, None)
        n += 1
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"{name:12s} {ms * 1000:8.1f} us per 64 MiB window  {2 * W / (ms * 1e-3) / 1e9:8.1f} GB/s (r+w)")
