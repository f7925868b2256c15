"""K1 with / without the second dirty-key lane, by in-flight row depth.

One 32 GiB device buffer in 512 spans of 64 MiB (the C4/C5 region shape),
synthetic content; crac_chunk_key_range with d_key = NULL (CRC only) or a key
array, CUDA-event timed on one stream, median of 5 after a warm-up.  The key
rows are read once per process (CRAC_K1_KEY_ROWS), so each case is a child.
"""
import os
import subprocess
import sys

CHILD = r'''
import ctypes as C, statistics, struct, sys
sys.path.insert(0, ".")
import torch
from paper_2008_10596_b200 import engine
L = engine.lib()
GIB, MIB = 1 << 30, 1 << 20
with_key = sys.argv[2] == "key"
n_sp, sp = 512, 64 * MIB
buf = torch.empty(n_sp * sp, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for k in range(n_sp):
    assert L.crac_fill_synth(C.c_void_p(buf.data_ptr() + k * sp), sp, 3, k, 0, C.c_void_p(st)) == 0
spans = b"".join(struct.pack("<QQ", buf.data_ptr() + k * sp, sp) for k in range(n_sp))
d_spans = torch.frombuffer(bytearray(spans), dtype=torch.uint8).cuda()
first = torch.tensor([k * (sp // 65536) for k in range(n_sp + 1)], dtype=torch.int64).cuda()
nch = n_sp * sp // 65536
crc = torch.empty(nch, dtype=torch.int32, device="cuda")
key = torch.empty(nch, dtype=torch.int32, device="cuda")
kp = C.c_void_p(key.data_ptr()) if with_key else None
def run():
    rc = L.crac_chunk_key_range(C.c_void_p(d_spans.data_ptr()), C.c_void_p(first.data_ptr()), n_sp,
                                65536, 0, nch, C.c_void_p(crc.data_ptr()), kp, 0, C.c_void_p(st))
    assert rc == 0, rc
ts = []
for i in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = statistics.median(ts[1:])
# parity on chunks around span boundaries (pairs straddle spans) and inside
sys.path.insert(0, "tests")
import zlib, dirtykey
per = sp // 65536
crc_h = crc.cpu().numpy().view("uint32")
key_h = key.cpu().numpy().view("uint32")
bad = 0
for c in [0, 1, 2, 3, per - 2, per - 1, per, per + 1, 5 * per - 1, 5 * per, nch - 3, nch - 2, nch - 1]:
    chunk = bytes(buf[c * 65536:(c + 1) * 65536].cpu().numpy())
    bad += int(crc_h[c]) != zlib.crc32(chunk)
    if with_key:
        bad += int(key_h[c]) != dirtykey.chunk_key(chunk)
assert bad == 0, f"parity: {bad} mismatches"
print(f"{sys.argv[1]:>10s} {sys.argv[2]:5s} 32 GiB {ms:7.3f} ms {32 * GIB / ms / 1e6:7.0f} GB/s  parity ok", flush=True)
'''

cases = [("16", "nokey", {}), ("8", "nokey", {"CRAC_K1_ROWS": "8"}),
         ("8", "key", {"CRAC_K1_KEY_ROWS": "8"}), ("12", "key", {"CRAC_K1_KEY_ROWS": "12"}),
         ("pair4", "key", {"CRAC_K1_PAIR": "4"}), ("pair4", "nokey", {"CRAC_K1_PAIR": "4"}),
         ("pair8", "nokey", {"CRAC_K1_PAIR": "8"}), ("pair8", "key", {"CRAC_K1_PAIR": "8"})]
only = sys.argv[1] if len(sys.argv) > 1 else None  # e.g. "8:key" (for ncu)
if only:
    rows, mode = only.split(":")
    env1 = ({"CRAC_K1_PAIR": rows[4:]} if rows.startswith("pair") else
            {"CRAC_K1_KEY_ROWS": rows} if mode == "key" else {"CRAC_K1_ROWS": rows})
    cases = [(rows, mode, env1)]
for rows, mode, extra in cases:
    env = dict(os.environ, **extra)
    r = subprocess.run([sys.executable, "-c", CHILD, f"rows={rows}", mode], env=env,
                       capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr.strip()[-800:], flush=True)
