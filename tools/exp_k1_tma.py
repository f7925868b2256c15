"""K1 register loads vs K1 staged through shared memory by cp.async.bulk
(CRAC_K1_TMA=A|B|C, see kernels.cu k1_chunk_crc_tma): parity against zlib,
then the hash-only time of a 32 GiB Device state.  One mode per process (the
variable is read once)."""
import os
import subprocess
import sys

CHILD = r'''
import sys, zlib, statistics
sys.path.insert(0, ".")
import torch
from paper_2008_10596_b200 import engine
GIB, MIB = 1 << 30, 1 << 20
# parity: odd sizes, tails, several chunks per warp
for n in (1, 511, 512, 4097, 65536, 65536 * 7 + 1234, 3 << 20):
    g = torch.Generator().manual_seed(n)
    h = bytes(torch.randint(0, 256, (n,), dtype=torch.uint8, generator=g).numpy())
    got = engine.hash_chunks(h, 65536)
    want = [zlib.crc32(h[i:i + 65536]) for i in range(0, n, 65536)]
    assert list(got) == want, n
s = engine.Session(seed=1, arena_bytes=33 * GIB)
for k in range(512):
    i, _ = s.alloc(1, 64 * MIB)
    s.fill_synthetic(i, 3)
ts = [s.hash_only()["hash_ms"] for _ in range(6)][1:]
ms = statistics.median(ts)
print(f"{sys.argv[1]:8s} parity ok  hash-only 32 GiB {ms:7.2f} ms  {32 * GIB / ms / 1e6:7.0f} GB/s")
'''

for mode in ("regs", "A", "B", "C"):
    env = dict(os.environ)
    if mode != "regs":
        env["CRAC_K1_TMA"] = mode
    r = subprocess.run([sys.executable, "-c", CHILD, mode], env=env, capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr.strip()[-600:], flush=True)
