"""Stall-reduced drain on a Device-only state: prints the app stall of
checkpoint_begin (hash+copy into the HBM shadow) against a synchronous drain.
Its first K1 launch is the fused hash+copy kernel (for ncu -k regex:k1 -c 1).

    python tools/stall_probe.py [GiB] [region MiB] [size skew bytes]
"""
import sys
import statistics

sys.path.insert(0, ".")
from paper_2008_10596_b200 import engine  # noqa: E402

GIB, MIB = 1 << 30, 1 << 20
gib = float(sys.argv[1]) if len(sys.argv) > 1 else 8
region = int(sys.argv[2]) if len(sys.argv) > 2 else 64
skew = int(sys.argv[3]) if len(sys.argv) > 3 else 16  # 16: every payload 16-byte aligned
n = int(gib * GIB) // (region * MIB)
s = engine.Session(seed=1, arena_bytes=n * region * MIB + GIB)
for k in range(n):
    i, _ = s.alloc(1, region * MIB - skew * (k % 3))
    s.fill_synthetic(i, 7)
live = sum(r.size for r in s.live_records())
s.reserve_shadow(live + 16 * n + 20 + 64 * MIB)
img = engine.Image()
rows = []
for _ in range(4):
    s.checkpoint_begin(img)
    rows.append(s.checkpoint_finish())
want = s.checkpoint(img)[1]
stall = statistics.median(r["stall_ms"] for r in rows[1:])
k1 = statistics.median(r["hash_ms"] for r in rows[1:])
print(f"{live / GIB:.1f} GiB: stall {stall:.2f} ms ({2 * live / stall / 1e6:.0f} GB/s read+write), "
      f"async total {statistics.median(r['total_ms'] for r in rows[1:]):.1f} ms, "
      f"sync drain {want['total_ms']:.1f} ms, shadow {rows[-1]['shadow_bytes'] / GIB:.2f} GiB; "
      f"K1 hash+copy {k1:.2f} ms ({2 * live / k1 / 1e6:.0f} GB/s)")
