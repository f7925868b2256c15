"""Where the C3 end-to-end step goes: checkpoint, session teardown, restart
(host wall clock around each public call).  python tools/teardown_probe.py [GiB]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2008_10596_b200 import engine  # noqa: E402

GIB, MIB = 1 << 30, 1 << 20
total = int(float(sys.argv[1]) * GIB) if len(sys.argv) > 1 else 16 * GIB
n = total // (256 * MIB)
s = engine.Session(seed=1, arena_bytes=n * 256 * MIB + 64 * MIB)
for _ in range(n):
    i, _ = s.alloc(engine.MANAGED, 256 * MIB)
    s.fill_synthetic(i, 1)
    for off in range(MIB, 256 * MIB, 2 * MIB):
        s.page_read(i, off, MIB, engine.HOST_SIDE)
img = engine.Image()
for step in range(3):
    t0 = time.perf_counter()
    d = s.checkpoint_into(img)
    t1 = time.perf_counter()
    s.close()
    t2 = time.perf_counter()
    addr, nb = img.address()
    s, r = engine.restart_from_address(addr, nb)
    t3 = time.perf_counter()
    print(f"step {step}: checkpoint {1e3*(t1-t0):.1f} ms (device {d['total_ms']:.1f}), "
          f"teardown {1e3*(t2-t1):.1f} ms, restart {1e3*(t3-t2):.1f} ms (device {r['total_ms']:.1f})",
          flush=True)
