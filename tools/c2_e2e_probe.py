"""Where the C2 end-to-end step spends its host time: checkpoint, session
close, restart (parse + refill), each timed on the host around the public
API call (bench.py's e2e step, split up)."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import torch  # noqa: F401  (CUDA context as in bench.py)
from paper_2008_10596_b200 import engine
import workloads

sess = engine.Session(seed=1, arena_bytes=2 << 30)
workloads.build_churn(sess, 40000, 1)
image = engine.Image()
rows = []
for it in range(8):
    t0 = time.perf_counter()
    dr = sess.checkpoint_into(image)
    t1 = time.perf_counter()
    addr, n = image.address()
    sess.close()
    t2 = time.perf_counter()
    sess, rf = engine.restart_from_address(addr, n)
    t3 = time.perf_counter()
    rows.append((1e3 * (t1 - t0), dr["total_ms"], 1e3 * (t2 - t1), 1e3 * (t3 - t2), rf["total_ms"]))
for r in rows[3:]:
    print("checkpoint host %.3f dev %.3f | close %.3f | restart host %.3f dev %.3f" % r)
