import random, sys, os
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2008_10596_b200 import engine as eng
import workloads
MIB = 1 << 20
import test_gpu_parity as T
T.test_random_mixed_paths_agree(eng, 1)
print("seed 1 done", flush=True)
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 3
rnd = random.Random(seed)
s = eng.Session(seed=seed, arena_bytes=1 << 30)
print("s fixed", s.fixed_va, flush=True)
ids = []
sizes = []
for k in range(40):
    size = rnd.choice([1, 17, 4096, 65536 * 6 + rnd.randrange(1000), 3 * MIB + rnd.randrange(9999), rnd.randrange(1, 40 * MIB)])
    i, addr = s.alloc(workloads.DEVICE, size); s.fill_synthetic(i, seed * 100 + k); ids.append(i); sizes.append((i, size, addr))
    if k % 7 == 3:
        victim = ids.pop(rnd.randrange(len(ids))); s.free(victim)
img, _ = s.checkpoint()
print("image", len(img), flush=True)
try:
    rs, _ = eng.restart(img)
    print("rs fixed", rs.fixed_va, "ok")
except Exception as e:
    print("restart failed:", e)
    for (i, size, addr) in sizes:
        print(i, size, hex(addr), hex(addr - 0xD0000000000))
