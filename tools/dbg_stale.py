import random, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2008_10596_b200 import engine as eng
from oracle import ref
import workloads
MIB = 1 << 20
L = eng.lib()
def peek(tag):
    e = L.crac_peek_cuda_error()
    print(f"{tag}: {e}", flush=True)
seed = 1
rnd = random.Random(seed)
s = eng.Session(seed=seed, arena_bytes=1 << 30)
ids = []
for k in range(40):
    size = rnd.choice([1, 17, 4096, 65536 * 6 + rnd.randrange(1000), 3 * MIB + rnd.randrange(9999), rnd.randrange(1, 40 * MIB)])
    i, _ = s.alloc(workloads.DEVICE, size); s.fill_synthetic(i, seed * 100 + k); ids.append(i)
    if k % 7 == 3:
        victim = ids.pop(rnd.randrange(len(ids))); s.free(victim)
peek("built")
img, _ = s.checkpoint(); peek("checkpoint")
rs, _ = eng.restart(img); peek("restart")
import test_gpu_parity as T
a = T._state(rs); peek("state rs")
b = T._state(s); peek("state s")
print("equal", a == b)
image = eng.Image(); s.checkpoint_into(image); peek("checkpoint_into")
s.mutate(seed=seed, epoch=1, threshold=(1 << 64) // 5); peek("mutate")
st = s.checkpoint_into(image, incremental=True); peek("incremental")
sync = s.checkpoint()[0]; peek("sync")
s.reserve_shadow(rnd.choice([0, 64, 128, 512]) * MIB); peek("reserve")
s.checkpoint_begin(image); peek("begin"); s.checkpoint_finish(); peek("finish")
s.reserve_shadow(0); peek("unreserve")
s.checkpoint_precopy_begin(image); peek("pc begin")
s.mutate(seed=seed, epoch=2, threshold=(1 << 64) // 50); peek("mutate2")
s.checkpoint_precopy_finish(); peek("pc finish")
final = s.checkpoint()[0]; peek("final")
rs2, _ = eng.restart(final); peek("restart2")
rs2.checkpoint(); peek("rs2 ckpt")
del rs2, rs, s, image; import gc; gc.collect(); peek("gc")
