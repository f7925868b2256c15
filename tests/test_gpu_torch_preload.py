"""GPU tier: PyTorch under libcrac_preload.so (SURVEY §8f.2 on a real
framework).  torch's caching allocator takes its device memory from the
logged session (cudaMalloc interposed), so a checkpoint of the process
contains every tensor byte at the tensor's own device address, and a new
process restarted from the image finds those bytes at the same addresses."""
import hashlib
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

from oracle import image_oracle as io
from oracle import ref

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
PRELOAD = ROOT / "paper_2008_10596_b200" / "libcrac_preload.so"


def test_torch_process_checkpoint_holds_every_tensor(tmp_path):
    if not PRELOAD.exists():
        from paper_2008_10596_b200 import build
        build.build()
    img = tmp_path / "torch.img"
    env = dict(os.environ, LD_PRELOAD=str(PRELOAD), CRAC_ARENA_BYTES=str(8 << 30))
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "torch_under_preload.py"), str(img)],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["preload"] and out["rc"] == 0, out
    data = img.read_bytes()
    ref.ref_decode_check(data)  # the reference reads the image of a torch process
    snap = io.decode_image(data)
    # logged allocations: (id -> address, size) of the live ones
    live = {}
    for (seq, op, kind, size, ident, addr) in snap.log:
        if op == 1:
            live[ident] = (addr, size)
        elif op == 2:
            live.pop(ident, None)
    payload = dict(snap.payloads)
    for t in out["tensors"]:
        owner = [i for i, (addr, size) in live.items() if addr <= t["ptr"] < addr + size]
        assert owner, t
        addr, _ = live[owner[0]]
        off = t["ptr"] - addr
        got = payload[owner[0]][off:off + t["nbytes"]]
        assert hashlib.sha256(got).hexdigest() == t["sha256"]
    # a new torch process restarted from the image: same addresses, same bytes
    env2 = dict(os.environ, LD_PRELOAD=str(PRELOAD), CRAC_RESTART_FROM=str(img))
    r2 = subprocess.run([sys.executable, str(ROOT / "tools" / "torch_under_preload.py"), "--resume"],
                        env=env2, capture_output=True, text=True, timeout=600)
    assert r2.returncode == 0, r2.stdout[-2000:] + r2.stderr[-4000:]
    back = json.loads(r2.stdout.strip().splitlines()[-1])
    assert back["resumed"] and all(back["tensors_intact"]) and len(back["tensors_intact"]) == 3
