"""A PyTorch process under LD_PRELOAD=libcrac_preload.so (SURVEY §8f.2 demo):
torch's caching allocator gets its device memory from the logged session,
its kernel launches pass the dispatch gate, and crac_preload_checkpoint
drains every byte torch holds into an image.  Prints JSON with the tensor
addresses and a digest of their bytes so a checker can find them in the image.

    LD_PRELOAD=.../libcrac_preload.so python tools/torch_under_preload.py <image>
    LD_PRELOAD=... CRAC_RESTART_FROM=<image> python tools/torch_under_preload.py --resume

--resume: a new process restarted from the image finds the tensors' bytes at
their old device addresses (torch.as_tensor over __cuda_array_interface__).
"""
import ctypes
import hashlib
import json
import sys

import torch

lib = ctypes.CDLL(None)


class Raw:  # a device range torch can wrap without copying
    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": (nbytes,), "typestr": "|u1",
                                         "version": 3}


if sys.argv[1] == "--resume":
    get = lib.crac_preload_app_state
    get.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_uint64)]
    p, n = ctypes.c_void_p(), ctypes.c_uint64()
    assert get(ctypes.byref(p), ctypes.byref(n)) == 0 and n.value > 0, "not restarted"
    saved = json.loads(ctypes.string_at(p, n.value).decode())
    ok = []
    for t in saved["tensors"]:
        view = torch.as_tensor(Raw(t["ptr"], t["nbytes"]), device="cuda")
        ok.append(hashlib.sha256(view.cpu().numpy().tobytes()).hexdigest() == t["sha256"])
    print(json.dumps({"resumed": True, "tensors_intact": ok}))
    sys.exit(0 if all(ok) else 1)

path = sys.argv[1]
torch.manual_seed(0)
a = torch.randn(3, 1 << 20, device="cuda")            # 12 MiB
b = torch.arange(1 << 22, device="cuda", dtype=torch.int32) * 7
c = (a @ a.T).contiguous()                              # cuBLAS output
torch.cuda.synchronize()
fn = getattr(lib, "crac_preload_checkpoint", None)
if fn is None:
    print(json.dumps({"preload": False}))
    sys.exit(0)
out = {"preload": True, "tensors": []}
for t in (a, b, c):
    data = t.cpu().numpy().tobytes()
    out["tensors"].append({"ptr": t.data_ptr(), "nbytes": len(data),
                           "sha256": hashlib.sha256(data).hexdigest()})
state = json.dumps(out).encode()
lib.crac_preload_set_app_state.argtypes = [ctypes.c_char_p, ctypes.c_uint64]
assert lib.crac_preload_set_app_state(state, len(state)) == 0
fn.argtypes = [ctypes.c_char_p]
out["rc"] = fn(path.encode())
print(json.dumps(out))
