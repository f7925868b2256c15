"""Direct copies between regions and the image, skipping the HBM ring: does a
D2H keep PCIe speed when the DEVICE side is misaligned but the host side is
4 KiB-aligned (a payload's middle copied straight from its region)?"""
import torch

MIB = 1 << 20
N = 1024 * MIB
dev = torch.empty(N + 8192, dtype=torch.uint8, device="cuda")
host = torch.empty(N + 8192, dtype=torch.uint8).pin_memory()
s = torch.cuda.Stream()


def bw(direction, host_off, dev_off, piece):
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0
    for rep in range(3):
        torch.cuda.synchronize()
        t0.record(s)
        with torch.cuda.stream(s):
            for c in range(0, N, piece):
                h = host[host_off + c:host_off + c + piece]
                d = dev[dev_off + c:dev_off + c + piece]
                if direction == "d2h":
                    h.copy_(d, non_blocking=True)
                else:
                    d.copy_(h, non_blocking=True)
        t1.record(s)
        torch.cuda.synchronize()
        best = max(best, N / (t0.elapsed_time(t1) * 1e-3) / 1e9)
    return best


for direction in ("d2h", "h2d"):
    for host_off, dev_off in ((0, 0), (0, 16), (0, 2048), (0, 4080), (16, 0), (4080, 0)):
        for piece in (16 * MIB, 32 * MIB, 64 * MIB):
            print(f"{direction} host+{host_off:<5} dev+{dev_off:<5} piece {piece // MIB:3d} MiB "
                  f"{bw(direction, host_off, dev_off, piece):6.1f} GB/s", flush=True)
