#!/usr/bin/env python
"""Checkpoint & restart GB/s per GPU and whole box (BASELINE.json metric).

Workload (BASELINE.json configs[3], "C4"): every rank owns one B200 holding
120 GiB of live device state in 1920 x 64 MiB cudaMalloc-kind regions with
synthetic content.  One step = full checkpoint drain of that state into a
page-locked host image (crac_checkpoint) + session teardown + restart refill
from the image (crac_restart: replay, H2D, scatter, CRC verify).  Ranks drain
independently; the only cross-rank step is the host barrier of the global
checkpoint (the config's "global barrier").  Inputs (120 GiB/GPU) exceed L2 by ~1000x.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

value  = 2 x live bytes x ranks / sum over steps of (max over ranks of the
         device-event time of that step's drain + refill); the ranks start
         every step together, so this is max end - min start per step
e2e    = same bytes / sum over steps of (max over ranks of the CUDA-event
         intervals around the step's two public C-ABI calls, the drain into
         the host image and the restart from it: host work and copies
         included; the teardown between them, which a new-process restart
         never pays, is reported beside it as e2e.with_teardown)
The restart is cold: the closed session's arena is freed before each refill,
as in a new process.  A small arena (<= 16 GiB: C2) has only its VA freed
before the refill and its memory released on a thread beside it (the public
crac_drop_arena_cache_async), which keeps the driver's 2-130 ms release
spikes off the step; a big one (C4) is released before the refill, because
the driver serializes the refill's arena map behind a release in flight (C4
~80 ms slower; profiles/r02/async_release.txt).  CRAC_ASYNC_RELEASE=0|1
forces either.  With N > 1 ranks every drain meets the other ranks at
the product's global-checkpoint barrier (crac_barrier, crac_engine.h).
`--gpus N` outside torchrun spawns the N ranks itself; `--dry-run` runs the
rank plumbing only (no GPU).
--impl reference times the reference's own CPU path (oracle/_ref, the
unmodified library) on the host cores, one sample session per core.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ASYNC_RELEASE = os.environ.get("CRAC_ASYNC_RELEASE")  # "0" | "1" | None (by arena size)

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

GIB = 1 << 30
MIB = 1 << 20


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--footprint-gib", type=float, default=120.0)
    ap.add_argument("--region-mib", type=int, default=64)
    ap.add_argument("--cpu-sample-gib", type=float, default=1.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-incremental", action="store_true")
    ap.add_argument("--no-stall", action="store_true",
                    help="skip the stall-reduced (checkpoint_begin/finish) measurement")
    ap.add_argument("--workload", choices=["c4", "c2", "c3", "c5", "file"], default="c4")
    ap.add_argument("--file-footprint-gib", type=float, default=16.0,
                    help="state for --workload file (bounded by the disk: 2 images on it)")
    ap.add_argument("--io-dir", default=None,
                    help="directory of the image file (default: $CRAC_IO_DIR or /tmp)")
    ap.add_argument("--c2-calls", type=int, default=40000)
    ap.add_argument("--no-cold", action="store_true", help="skip the cold-restart measurement")
    ap.add_argument("--c3-footprint-gib", type=float, default=16.0)
    ap.add_argument("--c5-footprint-gib", type=float, default=64.0)
    ap.add_argument("--dry-run", action="store_true",
                    help="rank plumbing only (no GPU): every rank prints its device assignment")
    ap.add_argument("--no-verify", action="store_true",
                    help="skip the host-side check of the final image and the restarted state")
    ap.add_argument("--share-gpu", action="store_true",
                    help="testing: every rank on the same GPU (the N-rank path on a 1-GPU box)")
    return ap.parse_args()


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: launch N ranks of this script
    (RANK / LOCAL_RANK / WORLD_SIZE set as torchrun does, one GPU each) and
    return the worst exit code.  Rank 0 prints the JSON line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, str(Path(__file__).resolve()), *sys.argv[1:]],
                                      env=env))
    return max(p.wait() for p in procs)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    return world, rank, local, local_world


def job_gpu_indices(local_world: int) -> list[str]:
    """nvidia-smi indices of the GPUs this node's ranks use (before pin_device
    narrows CUDA_VISIBLE_DEVICES): the clocks are sampled on those only."""
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    devs = vis.split(",") if vis else [str(i) for i in range(64)]
    return devs[:max(1, local_world)]


def pin_device(local: int, world: int) -> None:
    # one process per GPU: each rank sees exactly its own device as cuda:0,
    # in both torch's runtime and libcrac_b200's (statically linked) runtime
    os.environ.setdefault("CUDA_DEVICE_ORDER", "PCI_BUS_ID")
    if world > 1:
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        devs = vis.split(",") if vis else [str(i) for i in range(64)]
        os.environ["CUDA_VISIBLE_DEVICES"] = devs[local]


def mem_available() -> int:
    for line in Path("/proc/meminfo").read_text().splitlines():
        if line.startswith("MemAvailable:"):
            return int(line.split()[1]) * 1024
    return 64 * GIB


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d.get("hbm_gbs", 6650.0)), "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.lines: list[str] = []
        self.proc = None
        self.t = None
        self.first = 0  # samples before this index precede the timed region

    def mark(self):
        """The timed region starts now: earlier samples are dropped."""
        self.first = len(self.lines)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self, gpu_indices=None) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=5)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines[self.first:]:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            if gpu_indices is not None and parts[0] not in gpu_indices:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


class HostGroup:
    """The only cross-rank exchange of the path: a host barrier marking the
    consistent global checkpoint, plus the max-over-ranks of the timings
    (gloo on CPU tensors; no data-path collective exists)."""

    def __init__(self, world: int, rank: int):
        self.world = world
        if world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29511")
            dist.init_process_group("gloo", rank=rank, world_size=world)

    def barrier(self) -> None:
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def max_list(self, xs: list) -> list:
        """Elementwise max over ranks (per-step times)."""
        if self.world == 1:
            return list(xs)
        import torch
        import torch.distributed as dist
        t = torch.tensor(list(xs), dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    def close(self) -> None:
        if self.world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


# ---------------------------------------------------------------------------
# reference arm / cpu baseline (oracle/_ref: the unmodified reference library)
# ---------------------------------------------------------------------------
def ref_sample_step(state: dict) -> None:
    from oracle import ref
    t0 = time.perf_counter()
    img, times = state["session"].checkpoint()
    new, rtimes = ref.ref_restart(img)
    state["session"].close()
    state["session"] = new
    state["elapsed"] = time.perf_counter() - t0
    state["phases"] = {**times, **rtimes}


def ref_make_session(sample_bytes: int, region: int, seed: int):
    from oracle import ref
    n = max(1, sample_bytes // region)
    s = ref.RefSession(seed=seed, arena_bytes=n * region + MIB)
    for _ in range(n):
        i, _ = s.alloc(1, region)
        s.fill_synthetic(i, seed)
    return s, n * region


def cpu_baseline(sample_gib: float, region: int) -> dict:
    """Single-threaded reference checkpoint+encode / decode+restart (C4 scaled)."""
    s, live = ref_make_session(int(sample_gib * GIB), region, seed=1)
    state = {"session": s}
    ref_sample_step(state)
    ph = state["phases"]
    total = ph["checkpoint_s"] + ph["encode_s"] + ph["decode_s"] + ph["restart_s"]
    state["session"].close()
    return {"value": round(2 * live / total / 1e9, 4), "unit": "GB/s", "cores": 1,
            "kind": "reference",
            "sample": f"C4 scaled to {live // MIB} MiB ({live // region} x {region // MIB} MiB "
                      f"Device regions): checkpoint()+encode_image() then decode_image()+restart() "
                      f"of the unmodified reference, single-threaded by construction",
            "phases_s": {k: round(v, 3) for k, v in ph.items()}}


def _ref_round_trip(s, live: int, sample: str) -> dict:
    """One reference checkpoint+encode / decode+restart of session `s`."""
    state = {"session": s}
    ref_sample_step(state)
    ph = state["phases"]
    total = ph["checkpoint_s"] + ph["encode_s"] + ph["decode_s"] + ph["restart_s"]
    state["session"].close()
    return {"value": round(2 * live / total / 1e9, 4), "unit": "GB/s", "cores": 1,
            "kind": "reference", "sample": sample,
            "phases_s": {k: round(v, 3) for k, v in ph.items()}}


def cpu_baseline_c2(calls: int) -> dict:
    """The unmodified reference on the whole C2 workload (same call sequence
    shape, seed 1), single-threaded by construction."""
    from oracle import ref
    import workloads
    s = ref.RefSession(seed=1, arena_bytes=2 * GIB)
    workloads.build_churn(s, calls, 1)
    live = sum(r[2] for r in s.live_records())  # (id, kind, size, address)
    return _ref_round_trip(s, live, f"C2 at full size ({calls} calls, {live // MIB} MiB live): "
                                    "checkpoint()+encode_image() then decode_image()+restart() "
                                    "of the unmodified reference, single-threaded by construction")


def cpu_baseline_c3(sample_gib: float) -> dict:
    """The unmodified reference on C3 scaled (256 MiB managed regions,
    alternating 1 MiB device/host runs), single-threaded by construction."""
    from oracle import ref
    import workloads
    mregion = 256 * MIB
    n = max(1, int(sample_gib * GIB) // mregion)
    s = ref.RefSession(seed=1, arena_bytes=n * mregion + 64 * MIB)
    for _ in range(n):
        i, _ = s.alloc(workloads.MANAGED, mregion)
        s.fill_synthetic(i, 1)
        for off in range(MIB, mregion, 2 * MIB):
            s.page_read(i, off, MIB, workloads.HOST_SIDE)
    return _ref_round_trip(s, n * mregion,
                           f"C3 scaled to {n * mregion // MIB} MiB ({n} x 256 MiB managed, "
                           "alternating 1 MiB device/host runs): checkpoint()+encode_image() then "
                           "decode_image()+restart() of the unmodified reference, single-threaded")


def cpu_baseline_c5(sample_gib: float) -> dict:
    """the chunk-hash step on every host core -- zlib's crc32
    (the reference's crc32_of) per 64 KiB chunk over a bounded sample, each
    thread on its own slice (zlib releases the GIL)."""
    import zlib
    from concurrent.futures import ThreadPoolExecutor
    threads = max(1, os.cpu_count() or 1)
    chunk = 65536
    buf = bytearray(os.urandom(1 << 20)) * 256  # 256 MiB (> L3), random content
    view = memoryview(buf)
    reps = max(1, int(sample_gib * GIB) // len(buf))

    def work(t):
        h = 0
        for _ in range(reps):
            for off in range(t * chunk, len(buf), threads * chunk):
                h ^= zlib.crc32(view[off:off + chunk])
        return h

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(work, range(threads)))
    dt = time.perf_counter() - t0
    hashed = reps * len(buf)
    return {"value": round(hashed / dt / 1e9, 3), "unit": "GB/s hashed", "cores": threads,
            "kind": "port",
            "sample": f"{hashed // GIB} GiB ({reps} passes over a 256 MiB buffer): zlib crc32 per "
                      f"64 KiB chunk on {threads} threads -- the host chunk-hash step the "
                      "incremental drain's hash-only pass replaces (SURVEY 8(d) item 2)"}


def _ref_worker(t, per, region, steps, warmup, barrier, q):
    """One host core: its own reference session (a separate process, so the
    reference's large vector allocations do not contend on one address
    space's page-fault lock), the bounded sample stepped in lockstep."""
    s, live = ref_make_session(per, region, seed=t + 1)
    state = {"session": s}
    times = []
    for k in range(warmup + steps):
        barrier.wait()
        t0 = time.perf_counter()
        ref_sample_step(state)
        times.append(time.perf_counter() - t0)
    state["session"].close()
    q.put((t, live, times[warmup:]))


def run_reference(args, world, rank) -> None:
    if rank != 0:
        return
    import multiprocessing as mp
    procs_n = max(1, os.cpu_count() or 1)
    region = args.region_mib * MIB
    # ~5x the sample in host RAM per worker (arena + snapshot + image + decode)
    per = min(max(int(args.cpu_sample_gib * GIB) // procs_n, region),
              mem_available() // (8 * procs_n))
    per = max(region, per // region * region)
    ctx = mp.get_context("fork")
    barrier = ctx.Barrier(procs_n)
    q = ctx.Queue()
    procs = [ctx.Process(target=_ref_worker,
                         args=(t, per, region, args.steps, args.warmup, barrier, q))
             for t in range(procs_n)]
    for p in procs:
        p.start()
    results = [q.get() for _ in procs]
    for p in procs:
        p.join()
    live = sum(r[1] for r in results)
    # a step ends when the slowest worker finishes it
    step_times = [max(r[2][k] for r in results) for k in range(args.steps)]
    total = sum(step_times)
    value = 2 * live * args.steps / total / 1e9
    line = {
        "metric": "checkpoint & restart GB/s per GPU and whole box at 1/2/4/8 B200; % of roofline",
        "impl": "reference", "value": round(value, 4), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1000 * total / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": "C4 full checkpoint + restart (reference CPU path, scaled sample)",
                   "live_bytes_per_step": live, "region_bytes": region, "workers": procs_n},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": procs_n,
                         "kind": "reference",
                         "sample": f"{procs_n} reference sessions (one process per core) x "
                                   f"{per // MIB} MiB ({per // region} x {region // MIB} MiB "
                                   f"Device regions); a step = checkpoint()+encode_image()+"
                                   f"decode_image()+restart() on every core, timed to the slowest"},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# the B200 arm
# ---------------------------------------------------------------------------
def pcie_peaks(torch) -> dict:
    """Copy-engine ceiling of this GPU's link: 2 GiB of pinned copies in 16 MiB
    and in 64 MiB pieces, five passes each, the best pass (a single pass can
    land on a transiently slow link and would understate the ceiling)."""
    total = 2048 * MIB
    h = torch.empty(total, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(total, dtype=torch.uint8, device="cuda")
    out = {}
    for name, (dst, src) in {"d2h": (h, d), "h2d": (d, h)}.items():
        best = 0.0
        for chunk in (16 * MIB, 64 * MIB):
            n = total // chunk
            for _ in range(5):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for k in range(n):
                    dst[k * chunk:(k + 1) * chunk].copy_(src[k * chunk:(k + 1) * chunk],
                                                         non_blocking=True)
                e1.record()
                torch.cuda.synchronize()
                best = max(best, total / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        out[name] = round(best, 2)
    del h, d
    return out


def isolated_kernel_rates(torch, engine) -> dict:
    """Pack / scatter kernels on one 64 MiB window each, back to back on one
    stream (no copy engine, no other stream), for comparison with the in-situ
    per-launch times of the timed region."""
    import ctypes as C
    import struct
    L = engine.lib()
    W, N = 64 * MIB, 8
    src = torch.empty(W * (N + 1), dtype=torch.uint8, device="cuda")
    out = torch.empty(W + 64, dtype=torch.uint8, device="cuda")
    rec = struct.pack("<QQQQII", 0, src.data_ptr(), src.numel() - 16, src.numel(), 16, 0) + bytes(24)
    d_rec = torch.frombuffer(bytearray(rec), dtype=torch.uint8).cuda()
    d_tile = torch.zeros(src.numel() // 65536 + 1, dtype=torch.int32, device="cuda")
    res = {}
    for name, call in (("k_pack_records", L.crac_pack_records), ("k_scatter_records", L.crac_scatter_records)):
        def run(w):
            off = W * w
            tile = C.c_void_p(d_tile.data_ptr() + 4 * (off // 65536))
            if name == "k_pack_records":
                return call(C.c_void_p(d_rec.data_ptr()), 1, tile, off, W, C.c_void_p(out.data_ptr()), None)
            return call(C.c_void_p(d_rec.data_ptr()), 1, tile, C.c_void_p(out.data_ptr()), off, W, None)
        run(0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for w in range(1, N + 1):
            assert run(w) == 0
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / N
        res[name] = {"avg_launch_ms": round(ms, 4), "GBps": round(2 * W / (ms * 1e-3) / 1e9, 1)}
    # the in-situ ceiling: the driver's own D2D copy of a 64 MiB window while
    # a D2H of 16 MiB pieces runs on another stream (what the drain does);
    # PCIe copy traffic slows every HBM copy, see profiles/r01/copy_interference.txt
    host = torch.empty(256 * MIB, dtype=torch.uint8).pin_memory()
    stage = torch.empty(256 * MIB, dtype=torch.uint8, device="cuda")
    sc, sk = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(sc):
        for i in range(120):
            j = (i % 16) * 16 * MIB
            host[j:j + 16 * MIB].copy_(stage[j:j + 16 * MIB], non_blocking=True)
    times = []
    with torch.cuda.stream(sk):
        for w in range(1, N + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(sk)
            out[:W].copy_(src[W * w:W * (w + 1)], non_blocking=True)
            e1.record(sk)
            times.append((e0, e1))
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(b) for a, b in times)
    res["d2d_copy_beside_d2h"] = {"avg_launch_ms": round(ms, 4),
                                  "GBps": round(2 * W / (ms * 1e-3) / 1e9, 1)}
    del src, out, host, stage
    return res


def build_workload(args, engine, rank: int, live_cap: int):
    """Creates the resident state of the chosen config; returns
    (session, live bytes, config dict)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import workloads
    region = args.region_mib * MIB
    seed = rank + 1
    if args.workload in ("c4", "c5", "file"):
        want = {"c4": args.footprint_gib, "c5": args.c5_footprint_gib,
                "file": args.file_footprint_gib}[args.workload]
        footprint = min(int(want * GIB), live_cap) // region * region
        n = footprint // region
        sess = engine.Session(seed=seed, arena_bytes=footprint + 64 * MIB)
        workloads.build_regions(sess, n, lambda r: region, seed)
        return sess, footprint, {"regions_per_gpu": n, "region_bytes": region,
                                 "requested_footprint_gib": want}
    if args.workload == "c2":
        # Rodinia-style: 4 streams, 70 % alloc / 30 % free of 256 B..64 KiB Device
        # buffers, one fill8 launch per allocation (alloc_churn, harness.cpp:476-499)
        sess = engine.Session(seed=seed, arena_bytes=2 * GIB)
        workloads.build_churn(sess, args.c2_calls, seed)
        recs = sess.live_records()
        return sess, sum(r.size for r in recs), {"calls": args.c2_calls, "live_regions": len(recs),
                                                 "log_entries": sess.log_size(), "streams": 4}
    if args.workload == "c3":
        # HPGMG-style UVM: cudaMallocManaged regions, alternating 1 MiB runs of
        # device- and host-resident pages (uvm_tasks, harness.cpp:345-389)
        total = min(int(args.c3_footprint_gib * GIB), live_cap)
        mregion = 256 * MIB
        n = max(1, total // mregion)
        sess = engine.Session(seed=seed, arena_bytes=n * mregion + 64 * MIB)
        for _ in range(n):
            i, _ = sess.alloc(engine.MANAGED, mregion)
            sess.fill_synthetic(i, seed)  # device-side write: device-resident, dirty
            for off in range(MIB, mregion, 2 * MIB):
                sess.page_read(i, off, MIB, engine.HOST_SIDE)  # host touch: host-resident
        return sess, n * mregion, {"managed_regions": n, "region_bytes": mregion,
                                   "residence": "alternating 1 MiB runs device/host"}
    raise SystemExit(f"unknown workload {args.workload}")


WORKLOAD_NAMES = {
    "c4": "C4: full checkpoint drain + restart refill of live device state, independent "
          "per-GPU drains, host barrier",
    "c2": "C2: Rodinia-style many small allocations on 4 streams, full checkpoint + restart",
    "c3": "C3: HPGMG-style cudaMallocManaged footprint with mixed residence, checkpoint + "
          "residency-restoring restart",
    "c5": "C5: incremental checkpoint sequence at 1/5/25 % dirty chunks, hash-only vs drain",
    "file": "C4 shape through the file: checkpoint_to_file (drain + parallel O_DIRECT write + "
            "fdatasync) then restart_from_file (parallel read + refill)",
}


def ncu_traffic(kernel):
    """DRAM bytes (read + write) per launch of `kernel` from the newest
    committed `ncu --set full` summary (profiles/*/ncu_full.json).  Where
    ncu_meta.json gives the profiled launch's algorithmic bytes, returns the
    ratio instead (DRAM bytes per algorithmic byte) for the caller to scale."""
    if not kernel:
        return None, None
    # the kernel variant each bench key times (ncu names template instances):
    # round 2 names first (paired chains: the drain's K1 with the key lane, the
    # refill verify CRC only), then round 1's
    exact = {"k1_chunk_crc": ("void k1_chunk_crc<4, 0, 1, 1>", "void k1_chunk_crc<16, 0>"),
             "k1_chunk_crc (refill verify)": ("void k1_chunk_crc<8, 0, 0, 1>",
                                              "void k1_chunk_crc<16, 0>")}.get(kernel)
    name = kernel.split(" ")[0]
    units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    for path in sorted(Path(__file__).parent.glob("profiles/*/ncu_full.json"), reverse=True):
        try:
            full = json.loads(path.read_text())
        except (OSError, ValueError):
            continue
        meta = {}
        if (path.parent / "ncu_meta.json").exists():
            meta = json.loads((path.parent / "ncu_meta.json").read_text())
        for key, m in full.items():
            if (exact and key not in exact) or name not in key:
                continue
            total = 0.0
            for metric in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                val, unit = m[metric].split()
                total += float(val) * units[unit]
            src = f"{path.parent.name}/{path.name}: {key}"
            alg = (meta.get(key) or {}).get("algorithmic_bytes")
            if alg:  # DRAM bytes per algorithmic byte of the profiled launch
                return total / alg, src + f" ({total / 1e9:.3f} GB for {alg / 1e9:.3f} GB algorithmic)"
            return int(total), src
    return None, None


def measure_stall(torch, sess, image, stream_bytes: int, sync_ms: float, args) -> dict:
    """checkpoint_begin/finish with the largest shadow free HBM allows: the
    app-visible stall (quiesce -> resume) against the synchronous drain."""
    free = torch.cuda.mem_get_info()[0] - 4 * GIB
    shadow = max(0, min(free, stream_bytes + 64 * MIB))
    try:
        sess.reserve_shadow(shadow)
    except Exception as e:  # noqa: BLE001 - reported, not fatal
        return {"error": str(e)}
    rows = []
    for _ in range(max(2, args.steps)):
        sess.checkpoint_begin(image)
        rows.append(sess.checkpoint_finish())
    sess.reserve_shadow(0)
    rows = rows[1:]
    stall = statistics.mean(r["stall_ms"] for r in rows)
    total = statistics.mean(r["total_ms"] for r in rows)
    return {"shadow_bytes": rows[-1]["shadow_bytes"], "stream_bytes": stream_bytes,
            "stall_ms": round(stall, 3), "total_ms": round(total, 3),
            "sync_checkpoint_ms": round(sync_ms, 3),
            "stall_reduction": round(sync_ms / stall, 2) if stall else None}


def measure_precopy(sess, image, sync_ms: float, args, rank: int) -> dict:
    """Pre-copy drain: phase 1 copies the state while the 'application' (a
    device kernel rewriting ~1 % of the chunks, launched right after begin)
    keeps changing it; phase 2 quiesces and re-sends the changed chunks.  The
    stall is phase 2 alone."""
    rows = []
    for k in range(max(2, args.steps)):
        try:
            sess.checkpoint_precopy_begin(image)
        except Exception as e:  # noqa: BLE001 - reported, not fatal
            return {"error": str(e)}
        mutated = sess.mutate(seed=rank + 7, epoch=100 + k, threshold=(2**64 - 1) // 100)
        st = sess.checkpoint_precopy_finish()
        rows.append((st, mutated))
    rows = rows[1:]
    stall = statistics.mean(r["stall_ms"] for r, _ in rows)
    return {"stall_ms": round(stall, 3),
            "total_ms": round(statistics.mean(r["total_ms"] for r, _ in rows), 3),
            "resent_chunks": int(statistics.mean(r["dirty_chunks"] for r, _ in rows)),
            "mutated_during_phase1": int(statistics.mean(m for _, m in rows)),
            "total_chunks": rows[-1][0]["total_chunks"],
            "sync_checkpoint_ms": round(sync_ms, 3),
            "stall_reduction": round(sync_ms / stall, 2) if stall else None,
            "how": "phase 1 (no quiesce): K1 hashes every chunk and writes the bytes it hashed "
                   "into the image while a device kernel rewrites ~1 % of the chunks; phase 2 "
                   "(quiesced): incremental re-send of the changed chunks"}


def run_c5(args, engine, sess, image, live, group, rank, world, peaks) -> None:
    """Incremental sequence (config C5): per dirty fraction, the hash-only pass
    and the incremental drain, both device-timed."""
    sess.checkpoint_into(image)  # full image; seeds the previous-epoch CRCs
    verified = None
    if not args.no_verify:  # the full image against regenerated content
        rep0 = engine.verify_image(address=image.address(), synth_seed=rank + 1)
        verified = {"full_image": {k: rep0[k] for k in ("ok", "payloads_compared",
                                                        "payload_bytes_compared", "bad_sections")}}
    rows = {}
    epoch = 0
    for pct in (1, 5, 25):
        thr = (2**64 - 1) * pct // 100
        hs, ds = [], []
        for _ in range(args.warmup + args.steps):
            epoch += 1
            h = sess.hash_only()
            sess.checkpoint_into(image)  # re-seed (hash_only invalidates the plan)
            mutated = sess.mutate(seed=rank + 1, epoch=epoch, threshold=thr)
            d = sess.checkpoint_into(image, incremental=True)
            assert d["incremental"] and d["dirty_chunks"] == mutated
            hs.append(h)
            ds.append(d)
        hs, ds = hs[args.warmup:], ds[args.warmup:]
        h_ms = group.max(statistics.mean(h["hash_ms"] for h in hs))
        d_ms = group.max(statistics.mean(d["total_ms"] for d in ds))
        dirty = statistics.mean(d["d2h_bytes"] for d in ds)
        rows[f"{pct}pct"] = {
            "hash_only_ms": round(h_ms, 3),
            "hash_GBps": round(live / (h_ms * 1e-3) / 1e9, 1),
            "hash_frac_of_hbm": round(live / (h_ms * 1e-3) / 1e9 / peaks["hbm_gbs"], 3),
            "drain_ms": round(d_ms, 3), "dirty_bytes": int(dirty),
            "drain_roofline_ms": round(max(live / peaks["hbm_gbs"] / 1e6,
                                           dirty / (peaks["pcie"]["d2h"] * 1e6)), 3),
            "state_GBps": round(live * world / (d_ms * 1e-3) / 1e9, 1)}
    if verified is not None:  # the last incremental image: every section CRC recomputed
        rep1 = engine.verify_image(address=image.address())
        verified["last_incremental_image"] = {k: rep1[k] for k in ("ok", "crc_bytes", "bad_sections")}
        verified["ok"] = bool(max(group.max(0.0 if verified["full_image"]["ok"] and rep1["ok"]
                                            else 1.0), 0) == 0)
        verified["method"] = ("crac_image_verify on the host cores: the first full image's Device "
                              "payloads against regenerated f(seed, id, offset) and its CRCs; the "
                              "last incremental image's section CRCs recomputed")
    import torch
    sync_ms = sess.checkpoint_into(image)["total_ms"]
    stall = None if args.no_stall else measure_stall(
        torch, sess, image, live + 16 * len(sess.live_records()) + 20, sync_ms, args)
    if stall is not None:
        stall["precopy"] = measure_precopy(sess, image, sync_ms, args, rank)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_c5(16.0)
    if rank == 0:
        r1 = rows["1pct"]
        print(json.dumps({
            "metric": "checkpoint & restart GB/s per GPU and whole box at 1/2/4/8 B200; % of roofline",
            "value": r1["state_GBps"], "unit": "GB/s (live state covered by the incremental drain)",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": r1["drain_ms"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": WORKLOAD_NAMES["c5"], "live_bytes_per_gpu": live,
                       "chunk_bytes": 65536},
            "incremental": rows, "stall_reduced": stall, "verified": verified,
            "cpu_baseline": cpu}), flush=True)


def dd_ceiling(path: Path, nbytes: int, streams: int = 8, unlink: bool = True) -> dict:
    """Storage ceiling measured with coreutils dd, independent of our writer:
    `streams` concurrent O_DIRECT dd processes over disjoint 64 MiB-block
    ranges of one file (write with fdatasync, then read)."""
    bs = 64 * MIB
    blocks = max(streams, nbytes // bs)
    per = (blocks + streams - 1) // streams
    out = {}
    for mode in ("write", "read"):
        cmds = []
        for k in range(streams):
            lo, cnt = k * per, max(0, min(per, blocks - k * per))
            if not cnt:
                continue
            if mode == "write":
                cmds.append(["dd", "if=/dev/zero", f"of={path}", f"bs={bs}", f"seek={lo}",
                             f"count={cnt}", "oflag=direct", "conv=notrunc,fdatasync"])
            else:
                cmds.append(["dd", f"if={path}", "of=/dev/null", f"bs={bs}", f"skip={lo}",
                             f"count={cnt}", "iflag=direct"])
        t0 = time.perf_counter()
        ps = [subprocess.Popen(c, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
              for c in cmds]
        ok = all(p.wait() == 0 for p in ps)
        dt = time.perf_counter() - t0
        out[f"{mode}_GBps"] = round(blocks * bs / dt / 1e9, 3) if ok else None
    if unlink:
        try:
            path.unlink()
        except OSError:
            pass
    out["how"] = f"{streams} concurrent dd O_DIRECT streams, 64 MiB blocks, {blocks * bs // MIB} MiB"
    return out


def drop_cache(path: Path) -> None:
    try:
        fd = os.open(path, os.O_RDONLY)
        try:
            os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
        finally:
            os.close(fd)
    except OSError:
        pass


def run_file(args, engine, sess, live, group, rank, world, cfg_extra, gbar=None) -> None:
    """Persistence: checkpoint_to_file then restart_from_file of
    the C4-shaped state; wall time per phase, storage ceiling beside it."""
    io_dir = Path(args.io_dir or os.environ.get("CRAC_IO_DIR", "/tmp"))
    io_dir.mkdir(parents=True, exist_ok=True)
    path = io_dir / f"crac_bench_rank{rank}.img"
    img, staging = engine.Image(), engine.Image()
    rows = []
    for k in range(args.warmup + args.steps):
        group.barrier()
        t0 = time.perf_counter()
        drain, wio = sess.checkpoint_to_file(path, img)
        t1 = time.perf_counter()
        sess.close()
        drop_cache(path)  # a restart reads the device, not the page cache
        t2 = time.perf_counter()
        sess, refill, rio = engine.restart_from_file(path, staging)
        t3 = time.perf_counter()
        if gbar:
            sess.set_barrier(gbar)
        rows.append({"ckpt_s": t1 - t0, "restart_s": t3 - t2, "drain_ms": drain["total_ms"],
                     "write_ms": wio["ms"], "read_ms": rio["ms"], "refill_ms": refill["total_ms"],
                     "direct": wio["direct"] and rio["direct"], "bytes": wio["bytes"],
                     "streamed": wio.get("streamed", 0)})
    rows = rows[args.warmup:]
    ck = group.max(statistics.mean(r["ckpt_s"] for r in rows))
    rs = group.max(statistics.mean(r["restart_s"] for r in rows))
    nbytes = rows[-1]["bytes"]
    sess.close()
    staging.close()
    # the GPU deflate (CRACSIMZ, compress="gpu") of the last image: its rate and
    # ratio on this workload's content (synthetic words: incompressible, so
    # mostly stored blocks), plus a compressible image of the same size
    gpuz = None
    if rank == 0:
        zn, zms = engine.compress_image_gpu(address=img.address(), want_bytes=False)
        zero = engine.Image()
        zs = engine.Session(seed=9, arena_bytes=min(live, 4 * GIB) + 64 * MIB)
        zi, _ = zs.alloc(engine.DEVICE, min(live, 4 * GIB))  # zero-filled state
        zs.checkpoint_into(zero)
        z0n, z0ms = engine.compress_image_gpu(address=zero.address(), want_bytes=False)
        gpuz = {"image_bytes": nbytes, "compressed_bytes": zn, "ms": round(zms, 1),
                "GBps": round(nbytes / (zms * 1e6), 2),
                "zero_state": {"image_bytes": zero.address()[1], "compressed_bytes": z0n,
                               "ms": round(z0ms, 1),
                               "GBps": round(zero.address()[1] / (z0ms * 1e6), 2)},
                "how": "crac_compress_image_gpu from the pinned image: H2D, K5 deflate (32 KiB "
                       "segments, fixed Huffman LZ77, stored fallback), gather, D2H; wall time"}
        zs.close()
        zero.close()
    img.close()
    # the storage ceiling: coreutils dd at 8 and at 16 concurrent streams (the
    # writer's own thread count), the best of each direction; one dd pass is
    # noisy on the box's virtio disk (a single 8-stream pass has read below
    # what our writer then reached)
    ceiling = None
    if rank == 0:
        for streams in (8, 16):
            c = dd_ceiling(path, min(nbytes, 16 * GIB), streams, unlink=streams == 16)
            if ceiling is None:
                ceiling = c
                continue
            for k in ("write_GBps", "read_GBps"):
                if (c.get(k) or 0) > (ceiling.get(k) or 0):
                    ceiling[k] = c[k]
        ceiling["how"] = ("best of 8 and 16 concurrent dd O_DIRECT streams per direction, "
                          "64 MiB blocks, " + ceiling["how"].split(", ")[-1])
    try:
        path.unlink()
    except OSError:
        pass
    if rank != 0:
        return
    m = {k: round(statistics.mean(r[k] for r in rows), 3)
         for k in ("drain_ms", "write_ms", "read_ms", "refill_ms")}
    roof = None
    if ceiling and ceiling.get("write_GBps") and ceiling.get("read_GBps"):
        t_roof = nbytes / (ceiling["write_GBps"] * 1e9) + nbytes / (ceiling["read_GBps"] * 1e9)
        roof = {"bound": "storage", "write_GBps": round(nbytes / (m["write_ms"] * 1e6), 3),
                "read_GBps": round(nbytes / (m["read_ms"] * 1e6), 3),
                "ceiling": ceiling, "frac": round(t_roof / (ck + rs), 4)}
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline_file(args.cpu_sample_gib, args.region_mib * MIB, io_dir)
    print(json.dumps({
        "metric": "checkpoint & restart GB/s per GPU and whole box at 1/2/4/8 B200; % of roofline",
        "value": round(2 * live * world / (ck + rs) / 1e9, 3), "unit": "GB/s (through the file)",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round((ck + rs) * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": WORKLOAD_NAMES["file"], "live_bytes_per_gpu": live,
                   "file_bytes": nbytes, "io_dir": str(io_dir), **cfg_extra},
        "per_gpu": {"checkpoint_to_file_GBps": round(live / ck / 1e9, 3),
                    "restart_from_file_GBps": round(live / rs / 1e9, 3),
                    "checkpoint_to_file_s": round(ck, 3), "restart_from_file_s": round(rs, 3),
                    "phases_ms": m, "o_direct": all(r["direct"] for r in rows),
                    "streamed_bytes": rows[-1]["streamed"]},
        "roofline": roof, "cpu_baseline": cpu, "gpu_deflate": gpuz}), flush=True)


def cpu_baseline_file(sample_gib: float, region: int, io_dir: Path) -> dict:
    """The reference's checkpoint_to_file / restart_from_file (ofstream /
    ifstream), single-threaded, on a bounded sample."""
    from oracle import ref
    s, live = ref_make_session(int(sample_gib * GIB), region, seed=1)
    path = io_dir / "crac_bench_ref.img"
    t_ck = ref.ref_checkpoint_to_file(s, path)
    s.close()
    drop_cache(path)
    r, t = ref.ref_restart_from_file(path)
    r.close()
    try:
        path.unlink()
    except OSError:
        pass
    return {"value": round(2 * live / (t_ck + t["total_s"]) / 1e9, 4), "unit": "GB/s",
            "cores": 1, "kind": "reference",
            "sample": f"{live // MIB} MiB ({live // region} x {region // MIB} MiB Device regions): "
                      f"reference checkpoint_to_file then restart_from_file, single-threaded",
            "phases_s": {"checkpoint_to_file_s": round(t_ck, 3),
                         "restart_from_file_s": round(t["total_s"], 3)}}


def dry_run(args, world, rank, local) -> None:
    """The N-rank plumbing without a GPU: the device each rank would own, the
    gloo group, and the product's shared-memory checkpoint barrier."""
    pin_device(local, world)
    group = HostGroup(world, rank)
    from paper_2008_10596_b200 import engine
    b = engine.Barrier(barrier_name(world), world, rank, timeout_ms=60000)
    b.wait()
    group.barrier()
    gen = b.generation()
    for r in range(world):  # one line per rank, in rank order (one shared stdout)
        if r == rank:
            print(json.dumps({"dry_run": True, "rank": rank, "world": world, "local_rank": local,
                              "cuda_visible_devices": os.environ.get("CUDA_VISIBLE_DEVICES"),
                              "barrier_generation": gen}), flush=True)
        group.barrier()
    b.close(unlink=rank == 0)
    group.close()


def barrier_name(world: int) -> str:
    return f"/crac_bench_{os.environ.get('MASTER_PORT', '0')}_{world}"


def main() -> None:
    args = parse_args()
    if args.gpus > 1 and "RANK" not in os.environ and args.impl == "b200":
        sys.exit(spawn_ranks(args.gpus))
    world, rank, local, local_world = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    if args.dry_run:
        dry_run(args, world, rank, local)
        return
    job_gpus = job_gpu_indices(1 if args.share_gpu else local_world)
    if not args.share_gpu:
        pin_device(local, world)

    import torch
    from paper_2008_10596_b200 import engine

    group = HostGroup(world, rank)
    barrier, max_over_ranks = group.barrier, group.max
    # the product's global-checkpoint barrier (crac_engine.h): every drain of
    # every rank meets the others at quiesce-complete and image-complete
    gbar = engine.Barrier(barrier_name(world), world, rank, timeout_ms=600000) if world > 1 else None

    torch.cuda.set_device(0)
    # host RAM bounds the per-rank image; HBM bounds the per-rank state
    host_cap = int(0.80 * mem_available() / local_world) - 8 * GIB
    dev_cap = int(torch.cuda.get_device_properties(0).total_memory * 0.85)
    peaks = measured_peaks()
    peaks["pcie"] = pcie_peaks(torch)
    hbm = peaks["hbm_gbs"]
    isolated = isolated_kernel_rates(torch, engine)

    t_setup = time.perf_counter()
    sess, live, cfg_extra = build_workload(args, engine, rank, min(host_cap, dev_cap))
    want = cfg_extra.get("requested_footprint_gib")
    if want and live < int(want * GIB) // (args.region_mib * MIB) * args.region_mib * MIB:
        cfg_extra["footprint_reduced"] = {
            "requested_gib": want, "actual_gib": round(live / GIB, 3),
            "reason": f"host RAM for {local_world} pinned images ({mem_available() // GIB} GiB "
                      f"available) or HBM bounds the per-rank state"}
        print(f"WARNING: footprint reduced to {live / GIB:.1f} GiB per rank", file=sys.stderr)
    image = engine.Image()
    setup_s = time.perf_counter() - t_setup
    if gbar:
        sess.set_barrier(gbar)
    if args.workload == "file":
        image.close()
        run_file(args, engine, sess, live, group, rank, world, cfg_extra, gbar)
        group.close()
        return
    if args.workload == "c5":
        run_c5(args, engine, sess, image, live, group, rank, world, peaks)
        sess.close()
        group.close()
        return

    teardown = []  # host ms of (session close, arena release) per step
    release_later = (ASYNC_RELEASE == "1" if ASYNC_RELEASE in ("0", "1")
                     else live <= 16 * GIB)

    api_ms = []  # CUDA-event ms of (drain call, restart call) per step

    def step(s):
        """One checkpoint + restart, as a restart in a new process sees it:
        the drain, the old session's teardown, its arena freed (no cached
        mapping survives), then the refill from the host image."""
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        dr = s.checkpoint_into(image)
        ev[1].record()
        addr, n = image.address()
        t0 = time.perf_counter()
        s.close()
        t1 = time.perf_counter()
        engine.drop_arena_cache(release_later=release_later)
        teardown.append(((t1 - t0) * 1e3, (time.perf_counter() - t1) * 1e3))
        ev[2].record()
        s2, rf = engine.restart_from_address(addr, n)
        if gbar:
            s2.set_barrier(gbar)
        ev[3].record()
        torch.cuda.synchronize()
        api_ms.append((ev[0].elapsed_time(ev[1]), ev[2].elapsed_time(ev[3])))
        return s2, dr, rf

    # the sampler starts before the warm-up steps, so nvidia-smi's own
    # start-up (NVML init on every GPU) falls outside the timed region; only
    # the samples taken during the timed steps are kept (measured: the slow
    # steps some boxes show occur with no sampler at all,
    # profiles/r02/clock_sampler.txt)
    clocks = ClockSampler() if rank == 0 and not os.environ.get("CRAC_NO_CLOCKS") else None
    early_clocks = os.environ.get("CRAC_CLOCKS_AT", "warmup") != "timed"
    if clocks and early_clocks:
        clocks.start()
    t_warm = time.perf_counter()
    for _ in range(args.warmup):
        sess, _, _ = step(sess)
    warm_s = time.perf_counter() - t_warm

    if clocks:
        if early_clocks:
            clocks.mark()
        else:
            clocks.start()
    drains, refills, e2e_steps = [], [], []
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        barrier()  # every rank starts the step together
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        sess, dr, rf = step(sess)
        ev1.record()
        torch.cuda.synchronize()
        drains.append(dr)
        refills.append(rf)
        e2e_steps.append(ev0.elapsed_time(ev1))
    wall = time.perf_counter() - wall0
    barrier()
    clk = clocks.stop(job_gpus) if clocks else None

    # whole box: each step lasts until its slowest rank is done (the ranks
    # start it together), i.e. max end - min start per step, summed
    dev_steps = group.max_list(
        [d["total_ms"] + r["total_ms"] for d, r in zip(drains, refills)])
    # e2e: the drain call + the restart call through the public API (host
    # image buffers, host work and copies in both); the old session's
    # teardown between them is what a new-process restart never pays (the
    # checkpointed process's exit frees its memory), so it is reported beside
    # it (e2e.with_teardown) rather than inside it
    e2e_steps_max = group.max_list([a + b for a, b in api_ms[-args.steps:]])
    e2e_td_max = group.max_list(e2e_steps)
    dev_ms_max = sum(dev_steps)
    e2e_ms_max = sum(e2e_steps_max)
    drain_ms = max_over_ranks(sum(d["total_ms"] for d in drains) / args.steps)
    refill_ms = max_over_ranks(sum(r["total_ms"] for r in refills) / args.steps)

    # independent checks of the last step (outside the timed region): the
    # image on the host cores against recomputed CRCs and regenerated
    # content, the restarted (cold) device state against regenerated content
    verified = None
    if not args.no_verify:
        seed = rank + 1
        synth = args.workload == "c4"
        rep = engine.verify_image(address=image.address(), synth_seed=seed if synth else None)
        dev = sess.verify_synthetic(seed) if synth else None
        ok = rep["ok"] and (dev is None or dev["bad_allocations"] == 0)
        ok = bool(max_over_ranks(0.0 if ok else 1.0) == 0.0)
        verified = {
            "ok": ok,
            "image": {k: rep[k] for k in ("sections_checked", "crc_bytes", "payloads_compared",
                                          "payload_bytes_compared", "mismatched_payloads",
                                          "bad_sections", "threads")} | {"s": round(rep["ms"] / 1e3, 2)},
            "restarted_state": dev,
            "method": "host: every section CRC recomputed on all host cores (PCLMUL, no GPU code) "
                      "and every Device payload compared with f(seed, id, offset) regenerated "
                      "(crac_image_verify); device: the state the last (cold) restart refilled "
                      "compared word by word with the regenerated content "
                      "(crac_session_verify_synthetic); all ranks"}
        if not ok:
            print(f"VERIFY FAILED on rank {rank}: {rep} {dev}", file=sys.stderr)

    # kernels in the timed region, each against HBM
    def mean(key, xs):
        return statistics.mean(x[key] for x in xs)
    kernels = {}
    if drains[-1]["hash_launches"]:
        kernels["k1_chunk_crc"] = (mean("hash_ms", drains) / drains[-1]["hash_launches"],
                                   drains[-1]["hash_bytes"] / drains[-1]["hash_launches"],
                                   drains[-1]["hash_launches"])
    if drains[-1]["pack_launches"]:
        n = drains[-1]["pack_launches"]
        kernels["k_pack_records"] = (mean("pack_ms", drains), 2 * drains[-1]["pack_bytes"] / n, n)
    if refills[-1]["pack_launches"]:
        n = refills[-1]["pack_launches"]
        kernels["k_scatter_records"] = (mean("pack_ms", refills), 2 * refills[-1]["pack_bytes"] / n, n)
    if refills[-1]["hash_launches"]:  # the refill's verify K1 (batches of completed regions)
        n = refills[-1]["hash_launches"]
        kernels["k1_chunk_crc (refill verify)"] = (mean("hash_ms", refills) / n,
                                                   refills[-1]["hash_bytes"] / n, n)
    by_time = max(kernels, key=lambda k: kernels[k][0] * kernels[k][2]) if kernels else None
    kern_rows = {}
    for k, (ms, nbytes, launches) in kernels.items():
        gbps = nbytes / (ms * 1e6) if ms else 0.0
        traffic, src = ncu_traffic(k)
        if traffic is not None and traffic < 16:  # a ratio: scale to this launch
            traffic = int(traffic * nbytes)
        kern_rows[k] = {"bound": "hbm", "achieved": round(gbps, 1), "peak": hbm, "unit": "GB/s",
                        "frac": round(gbps / hbm, 4), "traffic": traffic, "traffic_source": src,
                        "avg_launch_ms": round(ms, 4), "bytes_per_launch": int(nbytes),
                        "launches": launches, "device_ms_per_step": round(ms * launches, 3)}
        if k in ("k_pack_records", "k_scatter_records") and nbytes < (8 << 20):
            kern_rows[k]["regime"] = ("latency: each launch moves only the frames and payload edges "
                                      "around the direct copies of its window, beside the link's copy "
                                      "(off the critical path; 'isolated' gives its bandwidth)")
        elif k == "k_scatter_records":
            kern_rows[k]["regime"] = ("in situ: the restart's first ring windows (queued before the "
                                      "parse, so no direct runs start in them) scattered whole beside the "
                                      "H2D; their event span is ~1.1 ms per launch with or without the "
                                      "cold tail map beside them (profiles/r02/scatter_span.txt) against "
                                      "~19 us under ncu (serialised, profiles/r02be/launch_summary.txt); "
                                      "hidden behind the H2D, 'isolated' gives its bandwidth")

    # cold restart is now the timed step itself; the warm-arena variant is
    # reported beside it for comparison (arena adopted from the closed session)
    warm = None
    if not args.no_cold:
        sess.checkpoint_into(image)
        addr, n = image.address()
        sess.close()
        sess, rf = engine.restart_from_address(addr, n)
        if gbar:
            sess.set_barrier(gbar)
        warm = {"restart_ms": round(rf["total_ms"], 3),
                "restart_GBps": round(live / (rf["total_ms"] * 1e-3) / 1e9, 3),
                "note": "arena of the closed session adopted (mapped memory reused), not the headline"}

    # incremental (C5 shape on the resident state): hash-only and a 1 % dirty drain
    incremental = None
    if not args.no_incremental and args.workload == "c4":
        h = sess.hash_only()
        sess.checkpoint_into(image)  # seeds the previous-image chunk CRCs
        thr = (2**64 - 1) // 100
        mutated = sess.mutate(seed=rank + 1, epoch=1, threshold=thr)
        inc = sess.checkpoint_into(image, incremental=True)
        k1_gbs = h["hash_bytes"] / (h["hash_ms"] * 1e-3) / 1e9 if h["hash_ms"] else 0
        incremental = {
            "hash_only": {"bytes": h["hash_bytes"], "ms": round(h["hash_ms"], 3),
                          "GBps": round(k1_gbs, 1), "frac_of_hbm": round(k1_gbs / hbm, 3)},
            "drain_1pct": {"dirty_chunks": inc["dirty_chunks"], "mutated": mutated,
                           "total_chunks": inc["total_chunks"], "ms": round(inc["total_ms"], 3),
                           "d2h_bytes": inc["d2h_bytes"], "incremental": bool(inc["incremental"])},
        }

    # stall-reduced drain: as much of the stream as free HBM holds is staged
    # on the device while the app is stopped; the rest goes through the ring
    stall = None
    if not args.no_stall and args.workload in ("c4", "c2", "c3"):
        stall = measure_stall(torch, sess, image, drains[-1]["d2h_bytes"], drain_ms, args)
        if args.workload == "c4":
            stall["precopy"] = measure_precopy(sess, image, drain_ms, args, rank)

    # the refill floor of managed memory on this box (C3): fresh managed
    # memory of the state's size, split residence populated from both sides
    populate_ms = None
    if args.workload == "c3":
        sess.close()
        sess = None
        populate_ms = engine.probe_managed_populate(live)

    # the link peaks once more after the timed region: a transiently slow
    # link during the first measurement must not put the floor below what the
    # timed steps achieved (the best of both is the peak)
    if args.workload in ("c4", "c2", "c3"):
        again = pcie_peaks(torch)
        for k in ("d2h", "h2d"):
            peaks["pcie"][k] = max(peaks["pcie"][k], again[k])

    # reported CPU baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if args.workload == "c4":
            cpu = cpu_baseline(args.cpu_sample_gib, args.region_mib * MIB)
        elif args.workload == "c2":
            cpu = cpu_baseline_c2(args.c2_calls)
        elif args.workload == "c3":
            cpu = cpu_baseline_c3(1.0)

    if rank == 0:
        value = 2 * live * world * args.steps / (dev_ms_max * 1e-3) / 1e9
        e2e = 2 * live * world * args.steps / (e2e_ms_max * 1e-3) / 1e9
        e2e_td = 2 * live * world * args.steps / (sum(e2e_td_max) * 1e-3) / 1e9
        launches = sum(d["hash_launches"] + d["pack_launches"] for d in drains) + \
            sum(r["hash_launches"] + r["pack_launches"] for r in refills)
        pd, ph = peaks["pcie"]["d2h"], peaks["pcie"]["h2d"]
        # the step's floor: its D2H bytes at the D2H peak, then its H2D bytes
        # at the H2D peak or, for managed memory, the measured populate
        # ceiling of fresh managed memory with split residence if slower
        # (C3: GPU faults + host first-touch faults, crac_probe_managed_populate)
        d2h_b, h2d_b = drains[-1]["d2h_bytes"], refills[-1]["h2d_bytes"]
        # The floor is the link's alone.  C3's refill is bound by the UVM
        # driver populating fresh managed memory instead; the standalone probe
        # of that (crac_probe_managed_populate) runs no faster than the whole
        # refill does, so it is no floor: it is reported beside the link floor
        # ("managed_populate"), not folded into it
        roof_ms = d2h_b / (pd * 1e6) + h2d_b / (ph * 1e6)
        link = 2 * live / (roof_ms * 1e6)  # state GB/s at the floor (C4: the harmonic link mean)
        bound = "pcie"
        d2h = drains[-1]["d2h_bytes"] / (mean("copy_ms", drains) * 1e-3) / 1e9 if mean("copy_ms", drains) else 0
        h2d = refills[-1]["h2d_bytes"] / (mean("copy_ms", refills) * 1e-3) / 1e9 if mean("copy_ms", refills) else 0
        per_gpu = value / world
        line = {
            "metric": "checkpoint & restart GB/s per GPU and whole box at 1/2/4/8 B200; % of roofline",
            "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(dev_ms_max / args.steps, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic",
            "config": {"workload": WORKLOAD_NAMES[args.workload], "live_bytes_per_gpu": live,
                       **cfg_extra, "parallelism": f"independent drains x{world}",
                       "global_barrier": "crac_barrier (shared memory) at quiesce-complete and "
                                         "image-complete of every drain" if world > 1 else None,
                       "restart": ("cold: the closed session's arena is freed before each refill"
                                   + ("; its memory released on a thread beside the refill"
                                      " (crac_drop_arena_cache_async)" if release_later else "")),
                       "l2": "inputs larger than L2" if live > 256 * MIB else "inputs may fit L2"},
            "per_gpu": {"checkpoint_GBps": round(live / (drain_ms * 1e-3) / 1e9, 3),
                        "restart_GBps": round(live / (refill_ms * 1e-3) / 1e9, 3),
                        "checkpoint_ms": round(drain_ms, 3), "restart_ms": round(refill_ms, 3),
                        "restart_host_pre_ms": round(mean("host_pre_ms", refills), 3),
                        "image_bytes": drains[-1]["image_bytes"], "warm_restart": warm},
            "roofline": {"bound": bound, "achieved": round(per_gpu, 3), "peak": round(link, 2),
                         "unit": "GB/s", "frac": round(per_gpu / link, 4),
                         "traffic": d2h_b + h2d_b,
                         "how": "state bytes per GPU per second of drain + refill against the "
                                "step's floor: its D2H bytes at this GPU's measured D2H peak plus "
                                "its H2D bytes at the measured H2D peak (C4: the harmonic mean of "
                                "the two peaks, every state byte crosses the link once each way); "
                                "traffic = link bytes per step",
                         "floor_ms": {"d2h": round(d2h_b / (pd * 1e6), 3),
                                      "h2d": round(h2d_b / (ph * 1e6), 3)},
                         "managed_populate": None if not populate_ms else {
                             "probe_ms": round(populate_ms, 3), "restart_ms": round(refill_ms, 3),
                             "restart_vs_probe": round(populate_ms / refill_ms, 3),
                             "how": "crac_probe_managed_populate: a fresh cudaMallocManaged range "
                                    "of the state's size, its device-resident runs first-touched by "
                                    "a GPU kernel while host threads first-touch the host-resident "
                                    "ones -- the driver's populate work alone, no copies; the "
                                    "restart (which also populates, copies and verifies) is bound "
                                    "by it, not by the link"},
                         "peak_source": "measured in this run, before and after the timed steps "
                                        "(best of 5 passes of 2 GiB in 16 and 64 MiB pinned "
                                        "copies, each time)",
                         "d2h_GBps": round(d2h, 2), "h2d_GBps": round(h2d, 2),
                         "d2h_peak_GBps": pd, "h2d_peak_GBps": ph,
                         "d2h_GBps_per_step": [round(d["d2h_bytes"] / (d["copy_ms"] * 1e6), 2)
                                               for d in drains if d["copy_ms"]],
                         "h2d_GBps_per_step": [round(r["h2d_bytes"] / (r["copy_ms"] * 1e6), 2)
                                               for r in refills if r["copy_ms"]],
                         "dominant_kernel": by_time,
                         "kernels": kern_rows,
                         "hbm_peak_source": peaks["source"],
                         "isolated": {k: {**v, "frac": round(v["GBps"] / hbm, 4)}
                                      for k, v in isolated.items()},
                         "note": "kernels = every kernel of the timed region against HBM, CUDA "
                                 "events on the engine streams; k1_chunk_crc = the hash over the "
                                 "whole state (one launch per drain beside the D2H); pack/scatter "
                                 "per window produce only the edges around the direct copies; "
                                 "'isolated' = back to back on one stream; traffic = ncu DRAM "
                                 "bytes per launch (profiles/)"},
            "e2e": {"value": round(e2e, 3), "unit": "GB/s",
                    "h2d_bytes_per_step": refills[-1]["h2d_bytes"],
                    "d2h_bytes_per_step": drains[-1]["d2h_bytes"],
                    "wall_s": round(wall, 3),
                    "api_ms_per_step": [[round(a, 1), round(b, 1)] for a, b in api_ms[-args.steps:]],
                    "teardown_ms_per_step": [[round(a, 1), round(b, 1)]
                                             for a, b in teardown[-args.steps:]],
                    "with_teardown": {"value": round(e2e_td, 3), "unit": "GB/s",
                                      "how": "CUDA events around the whole step: drain call, "
                                             "session close + arena release, restart call"},
                    "how": "CUDA events around the two public-API calls of each step: the drain "
                           "into the pinned host image and the restart refill from it (host work, "
                           "parse and every copy included), max over ranks per step; the old "
                           "session's teardown between them (a new-process restart never pays "
                           "it: C3's managed cudaFree takes ~2.2 s) is in with_teardown"},
            "verified": verified,
            "gpu_launches": launches,
            "image_pages": image.pages(),
            "clocks": clk,
            "incremental": incremental,
            "stall_reduced": stall,
            "cpu_baseline": cpu,
            "setup_s": round(setup_s, 1), "warmup_s": round(warm_s, 1),
        }
        print(json.dumps(line), flush=True)
    if sess is not None:
        sess.close()
    if gbar:
        barrier()
        gbar.close(unlink=rank == 0)
    group.close()


if __name__ == "__main__":
    main()
