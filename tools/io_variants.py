"""Which file set-up lets parallel O_DIRECT writes run at the disk's speed?
Fresh 16 GiB file per variant; the parallel writer (image_io.cpp) with its
experiment knobs, and coreutils dd beside it.

    python tools/io_variants.py [dir] [GiB]
"""
import mmap
import os
import subprocess
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2008_10596_b200 import engine  # noqa: E402

MIB = 1 << 20


def dd(p: Path, n: int, streams: int = 8) -> float:
    bs, blocks = 64 * MIB, n // (64 * MIB)
    per = blocks // streams
    t0 = time.perf_counter()
    ps = [subprocess.Popen(["dd", "if=/dev/zero", f"of={p}", f"bs={bs}", f"seek={k * per}",
                            f"count={per}", "oflag=direct", "conv=notrunc,fdatasync"],
                           stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
          for k in range(streams)]
    for q in ps:
        q.wait()
    return blocks * bs / (time.perf_counter() - t0) / 1e9


def main():
    d = Path(sys.argv[1] if len(sys.argv) > 1 else "/tmp")
    n = int(float(sys.argv[2] if len(sys.argv) > 2 else 16) * (1 << 30))
    buf = mmap.mmap(-1, n)
    for off in range(0, n, MIB):
        buf[off:off + 8] = off.to_bytes(8, "little")
    p = d / "crac_io_variants.bin"
    for rep in range(2):
        p.unlink(missing_ok=True)
        print(f"dd fresh file: {dd(p, n):.2f} GB/s", flush=True)
        print(f"dd same file again (overwrite): {dd(p, n):.2f} GB/s", flush=True)
        for pre in ("fallocate", "truncate", "none"):
            for fdpt in (False, True):
                os.environ["CRAC_IO_PREALLOC"] = pre
                if fdpt:
                    os.environ["CRAC_IO_FD_PER_THREAD"] = "1"
                else:
                    os.environ.pop("CRAC_IO_FD_PER_THREAD", None)
                p.unlink(missing_ok=True)
                w = engine.write_file(p, buf, threads=8, chunk_bytes=64 * MIB)
                print(f"writer prealloc={pre:9s} fd_per_thread={int(fdpt)}: {w['GBps']:.2f} GB/s",
                      flush=True)
    p.unlink(missing_ok=True)


if __name__ == "__main__":
    main()
