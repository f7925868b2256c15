"""Parallel image-file reader variants against dd on one 16 GiB file.
    python tools/io_read_variants.py [dir] [GiB]"""
import mmap
import os
import subprocess
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2008_10596_b200 import engine  # noqa: E402

MIB = 1 << 20


def drop(p):
    fd = os.open(p, os.O_RDONLY)
    os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
    os.close(fd)


def dd_read(p, n, streams=8):
    bs, blocks = 64 * MIB, n // (64 * MIB)
    per = blocks // streams
    t0 = time.perf_counter()
    ps = [subprocess.Popen(["dd", f"if={p}", "of=/dev/null", f"bs={bs}", f"skip={k * per}",
                            f"count={per}", "iflag=direct"], stdout=subprocess.DEVNULL,
                           stderr=subprocess.DEVNULL) for k in range(streams)]
    for q in ps:
        q.wait()
    return blocks * bs / (time.perf_counter() - t0) / 1e9


def main():
    d = Path(sys.argv[1] if len(sys.argv) > 1 else "/tmp")
    n = int(float(sys.argv[2] if len(sys.argv) > 2 else 16) * (1 << 30))
    buf = mmap.mmap(-1, n)
    p = d / "crac_read_variants.bin"
    engine.write_file(p, buf)
    for rep in range(2):
        drop(p)
        print(f"dd read 8 streams: {dd_read(p, n):.2f} GB/s", flush=True)
        for bounce in (False, True):
            for threads, chunk in ((8, 64), (16, 64), (8, 16), (32, 16)):
                if bounce:
                    os.environ["CRAC_IO_BOUNCE_READ"] = "1"
                else:
                    os.environ.pop("CRAC_IO_BOUNCE_READ", None)
                drop(p)
                _, r = engine.read_file(p, threads=threads, chunk_bytes=chunk * MIB)
                print(f"reader threads {threads:2d} piece {chunk:3d} MiB bounce={int(bounce)}: "
                      f"{r['GBps']:.2f} GB/s", flush=True)
    p.unlink()


if __name__ == "__main__":
    main()
