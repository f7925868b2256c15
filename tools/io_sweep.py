"""Sweep of the parallel image-file writer/reader (paper_2008_10596_b200
image_io.cpp, through the C-ABI; no GPU) on one directory:
threads x piece size x piece layout, write (with fdatasync) then read.

    python tools/io_sweep.py [dir] [GiB]
"""
import mmap
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2008_10596_b200 import engine  # noqa: E402


def main():
    d = Path(sys.argv[1] if len(sys.argv) > 1 else "/tmp")
    n = int(float(sys.argv[2] if len(sys.argv) > 2 else 16) * (1 << 30))
    buf = mmap.mmap(-1, n)
    for off in range(0, n, 1 << 20):
        buf[off:off + 8] = off.to_bytes(8, "little")
    p = d / "crac_io_sweep.bin"
    for layout in ("striped", "interleave"):
        os.environ["CRAC_IO_LAYOUT"] = layout
        for threads in (4, 8, 16, 32):
            for chunk in (16, 64, 256):
                w = engine.write_file(p, buf, threads=threads, chunk_bytes=chunk << 20)
                fd = os.open(p, os.O_RDONLY)
                os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
                os.close(fd)
                _, r = engine.read_file(p, threads=threads, chunk_bytes=chunk << 20)
                print(f"{layout:10s} threads {threads:2d} piece {chunk:3d} MiB: write "
                      f"{w['GBps']:.2f} GB/s, read {r['GBps']:.2f} GB/s "
                      f"(direct {w['direct']}/{r['direct']})", flush=True)
    p.unlink()


if __name__ == "__main__":
    main()
