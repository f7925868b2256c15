"""Builds libcrac_b200.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

    python -m paper_2008_10596_b200.build [--force]

Objects go to build/obj (git-ignored); the shared library lands next to this
file so it travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libcrac_b200.so"
PRELOAD = PKG / "libcrac_preload.so"   # cudart interposer
APP = ROOT / "build" / "interpose_app"  # test application, shared cudart

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + [
    "-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC,-O3,-Wall,-Wno-unused-function",
    "-I", str(ROOT / "include"), "-I", str(CSRC),
]
# per-file extra flags
EXTRA = {
    "std_kernels.cu": ["-fmad=false"],   # reference f32 kernels are built without contraction
    "kernels.cu": ["-Xptxas", "-v"] if os.environ.get("CRAC_PTXAS_V") else [],
}
SOURCES = ["kernels.cu", "device_core.cu", "drain.cu", "std_kernels.cu", "deflate.cu",
           "shim.cpp", "image.cpp", "image_io.cpp", "crc_host.cpp", "ckpt_engine.cpp", "capi.cpp",
           "global_barrier.cpp", "verify.cpp", "compress.cu"]


def _headers_mtime() -> float:
    paths = list((ROOT / "include").rglob("*.h*")) + list(CSRC.glob("*.h*"))
    return max(p.stat().st_mtime for p in paths)


def _compile(src: str, force: bool, hdr_mtime: float) -> Path:
    s = CSRC / src
    o = OBJ / (src + ".o")
    if not force and o.exists() and o.stat().st_mtime >= max(s.stat().st_mtime, hdr_mtime):
        return o
    cmd = [NVCC, *COMMON, *EXTRA.get(src, []), "-c", str(s), "-o", str(o)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip() and os.environ.get("CRAC_BUILD_VERBOSE"):
        print(r.stderr, file=sys.stderr)
    return o


def build(force: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    hdr = _headers_mtime()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, hdr), SOURCES))
    newest = max(o.stat().st_mtime for o in objs)
    if force or not LIB.exists() or LIB.stat().st_mtime < newest:
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lz", "-lpthread",
               "-Xlinker", "--no-undefined"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    _build_preload(force)
    return LIB


def _stale(out: Path, *deps: Path) -> bool:
    return not out.exists() or out.stat().st_mtime < max(d.stat().st_mtime for d in deps)


def _build_preload(force: bool) -> None:
    """libcrac_preload.so: host C++ (g++), links libcrac_b200.so by $ORIGIN;
    plus the shared-cudart test application it is exercised with."""
    src = CSRC / "preload.cpp"
    hdrs = [ROOT / "include" / "crac_preload.h", ROOT / "include" / "crac_engine.h"]
    if force or _stale(PRELOAD, src, LIB, *hdrs):
        cmd = ["g++", "-std=c++20", "-O2", "-g", "-fPIC", "-shared", "-Wall",
               "-I", str(ROOT / "include"), "-I", "/usr/local/cuda/include",
               str(src), "-o", str(PRELOAD), "-L", str(PKG), "-l:libcrac_b200.so",
               "-Wl,-rpath,$ORIGIN", "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"preload build failed:\n{r.stdout}\n{r.stderr}")
    app_src = ROOT / "tests" / "native" / "interpose_app.cu"
    if force or _stale(APP, app_src):
        cmd = [NVCC, *ARCH, "-O2", "-std=c++17", "-cudart", "shared", str(app_src),
               "-o", str(APP), "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"interpose_app build failed:\n{r.stdout}\n{r.stderr}")


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
