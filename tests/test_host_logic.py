"""CPU tier: host-side C++ logic of the engine, compiled natively here.

* HoleIndex (O(log n) first fit) vs the reference's linear first fit with
  two-sided coalescing (ref: src/device_core.cpp:45-103).
"""
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_hole_index_matches_reference_first_fit(tmp_path):
    exe = tmp_path / "hole_index_test"
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "native" / "hole_index_test.cpp"), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe), "60"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.strip() == "ok"
