"""Fuzz campaign over the randomized cross-path tests (many seeds, one process).
    python tools/fuzz_paths.py <first-seed> <count>"""
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
from paper_2008_10596_b200 import engine as eng  # noqa: E402
import test_gpu_parity as T  # noqa: E402

first, count = int(sys.argv[1]), int(sys.argv[2])
bad = 0
for seed in range(first, first + count):
    for name, fn in (("device", lambda sd: T.test_random_mixed_paths_agree(eng, sd)),
                     ("managed", lambda sd: T.test_random_managed_and_pinned_paths_agree(
                         eng, sd, Path(tempfile.mkdtemp()))),
                     ("churn", lambda sd: T.test_random_churn_paths_agree(eng, sd))):
        try:
            fn(seed)
        except Exception as e:  # noqa: BLE001
            bad += 1
            print(f"seed {seed} {name}: FAILED {type(e).__name__}: {str(e)[:300]}", flush=True)
print(f"done: {count} seeds, {bad} failures", flush=True)
