"""TEST INFRASTRUCTURE: regenerates tests/golden/ from the reference library.

    python oracle/make_golden.py        (needs oracle/_ref built: make -C oracle)

Every golden image is produced by the UNMODIFIED reference (oracle/_ref/
libcracsim_ref.so compiled from /root/reference/proj/src) through its own
public API, so the fixtures pin parity without /root/reference at run time.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle import ref  # noqa: E402
import workloads  # noqa: E402

GOLD = ROOT / "tests" / "golden"


def main() -> None:
    GOLD.mkdir(parents=True, exist_ok=True)
    manifest = {}

    def save(name: str, image: bytes, how: str) -> None:
        (GOLD / f"{name}.bin").write_bytes(image)
        summ = ref.ref_summarize(image)
        manifest[name] = {"how": how, "bytes": len(image), "lengths": summ["lengths"],
                          "crcs": [f"{c:08x}" for c in summ["crcs"]]}

    save("empty", ref.ref_fixture_image(0), "test_image.cpp:14-19 empty_snapshot")
    save("rich", ref.ref_fixture_image(1), "test_image.cpp:24-52 rich_snapshot")

    s = ref.RefSession(seed=3, arena_bytes=1 << 22)
    workloads.drive_small(s, seed=1)
    save("small_session", s.checkpoint()[0], "tests/workloads.py drive_small(seed=1), seed 3, 4 MiB arena")

    s = ref.RefSession(seed=1, arena_bytes=1 << 24)
    workloads.build_regions(s, 8, lambda r: 100 * 1024 - r % 3 * 17, seed=1)
    save("c1_mini", s.checkpoint()[0], "8 Device regions of 100 KiB - 17*(r%3), synth content seed 1")

    s = ref.RefSession(seed=7, arena_bytes=1 << 20)
    workloads.drive_random(s, seed=42, ops=300, arena=1 << 20)
    save("random_300", s.checkpoint()[0], "drive_random(seed=42, ops=300), seed 7, 1 MiB arena")

    # known-answer CRCs
    manifest["crc_known_answers"] = {"123456789": f"{ref.crc32(b'123456789'):08x}", "": "00000000"}
    (GOLD / "manifest.json").write_text(json.dumps(manifest, indent=1, sort_keys=True) + "\n")
    print(json.dumps({k: v.get("bytes") for k, v in manifest.items() if isinstance(v, dict)}))


if __name__ == "__main__":
    main()
