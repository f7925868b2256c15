"""Summarises ncu output into profiles/<round>/ (run here, after gpurun).

    python tools/ncu_summary.py <gpurun_out dir> <profiles/rNN>

* launches.csv (--metrics gpu__time_duration.sum)  -> launch_summary.txt
* prof_<kernel>.ncu-rep (--set full)                -> ncu_<kernel>.txt (+ ncu_full.json)
"""
from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__inst_executed.sum", "lts__t_bytes.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
]


def launch_summary(csv_path: Path) -> str:
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 10 and r[0].isdigit()]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        name = r[4].split("(")[0].replace("<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += float(r[-1])
    tot = sum(v[1] for v in agg.values()) or 1.0
    out = [f"{'kernel':28s} {'launches':>9s} {'total ms':>11s} {'avg us':>11s} {'share':>7s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:28s} {n:9d} {t / 1e6:11.3f} {t / n / 1e3:11.2f} {t / tot:7.1%}")
    return "\n".join(out) + "\n"


def full_summary(rep: Path) -> dict:
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return {}
    head, units = rows[0], rows[1]
    res = {}
    for row in rows[2:]:
        kname = row[head.index("Kernel Name")] if "Kernel Name" in head else rep.stem
        d = {}
        for m in METRICS:
            if m in head:
                d[m] = f"{row[head.index(m)]} {units[head.index(m)]}".strip()
        res[kname.split("(")[0].replace("<unnamed>::", "")] = d
    return res


def main() -> None:
    src, dst = Path(sys.argv[1]), Path(sys.argv[2])
    dst.mkdir(parents=True, exist_ok=True)
    if (src / "launches.csv").exists():
        (dst / "launch_summary.txt").write_text(launch_summary(src / "launches.csv"))
    full = {}
    for rep in sorted(src.glob("prof_*.ncu-rep")):
        s = full_summary(rep)
        full.update(s)
        with open(dst / f"ncu_{rep.stem.removeprefix('prof_')}.txt", "w") as f:
            for k, d in s.items():
                f.write(f"== {k}\n")
                for m, v in d.items():
                    f.write(f"{m:78s} {v}\n")
    if full:
        (dst / "ncu_full.json").write_text(json.dumps(full, indent=1) + "\n")
    print("\n".join(p.name for p in sorted(dst.iterdir())))


if __name__ == "__main__":
    main()
