"""Summarise ncu captures for profiles/ (runs in the build container, no GPU needed).

    python tools/ncu_summary.py launches <launches.csv> <out.md>
    python tools/ncu_summary.py full <report.ncu-rep> <out.json> [kernel-regex]

`launches`: per-kernel share of the device time in an `ncu --metrics gpu__time_duration.sum`
launch list (cold-cache, serialised: compare shares, not absolutes).
`full`: the metrics of one `--set full` capture that the roofline needs (DRAM bytes per
launch, FP64-pipe and issue utilisation, occupancy, stall reasons).
"""

from __future__ import annotations

import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict


def launches(path: str, out: str) -> None:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            d[r[ki]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    lines = ["| share | launches | avg (us) | kernel |", "|---:|---:|---:|---|"]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {100 * sum(v) / tot:.2f}% | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | `{k[:90]}` |")
    with open(out, "w") as f:
        f.write(f"Launch list from `{path}` (ncu gpu__time_duration.sum, --clock-control none)\n\n")
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__waves_per_multiprocessor",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
]


def _to_bytes(val: float, unit: str) -> float:
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return val * scale


def full(path: str, out: str, kregex: str | None = None) -> None:
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        if kregex and not re.search(kregex, name):
            continue
        rec = {"kernel": name}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                try:
                    rec[k] = float(r[i].replace(",", ""))
                except ValueError:
                    rec[k] = r[i]
                rec[k + ".unit"] = units[i]
        recs.append(rec)
    for rec in recs:
        rd = _to_bytes(rec.get("dram__bytes_read.sum", 0.0), rec.get("dram__bytes_read.sum.unit", "byte"))
        wr = _to_bytes(rec.get("dram__bytes_write.sum", 0.0), rec.get("dram__bytes_write.sum.unit", "byte"))
        rec["dram_bytes_per_launch"] = rd + wr
    summary = {"source": path, "launches": recs,
               "dram_bytes_per_launch": sum(r["dram_bytes_per_launch"] for r in recs) / max(1, len(recs))}
    with open(out, "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1)[:3000])


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
