#!/usr/bin/env python
"""Summarise a gpurun profiling session into profiles/.

  python tools/ncu_summary.py gpurun_out/<tag> profiles/<round>_<name>

reads <dir>/launches.csv (ncu --metrics gpu__time_duration.sum list),
<dir>/prof.ncu-rep (ncu --set full capture) and <dir>/bench.json, and writes
<prefix>_launches.txt (per-kernel launch count / mean / share), <prefix>_ncu.txt
(key metrics of the first captured launch + the hottest SASS lines) and
<prefix>_bench.json (the bench line). Needs the ncu CLI (present in this image).
"""
from __future__ import annotations

import collections
import csv
import io
import json
import shutil
import subprocess
import sys
from pathlib import Path

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__t_bytes.sum", "l1tex__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__average_warp_latency_per_inst_issued.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
]


def launches(path: Path) -> str:
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) > vi:
            agg.setdefault(r[ki].split("(")[0], []).append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = ["kernel launches (ncu gpu__time_duration.sum, cold-cache, serialised)",
           f"{'count':>6} {'mean_us':>9} {'share':>6}  kernel"]
    for k, v in agg.items():
        out.append(f"{len(v):6d} {sum(v) / len(v) / 1e3:9.2f} {sum(v) / tot:6.1%}  {k}")
    return "\n".join(out) + "\n"


def ncu_raw(rep: Path) -> str:
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hdr, unit = r[0], r[1]
    out = []
    for row in r[2:]:
        name = row[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        out.append(f"== {name[:100]}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                out.append(f"  {k:80s} {row[i]:>14s} {unit[i]}")
        try:
            rd = float(row[hdr.index("dram__bytes_read.sum")].replace(",", ""))
            wr = float(row[hdr.index("dram__bytes_write.sum")].replace(",", ""))
            ur = unit[hdr.index("dram__bytes_read.sum")]
            uw = unit[hdr.index("dram__bytes_write.sum")]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            out.append(f"  traffic_bytes(read+write) {rd * scale.get(ur, 1) + wr * scale.get(uw, 1):.0f}")
        except (ValueError, KeyError):
            pass
    return "\n".join(out) + "\n"


def ncu_source(rep: Path, top: int = 40) -> str:
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "source", "--csv", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hdr = r[1]
    rows = []
    for x in r[2:]:
        if x and x[0] == "Kernel Name":
            break
        if len(x) > 10 and x[0].startswith("0x"):
            rows.append(x)
    ia = hdr.index("Instructions Executed")
    sa = hdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(x[ia]) for x in rows)
    st = sum(int(x[sa]) for x in rows) or 1
    hot = sorted(rows, key=lambda x: -int(x[sa]))[:top]
    out = [f"first launch: {len(rows)} SASS lines, {tot} warp-instructions executed, "
           f"{st} stall samples", "top stall-sampled instructions (samples, share, executed):"]
    for x in hot:
        out.append(f"  {int(x[sa]):6d} {int(x[sa]) / st:6.1%} {int(x[ia]):9d}  {x[1].strip()[:90]}")
    return "\n".join(out) + "\n"


def main():
    src, prefix = Path(sys.argv[1]), sys.argv[2]
    Path(prefix).parent.mkdir(parents=True, exist_ok=True)
    if (src / "launches.csv").exists():
        Path(prefix + "_launches.txt").write_text(launches(src / "launches.csv"))
    if (src / "prof.ncu-rep").exists():
        Path(prefix + "_ncu.txt").write_text(ncu_raw(src / "prof.ncu-rep") +
                                             ncu_source(src / "prof.ncu-rep"))
    if (src / "bench.json").exists():
        lines = [l for l in (src / "bench.json").read_text().splitlines() if l.startswith("{")]
        if lines:
            Path(prefix + "_bench.json").write_text(json.dumps(json.loads(lines[0]), indent=1) + "\n")
    for extra in ("pytest_gpu.log",):
        if (src / extra).exists():
            shutil.copy(src / extra, prefix + "_" + extra)


if __name__ == "__main__":
    main()
