"""Summarise an `ncu --set full` report (and optionally a launch-list CSV) into JSON for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--launches gpurun_out/launches.csv] > profiles/x.json
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
    "lts__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        res.append({"kernel": d.get("Kernel Name"), **{k: d.get(k) for k in KEYS if k in d},
                    "units": {k: u for k, u in zip(hdr, units) if k in KEYS}})
    return res


def launches(path):
    per = defaultdict(list)
    with open(path) as f:
        lines = [ln for ln in f if not ln.startswith("==")]
    for d in csv.DictReader(lines):
        if d.get("Metric Name") == "gpu__time_duration.sum":
            per[d["Kernel Name"]].append(float(d["Metric Value"]))
    tot = sum(sum(v) for v in per.values())
    return {k: {"launches": len(v), "total_ns": sum(v), "mean_ns": sum(v) / len(v), "share": sum(v) / tot}
            for k, v in per.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--launches")
    a = ap.parse_args()
    out = {"ncu_full": raw(a.report)}
    if a.launches:
        out["launch_list"] = launches(a.launches)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
