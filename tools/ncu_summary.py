#!/usr/bin/env python3
"""Summarise an .ncu-rep: key SOL/occupancy/divergence metrics + stall breakdown (for profiles/)."""
import csv
import io
import subprocess
import sys

KEEP = ['Duration', 'DRAM Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate', 'Compute (SM) Throughput',
        'Executed Ipc Active', 'Issue Slots Busy', 'Avg. Active Threads Per Warp', 'Achieved Occupancy',
        'Registers Per Thread', 'Warp Cycles Per Issued Instruction', 'Eligible Warps Per Scheduler',
        'Executed Instructions', 'Branch Efficiency', 'Theoretical Occupancy', 'Memory Throughput']


def run(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    res = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") in KEEP:
            res[d["Metric Name"]] = f"{d['Metric Value']} {d['Metric Unit']}".strip()
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hh, vals = rr[0], rr[2]
    for i, n in enumerate(hh):
        if n in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors.sum", "gpu__time_duration.sum",
                 "launch__grid_size", "launch__registers_per_thread"):
            res[n] = f"{vals[i]} {rr[1][i]}"
    st = {n.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(vals[i] or 0) for i, n in enumerate(hh)
          if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")}
    tot = sum(st.values()) or 1
    res["stalls"] = {k: round(v / tot, 3) for k, v in sorted(st.items(), key=lambda x: -x[1]) if v / tot > 0.01}
    return res


if __name__ == "__main__":
    import json
    for rep in sys.argv[1:]:
        print(rep)
        print(json.dumps(run(rep), indent=1))
