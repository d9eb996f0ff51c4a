#!/usr/bin/env python
"""Key counters and stall shares of one kernel in an ncu --set full report.
usage: ncu_key.py <report.ncu-rep> [kernel-regex]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
args = ["ncu", "-i", rep, "--page", "raw", "--csv"]
if len(sys.argv) > 2:
    args += ["-k", "regex:" + sys.argv[2]]
rows = list(csv.reader(io.StringIO(subprocess.run(args, capture_output=True, text=True).stdout)))
h, v = rows[0], rows[2]
d = dict(zip(h, v))
keys = ["Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "dram__bytes_read.sum", "dram__bytes_write.sum"]
for k in keys:
    print(f"{k:80s} {d.get(k, '-')[:100]}")
st = {k: float(x) for k, x in d.items() if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio") and x}
tot = sum(st.values())
for k, x in sorted(st.items(), key=lambda t: -t[1])[:10]:
    print(f"  {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):24s} {x:6.3f}  {x / tot:6.1%}")
