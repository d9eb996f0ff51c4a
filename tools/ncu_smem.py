#!/usr/bin/env python
"""Top shared-memory instructions of one kernel in an ncu report (wavefronts,
excess over ideal) plus the kernel's LSU / fp64 / issue utilisation.
usage: ncu_smem.py <report.ncu-rep> <kernel-regex> [top]"""
import csv, io, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, r = rows[0], rows[2]
want = ["gpu__time_duration.sum", "sm__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.sum.per_cycle_active", "sm__warps_active.avg.per_cycle_active"]
for w in want:
    if w in hdr:
        print(f"{w:90s} {r[hdr.index(w)]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "sass", "--csv", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
c = [h.index(x) for x in ["Instructions Executed", "L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive",
                          "L1 Wavefronts Shared Ideal", "Source"]]
out = []
for q in rows[2:]:
    try:
        ex, wf, exc, ide = (float(q[i] or 0) for i in c[:4])
    except (ValueError, IndexError):
        continue
    if wf > 0:
        out.append((wf, exc, ide, ex, q[c[4]].strip()))
out.sort(reverse=True)
tw = sum(o[0] for o in out)
te = sum(o[1] for o in out)
print(f"shared wavefronts {tw / 1e6:.1f}M  excessive {te / 1e6:.1f}M")
for wf, exc, ide, ex, s in out[:top]:
    print(f"{wf / 1e6:8.1f}M wf {exc / 1e6:7.1f}M exc ideal {ide / 1e6:7.1f} inst {ex / 1e6:7.1f}M  {s}")
