#!/usr/bin/env python
"""Executed-instruction mix (by SASS opcode) of one kernel in an ncu report.
usage: ncu_mix.py <report.ncu-rep> <kernel-regex> [top]"""
import collections, csv, io, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "sass", "--csv", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
ie, isrc = h.index("Instructions Executed"), h.index("Source")
c, tot = collections.Counter(), 0.0
for r in rows[2:]:
    try:
        ex = float(r[ie] or 0)
    except (ValueError, IndexError):
        continue
    s = r[isrc].strip()
    if s.startswith("@"):
        s = s.split(None, 1)[1]
    op = s.split()[0].split(".")[0] if s else "?"
    c[op] += ex
    tot += ex
print(f"total warp instructions {tot / 1e9:.3f}G")
for k, v in c.most_common(top):
    print(f"{k:10s} {v / 1e9:7.3f}G {100 * v / tot:5.1f}%")
