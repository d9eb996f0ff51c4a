#!/usr/bin/env python
"""Hot straight-line blocks of one kernel in an ncu report: runs of SASS
instructions with equal execution counts, with their share of all executed
instructions and their opcode mix.
usage: ncu_blocks.py <report.ncu-rep> <kernel-regex> [top]"""
import collections, csv, io, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "sass", "--csv", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
ie, isrc, ia = h.index("Instructions Executed"), h.index("Source"), h.index("Address")
seq = []
for r in rows[2:]:
    try:
        seq.append((float(r[ie] or 0), r[isrc].strip(), r[ia]))
    except (ValueError, IndexError):
        pass
tot = sum(e for e, _, _ in seq)
blocks, cur = [], None
for i, (e, s, a) in enumerate(seq):
    if cur and cur["ex"] == e:
        cur["ins"].append(s)
    else:
        cur = {"ex": e, "ins": [s], "start": i, "addr": a}
        blocks.append(cur)
blocks.sort(key=lambda b: -b["ex"] * len(b["ins"]))
for b in blocks[:top]:
    ops = collections.Counter((s.split(None, 1)[1] if s.startswith("@") else s).split()[0].split(".")[0]
                              for s in b["ins"] if s)
    share = 100 * b["ex"] * len(b["ins"]) / tot
    print(f"{share:5.1f}%  #{b['start']:5d} len {len(b['ins']):4d} x {b['ex'] / 1e6:7.2f}M  "
          + " ".join(f"{k}:{v}" for k, v in ops.most_common(8)))
