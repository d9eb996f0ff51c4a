#!/usr/bin/env python
"""Per-source-line instruction / stall shares of one kernel: joins the SASS
page of an ncu report (ncu --page source --print-source sass --csv) with the
line table of the cubin (nvdisasm -g).
usage: ncu_lines.py <sass.csv> <nvdisasm.txt> <kernel-substring> <source.cu>"""
import collections, csv, re, sys

sass_csv, dis, kname, srcf = sys.argv[1:5]
lines = open(dis).read().split("\n")
start = [i for i, l in enumerate(lines) if l.startswith("//---------------------") and kname in l][0]
addr2line, cur, curfile = {}, None, None
for l in lines[start + 1:]:
    if l.startswith("//---------------------"):
        break
    m = re.search(r'## File "(.*)", line (\d+)', l)
    if m:
        cur, curfile = int(m.group(2)), m.group(1).split("/")[-1]
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m:
        addr2line[int(m.group(1), 16)] = (curfile, cur)
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
i_a, i_ex = hdr.index("Address"), hdr.index("Instructions Executed")
i_st = hdr.index("Warp Stall Sampling (All Samples)")
base = None
cnt, stc = collections.Counter(), collections.Counter()
tot = stt = 0.0
for r in rows[2:]:
    if len(r) <= i_ex:
        continue
    try:
        a = int(r[i_a], 16)
    except ValueError:
        continue
    base = a if base is None else base
    ex, st = float(r[i_ex] or 0), float(r[i_st] or 0)
    tot += ex
    stt += st
    key = addr2line.get(a - base, ("?", None))
    cnt[key] += ex
    stc[key] += st
src = open(srcf).read().split("\n")
for (f, ln), v in cnt.most_common(40):
    s = src[ln - 1].strip()[:90] if ln and f == srcf.split("/")[-1] else ""
    print(f"{100 * v / tot:5.1f}% stall {100 * stc[(f, ln)] / max(stt, 1):5.1f}%  {f}:{ln}  {s}")
