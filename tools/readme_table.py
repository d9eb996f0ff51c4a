#!/usr/bin/env python
"""The README's results table from the committed bench lines
(profiles/bench_r02_cfg2.json, profiles/r02_configs/).  python tools/readme_table.py"""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")


def line(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


def fmt(v):
    return f"{v / 1e6:.1f} M"


rows = [("cfg2", line(os.path.join(P, "bench_r02_cfg2.json")))]
for n in ("cfg2_tol", "cfg1", "cfg1_tol", "cfg3", "cfg3_tol", "cfg4", "cfg4_tol", "cfg5"):
    rows.append((n, line(os.path.join(P, "r02_configs", f"bench_{n}.json"))))
print("| config | N | particles/s (device) | e2e (public API, host buffers) | ms per step |")
print("|---|---|---|---|---|")
for n, d in rows:
    print(f"| {d['config']['workload']} | {d['config']['N']:.0e} | {fmt(d['value'])} | {fmt(d['e2e']['value'])} | "
          f"{d['ms_per_step']:.3f} |")
