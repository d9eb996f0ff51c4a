#!/usr/bin/env python
"""profiles/ncu_<round>_summary.json from ncu --set full captures of the hot
kernels (tools/gpu/round.sh -> gpurun_out/<tag>/{realspace,spread,gather}.ncu-rep).

Each entry records the kernel signature, the counters the bench's roofline
object quotes (DRAM bytes, fp64-pipe and issue utilisation, instructions)
and the hash of the kernel's source files at capture time; bench.py attaches
the real-space entry to its roofline only when that hash matches the
current sources (a profile of another build is never quoted).

  python tools/profile_summary.py <tag> <round> [workload]
"""

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SOURCES = {
    "realspace": ("paper_1712_04732_b200/csrc/se_realspace.cu", "paper_1712_04732_b200/csrc/se_erfc_coeffs.h",
                  "paper_1712_04732_b200/csrc/se_common.h", "paper_1712_04732_b200/csrc/se_host.cpp"),
    "spread": ("paper_1712_04732_b200/csrc/se_spread.cu", "paper_1712_04732_b200/csrc/se_common.h"),
    "gather": ("paper_1712_04732_b200/csrc/se_spread.cu", "paper_1712_04732_b200/csrc/se_common.h"),
}


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def num(d, k):
    try:
        return float(d[k].replace(",", ""))
    except Exception:
        return None


def scale(v, unit):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
         "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(unit, 1.0)
    return None if v is None else v * f


def main():
    from bench import _source_hash

    tag, rnd = sys.argv[1], sys.argv[2]
    workload = sys.argv[3] if len(sys.argv) > 3 else "cfg2"
    res = {"source": f"ncu --set full --import-source on --clock-control none, tools/gpu/profile_step.py "
                     f"{workload} <stage> (gpurun_out/{tag})", "workload": workload}
    for st, files in SOURCES.items():
        p = os.path.join(ROOT, "gpurun_out", tag, f"{st}.ncu-rep")
        if not os.path.exists(p):
            continue
        d, u = raw(p)[0]
        rd = scale(num(d, "dram__bytes_read.sum"), u.get("dram__bytes_read.sum"))
        wr = scale(num(d, "dram__bytes_write.sum"), u.get("dram__bytes_write.sum"))
        res[st] = {
            "kernel": d.get("Kernel Name", "")[:120],
            "workload": workload,
            "duration_ms": scale(num(d, "gpu__time_duration.sum"), u.get("gpu__time_duration.sum")),
            "dram_bytes": (rd or 0) + (wr or 0),
            "fp64_pipe_pct": num(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": num(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            "smem_wavefronts_pct": num(d, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
            "inst_executed": num(d, "smsp__inst_executed.sum"),
            "registers": num(d, "launch__registers_per_thread"),
            "source_hash": _source_hash(files),
            "source": f"gpurun_out/{tag}/{st}.ncu-rep",
        }
    out = os.path.join(ROOT, "profiles", f"ncu_{rnd}_summary.json")
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
