"""RunRecord CSV: the reference's per-evaluation record format (cli.py:23-28,
42-52, 120-134), so that its figure scripts read runs of this package
unchanged.  One row per evaluation with a fixed column set, preceded by a
'#'-prefixed preamble (time, git hash, threads).  The command-line driver
itself is out of scope; this is the data format either side of the path.
"""

from __future__ import annotations

import csv
import datetime
import math
import subprocess

from .core import ParticleSystem, Periodicity, SEParams

CSV_COLUMNS = [
    "command", "sweep_axis", "D", "N", "L", "seed", "window", "xi", "eps",
    "M", "P", "shape", "s0", "s", "s0_eff", "s_eff", "nI", "R", "rc",
    "rms_vs_oracle", "t_spread", "t_aft", "t_scale", "t_aift", "t_gather",
    "t_realspace", "t_precompute", "t_total",
]


def git_hash() -> str:
    try:
        out = subprocess.run(["git", "rev-parse", "--short", "HEAD"], capture_output=True, text=True, timeout=5)
        if out.returncode == 0:
            return out.stdout.strip()
    except Exception:
        pass
    return "unknown"


def make_record(system: ParticleSystem, params: SEParams, periodicity: Periodicity, timings: dict,
                t_total: float, command: str = "compute", sweep_axis: str = "", seed=0,
                rms_vs_oracle: float = math.nan) -> dict:
    """One RunRecord (cli.py:120-134); s0_eff / s_eff from the built grid."""
    from .sekspace import Grid

    g = Grid.build(system.L, params, periodicity)
    D = periodicity.D
    return {
        "command": command, "sweep_axis": sweep_axis, "D": D, "N": system.N,
        "L": system.L, "seed": seed, "window": params.window, "xi": params.xi,
        "eps": params.eps, "M": params.M, "P": params.P, "shape": params.shape,
        "s0": params.s0, "s": params.s,
        "s0_eff": g.g0 / g.Mt if D < 3 else 1.0,
        "s_eff": g.gs / g.Mt if D in (1, 2) else 1.0,
        "nI": params.nI, "R": params.R, "rc": params.rc, "rms_vs_oracle": rms_vs_oracle,
        "t_spread": timings.get("spread", 0.0), "t_aft": timings.get("aft", 0.0),
        "t_scale": timings.get("scale", 0.0), "t_aift": timings.get("aift", 0.0),
        "t_gather": timings.get("gather", 0.0), "t_realspace": timings.get("realspace", 0.0),
        "t_precompute": timings.get("precompute", 0.0), "t_total": t_total,
    }


def write_records(stream, records: list[dict], threads: int = 1) -> None:
    """Preamble + header + rows (cli.py:42-52); every column must be present."""
    stream.write(f"# pmewald run {datetime.datetime.now().isoformat()}\n")
    stream.write(f"# git {git_hash()}\n")
    stream.write(f"# threads {threads}\n")
    writer = csv.DictWriter(stream, fieldnames=CSV_COLUMNS)
    writer.writeheader()
    for rec in records:
        missing = set(CSV_COLUMNS) - set(rec)
        if missing:
            raise RuntimeError(f"record missing columns: {sorted(missing)}")
        writer.writerow(rec)


def read_records(stream) -> list[dict]:
    """Rows of a RunRecord CSV ('#' preamble skipped), values as strings."""
    return list(csv.DictReader(line for line in stream if not line.startswith("#")))
