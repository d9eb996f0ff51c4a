"""One profiled total-potential step of a BASELINE workload for ncu.

  ncu --profile-from-start off ... python tools/gpu/profile_step.py cfg2 [stage]

Warm-up evaluations (tables, cuFFT plans, CUDA graph) run outside the
profiler range; exactly one device-resident evaluation of the workload --
or, with stage = spread | gather | kspace | realspace, one call of that stage --
runs between cudaProfilerStart / cudaProfilerStop, so the ncu launch list
and --set full captures are of the same build and inputs the bench times.
"""

import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import workloads  # noqa: E402

import paper_1712_04732_b200 as se  # noqa: E402
from paper_1712_04732_b200 import _native  # noqa: E402
from paper_1712_04732_b200 import device as sedev  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    stage = sys.argv[2] if len(sys.argv) > 2 else "total"
    w = workloads.ALL[name]()
    dev = torch.device("cuda", 0)
    pos = torch.from_numpy(w["pos"]).to(dev)
    q = torch.from_numpy(w["q"]).to(dev)
    prm = se.SEParams(**w["prm"])
    peri = se.Periodicity(w["D"])
    L = w["L"]
    N = q.shape[0]
    pl = sedev.plan(L, prm, peri, dev)
    g = pl.grid()
    grid = torch.empty(tuple(g.shape), dtype=torch.float64, device=dev)
    phi = torch.empty(N, dtype=torch.float64, device=dev)

    def run():
        if stage == "total":
            sedev.total_potential(pos, q, L, prm, peri, out=phi)
        elif stage == "spread":
            _native.call("se_spread_dev", pl.handle, _native.ptr(pos), _native.ptr(q), N, _native.ptr(grid))
        elif stage == "gather":
            _native.call("se_gather_dev", pl.handle, _native.ptr(grid), _native.ptr(pos), N, _native.ptr(phi), 0)
        elif stage == "kspace":
            _native.call("se_kspace_apply_dev", pl.handle, _native.ptr(grid), 1, None)
        elif stage == "realspace":
            _native.call("se_realspace_dev", pl.handle, _native.ptr(pos), _native.ptr(q), N, _native.ptr(phi), 1)
        else:
            raise SystemExit(f"unknown stage {stage}")

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    run()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print(f"profiled one {stage} of {name} (N={N})")


if __name__ == "__main__":
    main()
