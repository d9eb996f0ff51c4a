"""A/B timing of spreading and gathering alone (stage entry points, plan
profiling events) on BASELINE workloads; SE_B200_LIB selects the library.
  python tools/gpu/ab_sg.py cfg2 cfg5 cfg4"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tools")]


def main():
    import torch

    import workloads
    import paper_1712_04732_b200 as se
    from paper_1712_04732_b200 import _native
    from paper_1712_04732_b200 import device as sedev
    dev = torch.device("cuda", 0)
    for name in sys.argv[1:]:
        w = workloads.ALL[name]()
        pos = torch.from_numpy(w["pos"]).to(dev)
        q = torch.from_numpy(w["q"]).to(dev)
        prm = se.SEParams(**w["prm"])
        pl = sedev.plan(w["L"], prm, se.Periodicity(w["D"]), dev)
        g = pl.grid()
        grid = torch.empty(tuple(g.shape), dtype=torch.float64, device=dev)
        phi = torch.empty(q.shape[0], dtype=torch.float64, device=dev)
        N = q.shape[0]
        for rep in range(2):
            pl.set_profiling(True)
            pl.kernel_times()
            for _ in range(10):
                _native.call("se_spread_dev", pl.handle, _native.ptr(pos), _native.ptr(q), N, _native.ptr(grid))
                _native.call("se_gather_dev", pl.handle, _native.ptr(grid), _native.ptr(pos), N, _native.ptr(phi), 0)
            torch.cuda.synchronize()
            kt = pl.kernel_times()
        out = {k: kt[k][0] / max(kt[k][1], 1) for k in ("spread", "gather", "sort")}
        print(name, os.environ.get("SE_B200_LIB", "current"), json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
