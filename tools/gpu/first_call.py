"""Plan creation and first-call latency: for each
workload, wall time of se_plan_create, of the FIRST total-potential call
(tables, BM quadrature, the D = 0 truncated-kernel table -- the reference's
precompute_truncated_greens, 12-14 s on the CPU at cfg5 --, cuFFT plans,
binning buffers), of the second call (CUDA-graph capture) and the steady
state; device-resident inputs, synchronised timings.

  python tools/gpu/first_call.py out.json cfg2 cfg5 cfg3_tol cfg4
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tools")]


def main():
    import torch

    import workloads
    import paper_1712_04732_b200 as se
    from paper_1712_04732_b200 import _native
    from paper_1712_04732_b200 import device as sedev

    out, names = sys.argv[1], sys.argv[2:]
    dev = torch.device("cuda", 0)
    torch.cuda.init()
    res = {}
    for name in names:
        w = workloads.ALL[name]()
        prm = se.SEParams(**w["prm"])
        peri = se.Periodicity(w["D"])
        pos = torch.from_numpy(w["pos"]).to(dev)
        q = torch.from_numpy(w["q"]).to(dev)
        phi = torch.empty(q.shape[0], dtype=torch.float64, device=dev)
        _native.clear_plans()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pl = sedev.plan(w["L"], prm, peri, dev)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        sedev.total_potential(pos, q, w["L"], prm, peri, out=phi)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        sedev.total_potential(pos, q, w["L"], prm, peri, out=phi)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        steady = []
        for _ in range(5):
            a = time.perf_counter()
            sedev.total_potential(pos, q, w["L"], prm, peri, out=phi)
            torch.cuda.synchronize()
            steady.append(time.perf_counter() - a)
        res[name] = {"plan_create_ms": 1e3 * (t1 - t0), "first_call_ms": 1e3 * (t2 - t1),
                     "second_call_ms": 1e3 * (t3 - t2), "steady_ms": 1e3 * min(steady), "N": int(q.shape[0]),
                     "D": w["D"]}
        if w["D"] == 0:
            nconv, g0, R = (_native.ctypes.c_int32(), _native.ctypes.c_int32(), _native.ctypes.c_double())
            _native.call("se_plan_d0_geometry", pl.handle, _native.ctypes.byref(nconv), _native.ctypes.byref(g0),
                         _native.ctypes.byref(R))
            res[name].update(nconv=nconv.value, g0=g0.value)
        print(name, json.dumps(res[name]), flush=True)
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
