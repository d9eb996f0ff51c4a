"""cfg2: device time of the fused total potential vs its parts alone."""
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
import workloads  # noqa: E402

import paper_1712_04732_b200 as se  # noqa: E402
from paper_1712_04732_b200 import _native  # noqa: E402
from paper_1712_04732_b200 import device as sedev  # noqa: E402

w = workloads.ALL[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]()
p = se.SEParams(**w["prm"])
peri = se.Periodicity(w["D"])
dev = torch.device("cuda", 0)
pos = torch.from_numpy(w["pos"]).to(dev)
q = torch.from_numpy(w["q"]).to(dev)
N = len(w["q"])
out = torch.empty(N, dtype=torch.float64, device=dev)
plan = sedev.plan(w["L"], p, peri, dev)


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


tot = timeit(lambda: sedev.total_potential(pos, q, w["L"], p, peri, out=out))
rs = timeit(lambda: _native.call("se_realspace_dev", plan.handle, _native.ptr(pos), _native.ptr(q), N,
                                 _native.ptr(out), 1))
ks = timeit(lambda: _native.call("se_kspace_potential_dev", plan.handle, _native.ptr(pos), _native.ptr(q), N,
                                 _native.ptr(out), 1, None))
print(f"total {tot:.3f} ms | real space alone {rs:.3f} | k-space alone {ks:.3f} | sum {rs + ks:.3f}")
