"""k-space pipeline alone (spread, transforms, multipliers, gather) for one workload: for ncu launch lists."""
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

w = workloads.ALL[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]()
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
p = se.SEParams(**w["prm"])
peri = se.Periodicity(w["D"])
dev = torch.device("cuda", 0)
pos = torch.from_numpy(w["pos"]).to(dev)
q = torch.from_numpy(w["q"]).to(dev)
N = len(w["q"])
out = torch.empty(N, dtype=torch.float64, device=dev)
plan = sedev.plan(w["L"], p, peri, dev)
for _ in range(reps):
    _native.call("se_kspace_potential_dev", plan.handle, _native.ptr(pos), _native.ptr(q), N,
                 _native.ptr(out), 1, None)
torch.cuda.synchronize()
print("ok")
