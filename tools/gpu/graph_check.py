"""Time repeated device-API calls with and without CUDA-graph replay."""
import os
import sys
import time

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
import workloads  # noqa: E402

import paper_1712_04732_b200 as se  # noqa: E402
from paper_1712_04732_b200 import device as sedev  # noqa: E402

for name in sys.argv[1:] or ["cfg1"]:
    w = workloads.ALL[name]()
    p = se.SEParams(**w["prm"])
    peri = se.Periodicity(w["D"])
    dev = torch.device("cuda", 0)
    pos = torch.from_numpy(w["pos"]).to(dev)
    q = torch.from_numpy(w["q"]).to(dev)
    out = torch.empty(len(w["q"]), dtype=torch.float64, device=dev)
    plan = sedev.plan(w["L"], p, peri, dev)
    ref = None
    for on in (False, True, False, True):
        plan.set_graphs(on)
        for _ in range(3):
            sedev.total_potential(pos, q, w["L"], p, peri, out=out)
        torch.cuda.synchronize()
        n = 50 if len(w["q"]) < 1e5 else 10
        t0 = time.perf_counter()
        for _ in range(n):
            sedev.total_potential(pos, q, w["L"], p, peri, out=out)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / n
        if ref is None:
            ref = out.clone()
        err = float((out - ref).abs().max() / ref.abs().max())
        print(f"{name} graphs={on}: {1e3 * dt:.4f} ms per call, max rel diff vs first {err:.2e}")
