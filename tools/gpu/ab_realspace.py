"""A/B timing of the real-space kernel on BASELINE workloads (one process
per library setting, e.g. SE_B200_DENSE_MIN): CUDA-event time per launch
of the real-space kernel (plan profiling slots) over `reps` calls after a
warm-up, and phi_R saved for cross-setting comparison.

  SE_B200_DENSE_MIN=410 python tools/gpu/ab_realspace.py out.json cfg2 cfg5
  python tools/gpu/ab_realspace.py --compare a.json b.json
"""

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def run(out, names, reps=10):
    import torch

    import workloads
    import paper_1712_04732_b200 as se
    from paper_1712_04732_b200 import _native
    from paper_1712_04732_b200 import device as sedev

    dev = torch.device("cuda", 0)
    res = {"env": {k: v for k, v in os.environ.items() if k.startswith("SE_B200")}}
    for name in names:
        w = workloads.ALL[name]()
        pos = torch.from_numpy(w["pos"]).to(dev)
        q = torch.from_numpy(w["q"]).to(dev)
        prm = se.SEParams(**w["prm"])
        peri = se.Periodicity(w["D"])
        N = q.shape[0]
        pl = sedev.plan(w["L"], prm, peri, dev)
        phi = torch.empty(N, dtype=torch.float64, device=dev)
        for _ in range(2):
            _native.call("se_realspace_dev", pl.handle, _native.ptr(pos), _native.ptr(q), N, _native.ptr(phi), 1)
        torch.cuda.synchronize()
        pl.set_profiling(True)
        pl.kernel_times()
        for _ in range(reps):
            _native.call("se_realspace_dev", pl.handle, _native.ptr(pos), _native.ptr(q), N, _native.ptr(phi), 1)
        torch.cuda.synchronize()
        kt = pl.kernel_times()
        pl.set_profiling(False)
        ms, n = kt["realspace"]
        path = f"{out}.{name}.npy"
        np.save(path, phi.cpu().numpy())
        res[name] = {"realspace_ms": ms / max(n, 1), "sort_ms": kt["sort"][0] / max(kt["sort"][1], 1), "phi": path}
        print(name, json.dumps(res[name]), flush=True)
    json.dump(res, open(out, "w"), indent=1)


def compare(a, b):
    A, B = json.load(open(a)), json.load(open(b))
    for k in A:
        if k == "env" or k not in B:
            continue
        pa, pb = np.load(A[k]["phi"]), np.load(B[k]["phi"])
        rel = float(np.sqrt(np.mean((pa - pb) ** 2) / np.mean(pb ** 2)))
        print(f"{k}: {A[k]['realspace_ms']:.3f} ms ({A['env']}) vs {B[k]['realspace_ms']:.3f} ms ({B['env']}); "
              f"ratio {A[k]['realspace_ms'] / B[k]['realspace_ms']:.3f}; phi_R rel rms {rel:.2e}")


if __name__ == "__main__":
    if sys.argv[1] == "--compare":
        compare(sys.argv[2], sys.argv[3])
    else:
        run(sys.argv[1], sys.argv[2:])
