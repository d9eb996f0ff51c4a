"""Where the end-to-end time of the public API goes at cfg2: the device-
resident pipeline, the C-ABI host entry (H2D + pipeline + D2H), the Python
API on top, and the raw pinned copies of the same bytes.
  python tools/gpu/e2e_breakdown.py"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tools")]


def main():
    import numpy as np
    import torch

    import workloads
    import paper_1712_04732_b200 as se
    from paper_1712_04732_b200 import _native
    from paper_1712_04732_b200 import device as sedev

    w = workloads.ALL["cfg2"]()
    dev = torch.device("cuda", 0)
    prm = se.SEParams(**w["prm"])
    peri = se.Periodicity(w["D"])
    N, L = w["q"].shape[0], w["L"]
    pos_p = torch.from_numpy(w["pos"]).pin_memory()
    q_p = torch.from_numpy(w["q"]).pin_memory()
    pos_d, q_d = pos_p.to(dev), q_p.to(dev)
    phi_d = torch.empty(N, dtype=torch.float64, device=dev)
    out = {}

    def timeit(fn, n=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(n):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return 1e3 * statistics.median(ts)

    out["device_pipeline_ms"] = timeit(lambda: sedev.total_potential(pos_d, q_d, L, prm, peri, out=phi_d))
    pl = _native.plan_for(peri.D, L, prm)
    phi_h = _native.host_out(N)
    out["c_abi_host_ms"] = timeit(lambda: _native.call("se_total_potential_host", pl.handle, _native.ptr(pos_p.numpy()),
                                                         _native.ptr(q_p.numpy()), N, _native.ptr(phi_h), None))
    system = se.ParticleSystem(pos_p.numpy(), q_p.numpy(), L)
    out["python_api_ms"] = timeit(lambda: se.total_potential(system, prm, peri))
    buf = torch.empty(4 * N, dtype=torch.float64, device=dev)
    out["h2d_32MB_ms"] = timeit(lambda: (buf[:3 * N].copy_(pos_p.view(-1), non_blocking=True),
                                         buf[3 * N:].copy_(q_p, non_blocking=True)))
    out["d2h_8MB_ms"] = timeit(lambda: torch.from_numpy(phi_h).copy_(phi_d, non_blocking=True))
    print(out)


if __name__ == "__main__":
    main()
