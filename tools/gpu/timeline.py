"""Kernel timeline (CUPTI via torch.profiler) of one fused total-potential step.

  python tools/gpu/timeline.py cfg2 [out.txt]

Prints every kernel / memset / memcpy of ONE device-resident evaluation after
warm-up (the CUDA-graph replay the bench times): stream, start and end in
microseconds relative to the first activity, duration -- the gaps and the
critical path between the real-space chain and the k-space side stream.
"""

import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import workloads  # noqa: E402

import paper_1712_04732_b200 as se  # noqa: E402
from paper_1712_04732_b200 import device as sedev  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    out = open(sys.argv[2], "w") if len(sys.argv) > 2 else sys.stdout
    w = workloads.ALL[name]()
    dev = torch.device("cuda", 0)
    pos = torch.from_numpy(w["pos"]).to(dev)
    q = torch.from_numpy(w["q"]).to(dev)
    prm = se.SEParams(**w["prm"])
    peri = se.Periodicity(w["D"])
    phi = torch.empty(q.shape[0], dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(4):
        sedev.total_potential(pos, q, w["L"], prm, peri, out=phi)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        flush.zero_()
        torch.cuda.synchronize()
        a.record()
        sedev.total_potential(pos, q, w["L"], prm, peri, out=phi)
        b.record()
        torch.cuda.synchronize()
    kin = prof.profiler.kineto_results.events()
    ev = []
    for e in kin:
        if e.device_type() != torch.autograd.DeviceType.CUDA:
            continue
        nm = e.name()
        if "FillFunctor" in nm or "fill" in nm.lower():
            continue  # the L2 flush
        st = e.start_ns() / 1e3 if hasattr(e, "start_ns") else e.start_us()
        du = e.duration_ns() / 1e3 if hasattr(e, "duration_ns") else e.duration_us()
        ev.append((st, st + du, e.device_resource_id(), nm))
    ev.sort()
    t0 = ev[0][0]
    print(f"# {name}: events {a.elapsed_time(b):.3f} ms; {len(ev)} device activities", file=out)
    print(f"# {'start_us':>10} {'end_us':>10} {'dur_us':>9}  stream  name", file=out)
    for s, t, sid, nm in ev:
        print(f"  {s - t0:10.1f} {t - t0:10.1f} {t - s:9.1f}  {sid:4d}  {nm[:80]}", file=out)


if __name__ == "__main__":
    main()
