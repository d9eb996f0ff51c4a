"""Host/device time per phase of distributed.total_potential_domain (one
rank, NCCL process group of size 1), cfg2, synchronised between phases."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tools")]

import torch
import torch.distributed as dist

import workloads
import paper_1712_04732_b200 as se
from paper_1712_04732_b200 import distributed as dd

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
w = workloads.ALL[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]()
prm = se.SEParams(**w["prm"])
peri = se.Periodicity(w["D"])
pos = torch.from_numpy(w["pos"]).to(dev)
q = torch.from_numpy(w["q"]).to(dev)
be = dd.NativeBackend(w["L"], prm, peri, dev)

# instrument: wrap the backend's and the module's heavy calls with synced timers
T = {}


def timed(name, fn):
    def inner(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        T[name] = T.get(name, 0.0) + time.perf_counter() - t0
        return r
    return inner


for n in ("realspace_domain", "spread_all", "kspace_apply", "gather_all", "check_system", "finish"):
    setattr(be, n, timed(n, getattr(be, n)))
dd._all_to_allv = timed("all_to_allv", dd._all_to_allv)
dd._slab_kspace_domain = timed("slab_kspace", dd._slab_kspace_domain)
for _ in range(3):
    dd.total_potential_domain(pos, q, be)
torch.cuda.synchronize()
T.clear()
reps = 5
t0 = time.perf_counter()
for _ in range(reps):
    dd.total_potential_domain(pos, q, be)
torch.cuda.synchronize()
tot = (time.perf_counter() - t0) / reps
print(f"total {1e3 * tot:.2f} ms per call (synchronised phases, so no overlap)")
for k, v in sorted(T.items(), key=lambda x: -x[1]):
    print(f"  {k:18s} {1e3 * v / reps:8.3f} ms")
print(f"  {'other (python)':18s} {1e3 * (tot - sum(T.values()) / reps):8.3f} ms")
dist.destroy_process_group()
