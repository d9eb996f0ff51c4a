"""Per-rank device time of the sharded pipeline at world W, one rank's work
alone on one GPU (no collectives: the grid and phi exchanges are replaced by
nothing), to estimate the N-GPU step: python shard_time.py [cfg] [W]."""
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.join(HERE, ".."), os.path.join(HERE, "..", "..")]
import workloads  # noqa: E402

import paper_1712_04732_b200 as se  # noqa: E402
from paper_1712_04732_b200.distributed import NativeBackend  # noqa: E402

w = workloads.ALL[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]()
W = int(sys.argv[2]) if len(sys.argv) > 2 else 8
p = se.SEParams(**w["prm"])
dev = torch.device("cuda", 0)
pos = torch.from_numpy(w["pos"]).to(dev)
q = torch.from_numpy(w["q"]).to(dev)
N = len(w["q"])
be = NativeBackend(w["L"], p, se.Periodicity(w["D"]), dev)
grid, phi, phik = be.empty_grid(), be.empty_phi(N), be.empty_phi(N)
cur, ks = torch.cuda.current_stream(), be.kstream


def step(rank):
    ks.wait_stream(cur)
    with torch.cuda.stream(ks):
        be.spread_shard(pos, q, rank, W, grid)
    be.realspace_shard(pos, q, rank, W, phi)
    with torch.cuda.stream(ks):
        be.kspace_apply(grid)
        be.gather_shard(grid, pos, rank, W, phik, accumulate=False)
    cur.wait_stream(ks)
    phi.add_(phik)
    be.finish()


def timed(fn, n=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


full = timed(lambda: step(0) if W == 1 else None) if W == 1 else None
r0 = timed(lambda: step(0))
rl = timed(lambda: step(W - 1))
rs = timed(lambda: be.realspace_shard(pos, q, 0, W, phi) or be.finish())
print(f"world {W}: rank 0 {r0:.3f} ms, rank {W - 1} {rl:.3f} ms (real-space shard alone {rs:.3f} ms)")

# per-stage spans of the real-space plan (binning vs kernel + finish)
be.plan.set_profiling(True)
be.plan.kernel_times()
for _ in range(5):
    be.realspace_shard(pos, q, 0, W, phi)
    be.finish()
kt = be.plan.kernel_times()
be.plan.set_profiling(False)
print("  real-space plan spans (ms/call):", {k: round(v[0] / max(1, v[1]), 3) for k, v in kt.items() if v[1]})
