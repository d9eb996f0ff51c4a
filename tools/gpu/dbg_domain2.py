import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1712_04732_b200 as se
from paper_1712_04732_b200 import device as sedev, _native
from paper_1712_04732_b200.distributed import NativeBackend, total_potential_domain
import paper_1712_04732_b200.distributed as dd
D = int(sys.argv[1])
rng = np.random.default_rng(21)
N, L = 40000, 4.0
pos = rng.random((N, 3)) * L
q = rng.uniform(-1, 1, N); q -= q.mean()
prm = se.SEParams(xi=6.0, rc=0.4, M=32, P=8, window="bm", shape=20.0, s0=4.0, R=3.5)
peri = se.Periodicity(D)
dev = torch.device("cuda", 0)
pd = torch.from_numpy(pos).to(dev); qd = torch.from_numpy(q).to(dev)
ref = sedev.total_potential(pd, qd, L, prm, peri).cpu().numpy()
refk = sedev.kspace_potential(pd, qd, L, prm, peri).cpu().numpy()
refr = ref - refk
bad = 0
for trial in range(8):
    be = NativeBackend(L, prm, peri, dev)
    # instrument: capture the pieces
    phi = total_potential_domain(pd, qd, be).cpu().numpy()
    e = se.relative_rms_error(phi, ref)
    if e > 1e-12:
        bad += 1
        print(trial, "total", e, flush=True)
        # which part: re-run real space alone on the same backend
        part = be.domain_partition(1, N)
        out = be.empty_phi(N)
        be.realspace_domain(pd, qd, N, part, 0, out); torch.cuda.synchronize(); be.finish()
        print("   realspace again", se.relative_rms_error(out.cpu().numpy(), refr), flush=True)
        print("   diff vs refk", se.relative_rms_error(phi - refr, refk), " vs refr", se.relative_rms_error(phi - refk, refr))
print("bad", bad, "of 8")
