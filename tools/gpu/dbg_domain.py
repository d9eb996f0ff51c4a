import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1712_04732_b200 as se
from paper_1712_04732_b200 import device as sedev
from paper_1712_04732_b200.distributed import NativeBackend, total_potential_domain
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
for trial in range(3):
    be = NativeBackend(L, prm, peri, dev)
    phi = total_potential_domain(pd, qd, be).cpu().numpy()
    print(trial, "total", se.relative_rms_error(phi, ref), flush=True)
    # k-space part through the backend calls alone
    grid = be.empty_grid(); phik = be.empty_phi(N)
    be.spread_all(pd, qd, grid); be.kspace_apply(grid); be.gather_all(grid, pd, phik)
    torch.cuda.synchronize()
    print(trial, "kspace", se.relative_rms_error(phik.cpu().numpy(), refk), flush=True)
