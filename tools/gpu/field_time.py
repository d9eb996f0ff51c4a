"""cfg2 field (forces) timing: device total_field vs total_potential (CUDA events)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))

import paper_1712_04732_b200 as se
from paper_1712_04732_b200 import device as sedev

rng = np.random.default_rng(2)
N, L = 1_000_000, 10.0
pos = torch.from_numpy(rng.random((N, 3)) * L).cuda()
q = rng.uniform(-1, 1, N)
q = torch.from_numpy(q - q.mean()).cuda()
p = se.SEParams(xi=4.2919, rc=1.0, M=128, P=8, window="bm", shape=20.0, eps=1e-8)
peri = se.Periodicity(3)
E = torch.empty((N, 3), dtype=torch.float64, device="cuda")
phi = torch.empty(N, dtype=torch.float64, device="cuda")


def t(fn, n=5):
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


tf = t(lambda: sedev.total_field(pos, q, L, p, peri, out=E))
tp = t(lambda: sedev.total_potential(pos, q, L, p, peri, out=phi))
print(f"cfg2 field {tf:.3f} ms ({N / tf / 1e3:.1f} M particles/s) | potential {tp:.3f} ms")
