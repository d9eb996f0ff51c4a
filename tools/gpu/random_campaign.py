"""Randomized parity campaign: many seeded configurations of the full device
pipeline against the CPU oracle (the test suite runs 24 of them)."""
import math
import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import se_oracle as orc  # noqa: E402

import paper_1712_04732_b200 as se  # noqa: E402
from paper_1712_04732_b200 import windows  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
worst, fails = 0.0, []
for case in range(n_cases):
    rng = np.random.default_rng(50000 + case)
    D = int(rng.integers(0, 4))
    window = ["bm", "gaussian", "kb"][int(rng.integers(0, 3))]
    Ps = [4, 6, 8, 10, 12, 14, 16, 18, 20, 24] if D in (1, 2) else [2, 3, 4, 5, 6, 7, 8, 9, 10, 12, 15, 17, 20, 25]
    P = int(rng.choice(Ps))
    M = max(int(rng.choice([8, 12, 16, 18, 20, 24, 28, 32])), P + P % 2)
    L = float(rng.choice([0.5, 0.7, 1.0, 2.3, 4.0]))
    N = int(rng.integers(2, 800))
    xi = float(rng.uniform(3.0, 10.0)) / L
    eps = float(rng.choice([1e-6, 1e-10, 1e-13]))
    rc = math.sqrt(-math.log(eps)) / xi
    h = L / M
    d = 3.0 - D
    if D < 3:
        s0 = max(1.0 + math.sqrt(d), ((1.0 + math.sqrt(d)) * L + 2.0 * rc) / (L + P * h))
        R = 0.5 * (se.aft.padded_size(s0, M + P) * h - L + math.sqrt(d) * L)
    else:
        s0, R = 1.0, 0.0
    s_up = max(1.0, math.log(1.0 / eps) / (2 * math.pi)) if D in (1, 2) else 1.0
    nI = int(rng.integers(0, M // 2 + 1)) if D in (1, 2) else 0
    prm = se.SEParams(xi=xi, rc=rc, M=M, P=P, window=window, shape=windows.default_shape(window, P),
                      s0=s0, s=s_up, nI=nI, R=R, eps=eps)
    q = rng.uniform(-1, 1, N)
    q -= q.mean()
    pos = rng.random((N, 3)) * L
    if case % 3 == 2 and N > 6:
        k = N // 3
        pos[:k] = np.mod(rng.random(3) * L + rng.normal(scale=0.02 * L, size=(k, 3)), L)
        pos[pos >= L] = 0.0
    try:
        s = se.ParticleSystem(pos, q, L)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            phi = se.total_potential(s, prm, se.Periodicity(D))
            ref = orc.total_potential(pos, q, L, D, dict(prm.__dict__))
        err = se.relative_rms_error(phi, ref)
    except Exception as e:  # noqa: BLE001
        fails.append((case, D, window, P, M, L, N, repr(e)[:120]))
        continue
    worst = max(worst, err)
    if not err < 1e-11:
        fails.append((case, D, window, P, M, L, N, err))
print(f"{n_cases} cases, worst rel RMS {worst:.2e}, {len(fails)} failures")
for f in fails[:30]:
    print(f)
