"""Randomized parity campaign for the Newton (half-shell column) real-space
path and the larger-N binning: seeded configurations with enough columns
(L / rc in [2.6, 5]) and N in [3e3, 1.5e4], every periodicity and window,
a third of the cases clustered; the full device pipeline against the CPU
oracle.  usage: random_campaign_newton.py [cases]"""
import math
import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.join(HERE, "..", ".."), os.path.join(HERE, "..", "..", "oracle")]
import se_oracle as orc  # noqa: E402

import paper_1712_04732_b200 as se  # noqa: E402
from paper_1712_04732_b200 import windows  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 120
worst, fails, by_d = 0.0, [], {}
for case in range(n_cases):
    rng = np.random.default_rng(70000 + case)
    D = int(rng.integers(0, 4))
    window = ["bm", "gaussian", "kb"][int(rng.integers(0, 3))]
    P = int(rng.choice([4, 6, 8, 10, 12]))
    M = int(rng.choice([16, 20, 24, 32, 40]))
    N = int(rng.integers(3000, 15000))
    rc = 1.0
    L = float(rng.uniform(2.6, 5.0)) * rc
    xi = float(rng.uniform(2.5, 6.5)) / rc
    eps = 1e-10
    h = L / M
    if D < 3:
        d = 3.0 - D
        Lt = L + P * h
        s0 = max(1.0 + math.sqrt(d), ((1.0 + math.sqrt(d)) * L + 2 * rc) / Lt) + 0.1
        R = 0.5 * (se.aft.padded_size(s0, M + P) * h - L + math.sqrt(d) * L)
    else:
        s0, R = 1.0, 0.0
    s_up = max(1.0, math.log(1.0 / eps) / (2 * math.pi)) if D in (1, 2) else 1.0
    nI = int(rng.integers(0, M // 2 + 1)) if D in (1, 2) else 0
    if D in (1, 2) and (M + P) % 2:
        P += 1
    prm = se.SEParams(xi=xi, rc=rc, M=M, P=P, window=window, shape=windows.default_shape(window, P),
                      s0=s0, s=s_up, nI=nI, R=R, eps=eps)
    q = rng.uniform(-1, 1, N)
    q -= q.mean()
    pos = rng.random((N, 3)) * L
    if case % 3 == 2:
        k = N // 3
        pos[:k] = np.mod(rng.random(3) * L + rng.normal(scale=0.05 * L, size=(k, 3)), L)
        pos[pos >= L] = 0.0
    try:
        s = se.ParticleSystem(pos, q, L)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            phi = se.total_potential(s, prm, se.Periodicity(D))
            ref = orc.total_potential(pos, q, L, D, dict(prm.__dict__))
        err = se.relative_rms_error(phi, ref)
    except Exception as e:  # noqa: BLE001
        fails.append((case, D, window, P, M, round(L, 2), N, repr(e)[:120]))
        continue
    worst = max(worst, err)
    by_d[D] = max(by_d.get(D, 0.0), err)
    if not err < 1e-11:
        fails.append((case, D, window, P, M, round(L, 2), N, err))
print(f"{n_cases} cases, worst rel RMS {worst:.2e} (per D: "
      + ", ".join(f"{k}: {v:.1e}" for k, v in sorted(by_d.items())) + f"), {len(fails)} failures")
for f in fails[:30]:
    print(f)
