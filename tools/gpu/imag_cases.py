"""The randomized cases where the reference's realness guard fires: compare
the device result with the oracle's real part (guard disabled)."""
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

ratios = {}
_real = orc._check_real


def probe(out):
    ref = np.max(np.abs(out.real)) + 1e-300
    ratios["imag/real"] = float(np.max(np.abs(out.imag)) / ref)


orc._check_real = probe
for case in (16, 62, 63, 216, 256):
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
    s0 = max(1.0 + math.sqrt(d), ((1.0 + math.sqrt(d)) * L + 2.0 * rc) / (L + P * h))
    R = 0.5 * (se.aft.padded_size(s0, M + P) * h - L + math.sqrt(d) * L)
    s_up = max(1.0, math.log(1.0 / eps) / (2 * math.pi))
    nI = int(rng.integers(0, M // 2 + 1))
    prm = se.SEParams(xi=xi, rc=rc, M=M, P=P, window=window, shape=windows.default_shape(window, P),
                      s0=s0, s=s_up, nI=nI, R=R, eps=eps)
    q = rng.uniform(-1, 1, N)
    q -= q.mean()
    pos = rng.random((N, 3)) * L
    if case % 3 == 2 and N > 6:
        k = N // 3
        pos[:k] = np.mod(rng.random(3) * L + rng.normal(scale=0.02 * L, size=(k, 3)), L)
        pos[pos >= L] = 0.0
    s = se.ParticleSystem(pos, q, L)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        phik = se.se_kspace(s, prm, se.Periodicity(D))
        refk = orc.se_kspace(pos, q, L, D, dict(prm.__dict__))
    print(case, D, window, P, M, f"imag/real {ratios.get('imag/real'):.2e}",
          f"device vs oracle real part {se.relative_rms_error(phik, refk):.2e}")
