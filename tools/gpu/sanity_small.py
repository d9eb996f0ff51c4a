"""Small end-to-end cases for compute-sanitizer (memcheck) runs: every
periodicity, both spreading paths (tile / direct), sharded entry points."""

import os
import sys
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tools")]
import workloads  # noqa: E402
import paper_1712_04732_b200 as se  # noqa: E402

rng = np.random.default_rng(0)
warnings.simplefilter("ignore")
for D in (0, 1, 2, 3):
    for N, L in ((37, 1.0), (900, 2.0)):
        pos = rng.random((N, 3)) * L
        q = rng.uniform(-1, 1, N)
        q -= q.mean()
        s = se.ParticleSystem(pos, q, L)
        for xi in (4.0, 9.0):
            p, _ = se.auto_params(s, se.Periodicity(D), xi, 1e-8)
            phi = se.total_potential(s, p, se.Periodicity(D))
            assert np.all(np.isfinite(phi))
            if D == 0:
                se.se_kspace(s, p, se.Periodicity(0), use_kernel=False)
s = se.ParticleSystem(rng.random((50, 3)), np.r_[np.ones(25), -np.ones(25)], 1.0)
p = se.SEParams(xi=12.0, rc=0.4, M=64, P=34, window="kb", shape=85.0, eps=1e-12)
se.se_kspace(s, p, se.Periodicity(3))
# the compile-time-P tile kernels (spread: 30-lane pair rows at P = 10, the
# warp-specialised kernel at P = 8), ES and Gaussian windows, D = 3 and D = 1
s = se.ParticleSystem(rng.random((3000, 3)) * 2.0, np.r_[np.ones(1500), -np.ones(1500)], 2.0)
for P in (4, 6, 8, 10, 12, 16):
    for window, shape in (("bm", 2.5 * P), ("gaussian", float(np.sqrt(P * np.pi)))):
        for D in (3, 1):
            p = se.SEParams(xi=6.0, rc=0.5, M=32, P=P, window=window, shape=shape, eps=1e-8,
                            **({} if D == 3 else dict(s0=2.5, s=3.0, nI=6, R=workloads._R(1, 2.0, 32, P, 2.5))))
            phi = se.se_kspace(s, p, se.Periodicity(D))
            assert np.all(np.isfinite(phi))
# fields (every D; Gaussian window for D < 3), default and deterministic mode,
# and a dense system whose real-space batches take the dense (Newton and
# full-shell) paths as well as the compacted ones
from paper_1712_04732_b200.realspace import real_space_field, real_space_sum  # noqa: E402

dense = se.ParticleSystem(rng.random((6000, 3)), np.r_[np.ones(3000), -np.ones(3000)], 1.0)
for det in (False, True):
    se.set_deterministic(det)
    for D in (0, 1, 2, 3):
        s = se.ParticleSystem(rng.random((700, 3)) * 2.0, np.r_[np.ones(350), -np.ones(350)], 2.0)
        p, _ = se.auto_params(s, se.Periodicity(D), 5.0, 1e-8, window="gaussian")
        E = se.total_field(s, p, se.Periodicity(D))
        phi = se.total_potential(s, p, se.Periodicity(D))
        assert np.all(np.isfinite(E)) and np.all(np.isfinite(phi))
        assert np.all(np.isfinite(real_space_sum(dense, 14.0, 0.25, se.Periodicity(D))))
        assert np.all(np.isfinite(real_space_field(dense, 14.0, 0.25, se.Periodicity(D))))
se.set_deterministic(False)
print("sanity ok")
