"""Seeded synthetic inputs and parameters for BASELINE.json configs[0..4]
(BASELINE.md 3.1): rng = default_rng(config number), charges
uniform in [-1, 1] shifted to zero mean, positions in [0, L).  Used by
bench.py (--workload) and the full-size GPU tests.  No public dataset exists
for this path; these are the benchmark inputs.
"""

from __future__ import annotations

import math

import numpy as np


def _charges(rng, N):
    q = rng.uniform(-1.0, 1.0, N)
    return q - q.mean()


def _padded(s, n):
    want = int(math.ceil(s * n - 1e-9))
    if want <= n:
        return n
    m = max(2, want)
    while True:
        k = m
        for p in (2, 3, 5, 7):
            while k % p == 0:
                k //= p
        if m % 2 == 0 and k == 1:
            return m
        m += 1


def _R(D, L, M, P, s0):
    """Truncation radius as params.auto_params derives it (params.py:134-144)."""
    h = L / M
    return 0.5 * (_padded(s0, M + P) * h - L + math.sqrt(3.0 - D) * L)


def cfg1():
    """D=3, N=2000, L=1, Gaussian P=16, M=32, rc=0.3, xi=12.94."""
    rng = np.random.default_rng(1)
    N, L = 2000, 1.0
    pos = rng.random((N, 3)) * L
    return dict(name="cfg1", D=3, L=L, pos=pos, q=_charges(rng, N),
                prm=dict(xi=12.94, rc=0.3, M=32, P=16, window="gaussian", shape=math.sqrt(16 * math.pi),
                         eps=1e-8))


def cfg2():
    """D=3, N=1e6, L=10, ES P=8 beta=20, M=128, rc=1.0, xi=sqrt(-ln 1e-8)."""
    rng = np.random.default_rng(2)
    N, L = 1_000_000, 10.0
    pos = rng.random((N, 3)) * L
    return dict(name="cfg2", D=3, L=L, pos=pos, q=_charges(rng, N),
                prm=dict(xi=math.sqrt(-math.log(1e-8)) / 1.0, rc=1.0, M=128, P=8, window="bm", shape=20.0,
                         eps=1e-8))


def cfg3(variant="as_worded"):
    """D=2 (x, y periodic), N=2e5, L=5, ES P=8, M=96, s0=4, s=2, nI=10, xi=6.
    variant="tolerance": P=10, s=4, nI=48 (meets 1e-8)."""
    rng = np.random.default_rng(3)
    N, L = 200_000, 5.0
    pos = rng.random((N, 3)) * L
    xi, eps = 6.0, 1e-8
    rc = math.sqrt(-math.log(eps)) / xi
    if variant == "tolerance":
        P, s, nI = 10, 4.0, 48
    else:
        P, s, nI = 8, 2.0, 10
    s0 = 4.0
    return dict(name=f"cfg3_{variant}", D=2, L=L, pos=pos, q=_charges(rng, N),
                prm=dict(xi=xi, rc=rc, M=96, P=P, window="bm", shape=2.5 * P, s0=s0, s=s, nI=nI,
                         R=_R(2, L, 96, P, s0), eps=eps))


def cfg4():
    """D=1, N=2e5 in a 4x4x8 box with the periodic axis first (cubic
    embedding L=8: x <- config z in [0, 8), y, z <- config x, y in [0, 4)),
    Gaussian P=12, M=128, xi=4, rc at 1e-9, s0=2.4674, s=ln(1e9)/2pi, nI=39."""
    rng = np.random.default_rng(4)
    N, L = 200_000, 8.0
    pos = np.empty((N, 3))
    pos[:, 0] = rng.random(N) * 8.0
    pos[:, 1:] = rng.random((N, 2)) * 4.0
    xi, eps = 4.0, 1e-9
    rc = math.sqrt(-math.log(eps)) / xi
    s0, s = 2.4674, math.log(1.0 / eps) / (2 * math.pi)
    return dict(name="cfg4", D=1, L=L, pos=pos, q=_charges(rng, N),
                prm=dict(xi=xi, rc=rc, M=128, P=12, window="gaussian", shape=math.sqrt(12 * math.pi), s0=s0,
                         s=s, nI=39, R=_R(1, L, 128, 12, s0), eps=eps))


def cfg5():
    """D=0, N=5e5, L=4: 250k uniform in the ball r<2 about (2,2,2) and 250k in
    32 Gaussian clusters (sigma 0.05, centres uniform in the ball r<1.75),
    clipped to [0, 4); ES P=10 beta=25, M=96, xi=6, s0=4 (kernel path)."""
    rng = np.random.default_rng(5)
    N, L = 500_000, 4.0
    c = np.array([2.0, 2.0, 2.0])

    def ball(n, rad):
        out = np.empty((0, 3))
        while len(out) < n:
            p = rng.uniform(-rad, rad, (2 * n, 3))
            out = np.vstack([out, p[np.sum(p * p, axis=1) < rad * rad]])
        return out[:n]

    uni = ball(N // 2, 2.0) + c
    centres = ball(32, 1.75) + c
    lab = rng.integers(0, 32, N - N // 2)
    clus = centres[lab] + rng.normal(0.0, 0.05, (N - N // 2, 3))
    pos = np.clip(np.vstack([uni, clus]), 0.0, np.nextafter(L, 0.0))
    xi, eps = 6.0, 1e-8
    rc = math.sqrt(-math.log(eps)) / xi
    s0 = 4.0
    return dict(name="cfg5", D=0, L=L, pos=pos, q=_charges(rng, N),
                prm=dict(xi=xi, rc=rc, M=96, P=10, window="bm", shape=25.0, s0=s0, R=_R(0, L, 96, 10, s0),
                         eps=eps))


def cfg1_tol():
    """cfg1 re-parameterised to meet its 1e-8 tolerance (keep rc=0.3,
    xi=14.31, M=40 from select_kinf).  Measured with the reference on the cfg1
    inputs against a tight auto_params run (eps=1e-14): total potential
    3.7e-9 relative RMS (cfg1 as worded: 2.7e-8)."""
    w = cfg1()
    w["name"] = "cfg1_tol"
    w["prm"].update(xi=14.31, M=40)
    return w


def cfg2_tol():
    """cfg2 with the ES window widened to P=10, beta=2.5P=25 -- the reference's
    own D=3 p-sweep (frontend/test/fixtures/p_sweep_bm_d3.csv:7-8: P=8 1.38e-8,
    P=10 9.2e-11).  Same inputs, xi, rc and M.  Measured with the reference on
    a 1,500-particle probe of the cfg2 box against a tight SE run (P=20, M=192):
    k-space 2.1e-9 relative RMS (P=8, beta=20: 3.2e-8)."""
    w = cfg2()
    w["name"] = "cfg2_tol"
    w["prm"].update(P=10, shape=25.0)
    return w


def cfg4_tol():
    """cfg4 at its 1e-9 tolerance.  The Gaussian P=12 window is the limit, not
    the free-axis upsampling: on a 60-particle probe of the cfg4 box against the
    reference's singly periodic direct sum (oracle.kspace_direct_1p, kmax at
    1e-13) P=12 gives 7.9e-8 at s = 3.3, 4 and 5 alike; P=14 5.6e-9; P=16
    4.6e-10.  So P=16 (m = sqrt(16 pi)), s, nI, s0 as in cfg4 (M+P=144 even)."""
    w = cfg4()
    w["name"] = "cfg4_tol"
    P, s0 = 16, w["prm"]["s0"]
    w["prm"].update(P=P, shape=math.sqrt(P * math.pi), R=_R(1, w["L"], 128, P, s0))
    return w


ALL = {"cfg1": cfg1, "cfg1_tol": cfg1_tol, "cfg2": cfg2, "cfg2_tol": cfg2_tol, "cfg3": cfg3,
       "cfg3_tol": lambda: cfg3("tolerance"), "cfg4": cfg4, "cfg4_tol": cfg4_tol, "cfg5": cfg5}
