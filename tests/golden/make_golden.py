"""Generate golden vectors by running the UNMODIFIED reference (`pmewald`).

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes `tests/golden/<case>.npz`.  Each case stores the seeded inputs, the
SEParams fields, and the reference's outputs for the hot-path stages:
spread grid H (sekspace.spread), Fourier potential (sekspace.se_kspace),
real-space potential (realspace.real_space_sum), self term and total
potential (core.total_potential).  Table cases pin window transforms
(windows.fourier), zero-block Green's functions (greens.zero_mode_values)
and the D=0 truncated kernel (sekspace.precompute_truncated_greens).
"""

from __future__ import annotations

import math
import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from pmewald import aft, core, greens, oracle, params as pm, realspace, sekspace, windows  # noqa: E402
from pmewald.core import ParticleSystem, Periodicity, SEParams  # noqa: E402


def system(N, L, seed):
    rng = np.random.default_rng(seed)
    pos = rng.random((N, 3)) * L
    q = rng.uniform(-1.0, 1.0, N)
    q -= q.mean()
    return ParticleSystem(pos, q, float(L))


def explicit(D, L, M, P, xi, window, eps, nI=None, s_override=None, s0_min=None, shape=None):
    """Parameters in the style of the reference tests (test_sekspace.py:16-34)."""
    h = L / M
    Lt = L + P * h
    d = 3.0 - D
    rc = min(math.sqrt(-math.log(eps)) / xi, L / 2 if D >= 1 else L)
    if D < 3:
        s0 = max(1.0 + math.sqrt(d), ((1.0 + math.sqrt(d)) * L + 2 * rc) / Lt)
        if s0_min:
            s0 = max(s0, s0_min)
        R = 0.5 * (aft.padded_size(s0, M + P) * h - L + math.sqrt(d) * L)
    else:
        s0, R = 1.0, 0.0
    s = (s_override or max(1.0, math.log(1.0 / eps) / (2 * math.pi))) if D in (1, 2) else 1.0
    nIv = nI if nI is not None else (M // 2 if D in (1, 2) else 0)
    shp = windows.default_shape(window, P) if shape is None else shape
    return SEParams(xi=xi, rc=rc, M=M, P=P, window=window, shape=shp, s0=s0, s=s,
                    nI=nIv, R=R, eps=eps)


def prm_dict(p: SEParams):
    return dict(xi=p.xi, rc=p.rc, M=p.M, P=p.P, window=p.window, shape=p.shape,
                s0=p.s0, s=p.s, nI=p.nI, R=p.R, eps=p.eps)


def save_pipeline(name, s, D, p, use_kernel=None, with_real=True):
    peri = Periodicity(D)
    grid = sekspace.Grid.build(s.L, p, peri)
    wspec = windows.WindowSpec(p.window, p.P, grid.h, p.shape)
    H = sekspace.spread(s, wspec, grid, peri)
    phik = sekspace.se_kspace(s, p, peri, use_kernel=use_kernel)
    out = dict(pos=s.positions, q=s.charges, L=s.L, D=D, H=H.values, phi_k=phik,
               g0=grid.g0, gs=grid.gs, Mt=grid.Mt,
               use_kernel=-1 if use_kernel is None else int(use_kernel))
    if with_real:
        phir = realspace.real_space_sum(s, p.xi, p.rc, peri)
        phis = realspace.self_term(s.charges, p.xi)
        if use_kernel is None:
            tot = core.total_potential(s, p, peri)
        else:
            tot = phir + phik + phis
        out.update(phi_r=phir, phi_s=phis, phi=tot)
    for k, v in prm_dict(p).items():
        out["prm_" + k] = v
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, {k: (v.shape if hasattr(v, "shape") else v) for k, v in out.items()
                 if k in ("H", "phi_k")})


def main():
    warnings.simplefilter("ignore")
    # --- D=3: cfg1-shaped (Gaussian P=16, M=32, rc=0.3, xi=12.94) at N=400
    s = system(400, 1.0, 101)
    p = SEParams(xi=12.94, rc=0.3, M=32, P=16, window="gaussian",
                 shape=math.sqrt(16 * math.pi), eps=1e-8)
    save_pipeline("d3_gauss_cfg1", s, 3, p)
    # --- D=3: cfg2-shaped (ES P=8, beta=20, rc = L/10) at L=2, N=500
    s = system(500, 2.0, 102)
    p = SEParams(xi=4.2919 * 5, rc=0.2, M=24, P=8, window="bm", shape=20.0, eps=1e-8)
    save_pipeline("d3_bm_cfg2", s, 3, p)
    # --- D=3: KB window
    s = system(200, 1.0, 103)
    p = SEParams(xi=8.0, rc=0.45, M=20, P=8, window="kb", shape=20.0, eps=1e-8)
    save_pipeline("d3_kb", s, 3, p)
    # --- D=3: small grid, wrap-heavy (P close to M)
    s = system(60, 1.0, 104)
    p = SEParams(xi=5.0, rc=0.5, M=10, P=8, window="bm", shape=20.0, eps=1e-6)
    save_pipeline("d3_bm_wrap", s, 3, p)
    # --- D=2: cfg3-shaped (ES P=8, s0 >= 4, s = 2, nI small)
    s = system(300, 1.0, 201)
    p = explicit(2, 1.0, 16, 8, 7.0, "bm", 1e-8, nI=3, s_override=2.0, s0_min=4.0)
    save_pipeline("d2_bm_cfg3", s, 2, p)
    s = system(250, 1.0, 202)
    p = explicit(2, 1.0, 18, 10, 6.0, "gaussian", 1e-8, nI=4)
    save_pipeline("d2_gauss", s, 2, p)
    # --- D=1: cfg4-shaped (Gaussian P=12, nI = 4)
    s = system(250, 1.0, 301)
    p = explicit(1, 1.0, 16, 12, 6.0, "gaussian", 1e-9, nI=4)
    save_pipeline("d1_gauss_cfg4", s, 1, p)
    s = system(200, 1.0, 302)
    p = explicit(1, 1.0, 14, 8, 5.0, "bm", 1e-8, nI=3)
    save_pipeline("d1_bm", s, 1, p)
    # --- D=0: cfg5-shaped (ES P=10), kernel path and full upsampling path
    s = system(300, 1.0, 401)
    p = explicit(0, 1.0, 16, 10, 6.0, "bm", 1e-8)
    save_pipeline("d0_bm_kernel", s, 0, p)
    save_pipeline("d0_bm_full", s, 0, p, use_kernel=False, with_real=False)
    s = system(150, 1.0, 402)
    p = explicit(0, 1.0, 14, 8, 7.0, "gaussian", 1e-8)
    save_pipeline("d0_gauss_kernel", s, 0, p)
    # --- auto_params end to end (params.py:102-164), every D
    for D in (0, 1, 2, 3):
        s = system(80, 1.0, 500 + D)
        p, _ = pm.auto_params(s, Periodicity(D), 6.0, 1e-9)
        save_pipeline(f"auto_d{D}", s, D, p)
    # --- real space only: image path (rc > L/2) and mixed periodicities
    rs = {}
    s = system(40, 1.0, 601)
    rs["img_pos"], rs["img_q"] = s.positions, s.charges
    rs["img_d3"] = realspace.real_space_sum(s, 4.0, 1.2, Periodicity(3))
    rs["img_d2"] = realspace.real_space_sum(s, 4.0, 0.8, Periodicity(2))
    rs["img_d1"] = realspace.real_space_sum(s, 4.0, 0.7, Periodicity(1))
    s = system(600, 1.0, 602)
    rs["cell_pos"], rs["cell_q"] = s.positions, s.charges
    for D in (0, 1, 2, 3):
        rs[f"cell_d{D}"] = realspace.real_space_sum(s, 7.0, 0.23, Periodicity(D))
        rs[f"cell2_d{D}"] = realspace.real_space_sum(s, 5.0, 0.45, Periodicity(D))
    np.savez_compressed(os.path.join(HERE, "realspace.npz"), **rs)
    # --- tables
    tb = {}
    for kind, P, shape in (("bm", 8, 20.0), ("bm", 10, 25.0), ("bm", 16, 40.0),
                           ("gaussian", 12, math.sqrt(12 * math.pi)), ("kb", 8, 20.0)):
        h = 1.0 / 24
        spec = windows.WindowSpec(kind, P, h, shape)
        for n in (24, 70, 210):
            k = sekspace.mode_values(n, h)
            tb[f"wf_{kind}_{P}_{n}"] = np.asarray(windows.fourier(k, spec), dtype=float)
        x = np.linspace(-spec.w * 1.1, spec.w * 1.1, 101)
        tb[f"we_{kind}_{P}"] = windows.evaluate(x, spec)
    kap = np.concatenate([np.linspace(0, 0.02, 21), np.linspace(0.02, 200, 301)])
    tb["kappa"] = kap
    for D in (0, 1, 2):
        for R in (1.7, 3.2):
            tb[f"g_{D}_{R}"] = greens.zero_mode_values(D, R, kap)
    np.savez_compressed(os.path.join(HERE, "tables.npz"), **tb)
    kern = sekspace.precompute_truncated_greens(1.0, 16, 8, 1 + math.sqrt(3.0), rc=0.5)
    np.savez_compressed(os.path.join(HERE, "d0_kernel.npz"), ghat=kern.ghat, nconv=kern.nconv,
                        g0=kern.g0, R=kern.R, Mt=kern.Mt)
    # --- parameter selection
    ap = {}
    for i, (D, xi, eps, win, N, L) in enumerate([(3, 6.0, 1e-8, "bm", 50, 1.0),
                                                  (2, 6.0, 1e-10, "bm", 50, 1.0),
                                                  (1, 4.0, 1e-9, "gaussian", 60, 2.0),
                                                  (0, 6.0, 1e-8, "bm", 40, 1.0),
                                                  (3, 4.2919, 1e-8, "bm", 100, 10.0)]):
        s = system(N, L, 700 + i)
        p, _ = pm.auto_params(s, Periodicity(D), xi, eps, window=win)
        ap[f"case{i}"] = np.array([D, xi, eps, N, L, 700 + i])
        ap[f"case{i}_win"] = win
        ap[f"case{i}_out"] = np.array([p.xi, p.rc, p.M, p.P, p.shape, p.s0, p.s, p.nI, p.R, p.eps])
    np.savez_compressed(os.path.join(HERE, "auto_params.npz"), **ap)


def direct_golden():
    """The reference's direct Ewald evaluators (oracle.py:109-118, 181-192) on
    small seeded systems: pins the device direct sums (se_direct.cu)."""
    out = {}
    for i, (N, L, xi, eps) in enumerate([(40, 1.0, 6.3, 1e-12), (35, 2.0, 3.0, 1e-12)]):
        s = system(N, L, 900 + i)
        kmax = oracle.OracleConfig.for_accuracy(xi, L, eps).kmax
        out[f"d3_{i}_in"] = np.array([N, L, xi, kmax, 900 + i])
        out[f"d3_{i}_pos"], out[f"d3_{i}_q"] = s.positions, s.charges
        out[f"d3_{i}_phi"] = oracle.kspace_direct_3p(s, xi, kmax)
    for i, (N, L, xi, eps) in enumerate([(25, 1.0, 6.3, 1e-12), (20, 2.0, 3.0, 1e-12)]):
        s = system(N, L, 920 + i)
        kmax = oracle.OracleConfig.for_accuracy(xi, L, eps).kmax
        out[f"d2_{i}_in"] = np.array([N, L, xi, kmax, 920 + i])
        out[f"d2_{i}_pos"], out[f"d2_{i}_q"] = s.positions, s.charges
        out[f"d2_{i}_phi"] = oracle.kspace_direct_2p(s, xi, kmax)
    for i, (N, L, xi, eps) in enumerate([(14, 1.0, 6.3, 1e-12), (12, 2.0, 3.0, 1e-12)]):
        s = system(N, L, 940 + i)
        kmax = oracle.OracleConfig.for_accuracy(xi, L, eps).kmax
        out[f"d1_{i}_in"] = np.array([N, L, xi, kmax, 940 + i])
        out[f"d1_{i}_pos"], out[f"d1_{i}_q"] = s.positions, s.charges
        out[f"d1_{i}_phi"] = oracle.kspace_direct_1p(s, xi, kmax)
    for i, (N, L, xi) in enumerate([(60, 1.0, 6.3), (50, 3.0, 2.0)]):
        s = system(N, L, 950 + i)
        out[f"d0_{i}_in"] = np.array([N, L, xi, 950 + i])
        out[f"d0_{i}_pos"], out[f"d0_{i}_q"] = s.positions, s.charges
        out[f"d0_{i}_phi"] = oracle.kspace_direct_0p(s, xi)
    np.savez_compressed(os.path.join(HERE, "direct.npz"), **out)


if __name__ == "__main__":
    if sys.argv[1:] == ["direct"]:
        sys.exit(direct_golden())
    main()
    sys.exit(direct_golden())
