"""Electric field / forces (D = 3) on the device against the field oracle
(pinned to the reference by central differences, tests/test_field_cpu.py)
and against the direct Ewald field."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import se_oracle as orc  # noqa: E402

import paper_1712_04732_b200 as se  # noqa: E402

pytestmark = pytest.mark.gpu

G = np.load(os.path.join(ROOT, "tests", "golden", "field.npz"))


def _rel(a, b):
    return float(np.sqrt(np.mean((a - b) ** 2)) / np.sqrt(np.mean(b ** 2)))


def _system(N, L, seed):
    rng = np.random.default_rng(seed)
    pos = rng.random((N, 3)) * L
    q = rng.uniform(-1, 1, N)
    q -= q.mean()
    return pos, q


def _prm_dict(p):
    return dict(xi=p.xi, rc=p.rc, M=p.M, P=p.P, window=p.window, shape=p.shape)


def test_field_matches_oracle_and_reference_differences():
    # small box: few columns -> the minimum-image kernel
    pos, q, L = G["pos"], G["q"], float(G["L"])
    p = se.SEParams(xi=float(G["xi"]), rc=float(G["rc"]), M=32, P=16, window="gaussian",
                    shape=float(np.sqrt(16 * np.pi)), eps=1e-12)
    s = se.ParticleSystem(pos, q, L)
    E = se.total_field(s, p, se.Periodicity(3))
    ref = orc.total_field(pos, q, L, _prm_dict(p))
    assert _rel(E, ref) < 1e-12
    # against the reference's own potentials (real space + direct Fourier sum)
    assert _rel(E, G["E_real_fd"] + G["E_kspace_direct_fd"]) < 1e-7
    F = se.forces(s, p, se.Periodicity(3))  # a second evaluation: fp64 atomics reorder the last bits
    assert _rel(F, q[:, None] * E) < 1e-14


@pytest.mark.parametrize("window,P,shape", [("bm", 8, 20.0), ("gaussian", 12, float(np.sqrt(12 * np.pi))),
                                            ("kb", 10, 25.0)])
def test_field_newton_path_vs_oracle(window, P, shape):
    # enough columns for the half-shell (Newton) kernel; all three windows
    pos, q = _system(20000, 2.0, 61)
    p = se.SEParams(xi=7.0, rc=0.55, M=40, P=P, window=window, shape=shape, eps=1e-8)
    E = se.total_field(se.ParticleSystem(pos, q, 2.0), p, se.Periodicity(3))
    sel = np.random.default_rng(1).choice(len(q), 300, replace=False)
    er = orc.realspace_field(pos, q, 2.0, 3, p.xi, p.rc, targets=sel)
    ek = orc.kspace_field_d3(pos, q, 2.0, _prm_dict(p))[sel]
    assert _rel(E[sel], er + ek) < 1e-12


def test_field_image_path_and_wide_erfc():
    # rc > L/2: explicit images; xi rc > 6: the library-erfc kernel variant
    pos, q = _system(200, 1.0, 62)
    for xi, rc in ((5.0, 0.7), (14.0, 0.45)):
        p = se.SEParams(xi=xi, rc=rc, M=32, P=12, window="bm", shape=30.0, eps=1e-8)
        E = se.total_field(se.ParticleSystem(pos, q, 1.0), p, se.Periodicity(3))
        ref = orc.total_field(pos, q, 1.0, _prm_dict(p))
        assert _rel(E, ref) < 1e-12, (xi, rc)


def test_field_device_api_and_rejections():
    import torch

    from paper_1712_04732_b200 import device as sedev

    pos, q = _system(3000, 1.5, 63)
    p = se.SEParams(xi=8.0, rc=0.45, M=32, P=8, window="bm", shape=20.0, eps=1e-8)
    host = se.total_field(se.ParticleSystem(pos, q, 1.5), p, se.Periodicity(3))
    dev = sedev.total_field(torch.from_numpy(pos).cuda(), torch.from_numpy(q).cuda(), 1.5, p,
                            se.Periodicity(3)).cpu().numpy()
    assert _rel(dev, host) < 1e-14
    with pytest.raises(ValueError):
        se.total_field(se.ParticleSystem(pos, q, 1.5), p, se.Periodicity(2))
    with pytest.raises(ValueError):  # non-neutral periodic system
        se.total_field(se.ParticleSystem(pos, q + 1.0, 1.5), p, se.Periodicity(3))


def test_field_full_size_cfg2_momentum_and_differences():
    # cfg2 at full size: Newton's third law holds pairwise in real space and
    # the ik-differentiated Fourier field conserves momentum exactly, so
    # sum q E = 0 to rounding; E = -grad phi against central differences of
    # the device potential at a few particles (SE discretisation ~1e-6)
    rng = np.random.default_rng(2)
    N, L = 1_000_000, 10.0
    pos = rng.random((N, 3)) * L
    q = rng.uniform(-1, 1, N)
    q -= q.mean()
    p = se.SEParams(xi=4.2919, rc=1.0, M=128, P=8, window="bm", shape=20.0, eps=1e-8)
    s = se.ParticleSystem(pos, q, L)
    E = se.total_field(s, p, se.Periodicity(3))
    F = q[:, None] * E
    assert np.abs(F.sum(0)).max() < 1e-10 * np.abs(F).sum(0).max()
    sel = np.random.default_rng(3).choice(N, 200, replace=False)
    # sampled parity against the oracle at full size (the oracle spreads all
    # 1e6 charges in numpy: ~15 s)
    er = orc.realspace_field(pos, q, L, 3, p.xi, p.rc, targets=sel)
    ek = orc.kspace_field_d3(pos, q, L, _prm_dict(p), targets=sel)
    assert _rel(E[sel], er + ek) < 1e-11
    d = 1e-4
    for m in sel[:3]:
        for a in range(3):
            p1, p2 = pos.copy(), pos.copy()
            p1[m, a] += d
            p2[m, a] -= d
            f1 = se.total_potential(se.ParticleSystem(p1, q, L), p, se.Periodicity(3))[m]
            f2 = se.total_potential(se.ParticleSystem(p2, q, L), p, se.Periodicity(3))[m]
            fd = -(f1 - f2) / (2 * d)
            assert abs(fd - E[m, a]) < 1e-4 * np.abs(E[m]).max(), (m, a, fd, E[m, a])


def test_field_randomized_configurations():
    # seeded random D = 3 configurations across the kernel variants (minimum
    # image / Newton / image path / wide erfc), windows and supports
    rng = np.random.default_rng(2024)
    worst = 0.0
    for case in range(12):
        N = int(rng.integers(40, 1500))
        L = float(rng.uniform(0.8, 3.0))
        M = int(rng.choice([16, 24, 32, 40]))
        P = int(rng.choice([4, 6, 8, 10, 12]))
        P = min(P, M)
        window = str(rng.choice(["gaussian", "bm", "kb"]))
        shape = {"gaussian": float(np.sqrt(np.pi * P)), "bm": 2.5 * P, "kb": 2.5 * P}[window]
        rc = float(rng.uniform(0.15, 0.7)) * L
        xi = float(rng.uniform(2.5, 7.5)) / rc
        pos, q = _system(N, L, 1000 + case)
        p = se.SEParams(xi=xi, rc=rc, M=M, P=P, window=window, shape=shape, eps=1e-8)
        E = se.total_field(se.ParticleSystem(pos, q, L), p, se.Periodicity(3))
        ref = orc.total_field(pos, q, L, _prm_dict(p))
        err = _rel(E, ref)
        worst = max(worst, err)
        assert err < 1e-11, (case, N, L, M, P, window, rc, xi, err)
    print(f"randomized field cases: worst relative RMS {worst:.2e}")


def test_field_stages_match_oracle_parts_all_periodicities():
    # the two parts separately: real-space pair field for every D (image path
    # included), Fourier field for D = 3; their sum is total_field
    pos, q = _system(1500, 1.2, 64)
    s = se.ParticleSystem(pos, q, 1.2)
    for D in (0, 1, 2, 3):
        for rc in (0.35, 0.7):
            Er = se.realspace.real_space_field(s, 7.0 / rc, rc, se.Periodicity(D))
            ref = orc.realspace_field(pos, q, 1.2, D, 7.0 / rc, rc)
            assert _rel(Er, ref) < 1e-13, (D, rc)
    p = se.SEParams(xi=12.0, rc=0.45, M=32, P=8, window="bm", shape=20.0, eps=1e-8)
    Ek = se.sekspace.se_kspace_field(s, p, se.Periodicity(3))
    assert _rel(Ek, orc.kspace_field_d3(pos, q, 1.2, _prm_dict(p))) < 1e-12
    Et = se.total_field(s, p, se.Periodicity(3))
    Er = se.realspace.real_space_field(s, p.xi, p.rc, se.Periodicity(3))
    assert _rel(Et, Er + Ek) < 1e-14


def test_field_empty_and_zero_charge_systems():
    p = se.SEParams(xi=8.0, rc=0.4, M=24, P=8, window="bm", shape=20.0, eps=1e-8)
    E = se.total_field(se.ParticleSystem(np.zeros((0, 3)), np.zeros(0), 1.0), p, se.Periodicity(3))
    assert E.shape == (0, 3)
    pos, _ = _system(300, 1.0, 65)
    E0 = se.total_field(se.ParticleSystem(pos, np.zeros(300), 1.0), p, se.Periodicity(3))
    assert E0.shape == (300, 3) and np.all(E0 == 0.0)
    Er = se.realspace.real_space_field(se.ParticleSystem(np.zeros((0, 3)), np.zeros(0), 1.0), 8.0, 0.4,
                                       se.Periodicity(1))
    assert Er.shape == (0, 3)


G3 = np.load(os.path.join(ROOT, "tests", "golden", "field_dlt3.npz"))


@pytest.mark.parametrize("D", [2, 1, 0])
@pytest.mark.parametrize("window", ["gaussian", "kb"])
def test_field_dlt3_matches_oracle(D, window):
    # D < 3: real-space pair field + the gradient of the gather on the
    # filtered grid (window derivative), device vs oracle restatement
    pos, q = _system(3000, 1.5, 70 + D)
    shape = np.sqrt(8 * np.pi) if window == "gaussian" else 2.3 * 8
    p = se.SEParams(xi=7.0, rc=0.5, M=24, P=8, window=window, shape=shape, s0=3.0, s=2.0, nI=4, R=2.5,
                    eps=1e-8)
    s = se.ParticleSystem(pos, q, 1.5)
    E = se.total_field(s, p, se.Periodicity(D))
    prm = dict(xi=p.xi, rc=p.rc, M=p.M, P=p.P, window=p.window, shape=p.shape, s0=p.s0, s=p.s, nI=p.nI, R=p.R)
    ref = orc.realspace_field(pos, q, 1.5, D, p.xi, p.rc) + orc.kspace_field_grad(pos, q, 1.5, D, prm)
    err = _rel(E, ref)
    Ek = se.sekspace.se_kspace_field(s, p, se.Periodicity(D))
    errk = _rel(Ek, orc.kspace_field_grad(pos, q, 1.5, D, prm))
    print(f"D={D} {window}: total {err:.2e} k-space {errk:.2e}")
    assert err < 1e-12 and errk < 1e-12


@pytest.mark.parametrize("D", [2, 1, 0])
def test_field_dlt3_vs_reference_differences(D):
    # tight parameters: the device field against central differences of the
    # reference's own real_space_sum and direct Fourier-space sums
    L, xi, rc, kmax, delta = G3[f"D{D}_prm"]
    pos, q = G3[f"D{D}_pos"], G3[f"D{D}_q"]
    s = se.ParticleSystem(pos, q, L)
    p, _ = se.auto_params(s, se.Periodicity(D), xi, 1e-13, window="gaussian")
    pr = se.SEParams(xi=p.xi, rc=rc, M=p.M, P=p.P, window=p.window, shape=p.shape, s0=p.s0, s=p.s, nI=p.nI,
                     R=p.R, eps=p.eps)
    E = se.total_field(s, pr, se.Periodicity(D))
    ref = G3[f"D{D}_E_real_fd"] + G3[f"D{D}_E_kspace_direct_fd"]
    err = _rel(E, ref)
    print(f"D={D}: device field vs reference differences {err:.2e}")
    assert err < 1e-6


def test_field_dlt3_rejects_es_window():
    pos, q = _system(500, 1.0, 3)
    p = se.SEParams(xi=7.0, rc=0.45, M=20, P=8, window="bm", shape=20.0, s0=3.0, s=2.0, nI=4, R=2.0)
    with pytest.raises(ValueError):
        se.total_field(se.ParticleSystem(pos, q, 1.0), p, se.Periodicity(2))


@pytest.mark.parametrize("D", [0, 1, 2, 3])
def test_field_newton_dense_batches_match_full_shell(D):
    # a dense system (~2000 partners per particle: most batches take the
    # dense Newton path, dense_batch_field_poly) against the deterministic
    # mode's full-shell field, which sums every target's partners itself
    N, L = 30000, 1.0
    pos, q = _system(N, L, 77 + D)
    xi, rc = 14.0, 0.25
    from paper_1712_04732_b200.realspace import real_space_field

    system = se.ParticleSystem(pos, q, L)
    e_newton = real_space_field(system, xi, rc, se.Periodicity(D))
    se.set_deterministic(True)
    try:
        e_full = real_space_field(system, xi, rc, se.Periodicity(D))
    finally:
        se.set_deterministic(False)
    assert _rel(e_newton, e_full) < 1e-13
    # Newton's third law pairwise: the real-space forces sum to zero
    F = q[:, None] * e_newton
    assert np.abs(F.sum(0)).max() < 1e-11 * np.abs(F).sum(0).max()
    sel = np.random.default_rng(5).choice(N, 40, replace=False)
    ref = orc.realspace_field(pos, q, L, D, xi, rc, targets=sel)
    assert _rel(e_newton[sel], ref) < 1e-12
