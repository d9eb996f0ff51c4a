"""Device direct Ewald sums (paper_1712_04732_b200.direct, csrc/se_direct.cu)
against the reference's own oracle outputs, and the SE k-space path checked
against them at FULL size (cfg2: N = 1e6, D = 3; cfg3: N = 2e5, D = 2; cfg4:
N = 2e5, D = 1; cfg5: N = 5e5, D = 0) on a sample of targets.  The SE-vs-direct bound is the method's own
discretisation error at the configs' parameters (eps = 1e-8 class), not a
rounding bound; the device-vs-reference bound is rounding.
"""

import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN

import paper_1712_04732_b200 as se
from paper_1712_04732_b200 import direct

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLDEN, "direct.npz"))


@pytest.mark.parametrize("i", [0, 1])
def test_direct_3p_matches_reference(gold, i):
    N, L, xi, kmax, _ = gold[f"d3_{i}_in"]
    s = se.ParticleSystem(gold[f"d3_{i}_pos"], gold[f"d3_{i}_q"], L)
    phi = direct.kspace_direct_3p(s, xi, int(kmax))
    ref = gold[f"d3_{i}_phi"]
    assert se.relative_rms_error(phi, ref) < 1e-12
    sub = np.array([5, 0, 11])
    assert np.allclose(direct.kspace_direct_3p(s, xi, int(kmax), targets=sub), ref[sub], rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("i", [0, 1])
def test_direct_2p_matches_reference(gold, i):
    N, L, xi, kmax, _ = gold[f"d2_{i}_in"]
    s = se.ParticleSystem(gold[f"d2_{i}_pos"], gold[f"d2_{i}_q"], L)
    ref = gold[f"d2_{i}_phi"]
    assert se.relative_rms_error(direct.kspace_direct_2p(s, xi, int(kmax)), ref) < 1e-12
    sub = np.array([4, 0])
    assert np.allclose(direct.kspace_direct(s, xi, se.Periodicity(2), int(kmax), targets=sub), ref[sub],
                       rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("i", [0, 1])
def test_direct_1p_matches_reference(gold, i):
    N, L, xi, kmax, _ = gold[f"d1_{i}_in"]
    s = se.ParticleSystem(gold[f"d1_{i}_pos"], gold[f"d1_{i}_q"], L)
    ref = gold[f"d1_{i}_phi"]
    err = se.relative_rms_error(direct.kspace_direct_1p(s, xi, int(kmax)), ref)
    print(f"1p vs reference oracle: {err:.2e}")
    assert err < 1e-12
    sub = np.array([2, 7])
    assert np.allclose(direct.kspace_direct(s, xi, se.Periodicity(1), int(kmax), targets=sub), ref[sub],
                       rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("i", [0, 1])
def test_direct_0p_matches_reference(gold, i):
    N, L, xi, _ = gold[f"d0_{i}_in"]
    s = se.ParticleSystem(gold[f"d0_{i}_pos"], gold[f"d0_{i}_q"], L)
    phi = direct.kspace_direct_0p(s, xi)
    ref = gold[f"d0_{i}_phi"]
    assert se.relative_rms_error(phi, ref) < 1e-13
    sub = np.array([3, 1])
    assert np.allclose(direct.kspace_direct_0p(s, xi, targets=sub), ref[sub], rtol=1e-13, atol=1e-14)
    assert direct.kspace_direct(s, xi, se.Periodicity(0), 0, targets=sub).shape == (2,)


def test_direct_errors():
    s = se.ParticleSystem(np.array([[0.2, 0.2, 0.2], [0.2, 0.2, 0.2], [0.5, 0.5, 0.5]]),
                          np.array([1.0, -0.5, -0.5]), 1.0)
    with pytest.raises(se.SingularConfigurationError):
        direct.kspace_direct_0p(s, 3.0)
    ok = se.ParticleSystem(np.array([[0.2, 0.2, 0.2], [0.5, 0.5, 0.5]]), np.array([1.0, -1.0]), 1.0)
    with pytest.raises(ValueError):
        direct.kspace_direct_3p(ok, 3.0, 0)
    with pytest.raises(ValueError):
        direct.kspace_direct_3p(ok, 3.0, 4, targets=[0, 2])
    shared = se.ParticleSystem(np.array([[0.2, 0.3, 0.4], [0.7, 0.3, 0.4], [0.5, 0.5, 0.5]]),
                               np.array([1.0, -0.5, -0.5]), 1.0)
    with pytest.raises(se.SingularConfigurationError):  # same transverse coordinates (D = 1)
        direct.kspace_direct_1p(shared, 3.0, 4)


def test_se_kspace_vs_direct_small_all_periodicities_d3_d0():
    # SE with tight parameters == direct sum (the reference's
    # test_sekspace.py:177-192 property, N = 20, all of D = 3, 0)
    rng = np.random.default_rng(5)
    pos = rng.random((20, 3))
    q = rng.uniform(-1, 1, 20)
    q -= q.mean()
    s = se.ParticleSystem(pos, q, 1.0)
    p3, _ = se.auto_params(s, se.Periodicity(3), 6.3, 1e-14)
    ref3 = direct.kspace_direct_3p(s, 6.3, direct.OracleConfig.for_accuracy(6.3, 1.0, 1e-14).kmax)
    assert se.relative_rms_error(se.se_kspace(s, p3, se.Periodicity(3)), ref3) < 1e-11
    p0, _ = se.auto_params(s, se.Periodicity(0), 6.3, 1e-14)
    assert se.relative_rms_error(se.se_kspace(s, p0, se.Periodicity(0)), direct.kspace_direct_0p(s, 6.3)) < 1e-11


def test_cfg2_full_size_kspace_vs_direct_sum():
    import workloads

    w = workloads.ALL["cfg2"]()
    p = se.SEParams(**w["prm"])
    s = se.ParticleSystem(w["pos"], w["q"], w["L"])
    phik = se.se_kspace(s, p, se.Periodicity(3))
    sel = np.random.default_rng(11).choice(s.N, 256, replace=False)
    kmax = direct.OracleConfig.for_accuracy(p.xi, s.L, 1e-14).kmax
    ref = direct.kspace_direct_3p(s, p.xi, kmax, targets=sel)
    err = se.relative_rms_error(phik[sel], ref)
    print(f"cfg2 SE k-space vs direct sum (kmax={kmax}): rel RMS {err:.3e}")
    # ES P=8 at M=128: the window / aliasing error of the eps = 1e-8 class
    # (measured 2.35e-8; the reference's own P=8 sweep fixture shows 1.4e-8)
    assert err < 7e-8


@pytest.mark.parametrize("name", ["cfg1_tol", "cfg2_tol"])
def test_tol_variants_d3_meet_requested_tolerance(name):
    # the tolerance-meeting parameter sets (tools/workloads.py) against the
    # direct Ewald Fourier sum at full size: the REQUESTED eps is the bound
    import workloads

    w = workloads.ALL[name]()
    p = se.SEParams(**w["prm"])
    s = se.ParticleSystem(w["pos"], w["q"], w["L"])
    phik = se.se_kspace(s, p, se.Periodicity(3))
    sel = np.random.default_rng(11).choice(s.N, min(s.N, 256), replace=False)
    kmax = direct.OracleConfig.for_accuracy(p.xi, s.L, 1e-14).kmax
    ref = direct.kspace_direct_3p(s, p.xi, kmax, targets=sel)
    err = se.relative_rms_error(phik[sel], ref)
    print(f"{name} SE k-space vs direct sum (kmax={kmax}): rel RMS {err:.3e} (requested {p.eps:.0e})")
    assert err <= p.eps


def test_cfg1_tol_total_meets_tolerance_vs_converged():
    # the total potential (real space + k-space + self) against a converged SE
    # evaluation (auto_params at eps = 1e-14, xi-invariant to ~1e-13): the
    # metric's "at rms tol 1e-8" for the whole potential, not only its Fourier part
    import workloads

    w = workloads.ALL["cfg1_tol"]()
    s = se.ParticleSystem(w["pos"], w["q"], w["L"])
    p = se.SEParams(**w["prm"])
    tight, _ = se.auto_params(s, se.Periodicity(3), 14.31, 1e-14)
    err = se.relative_rms_error(se.total_potential(s, p, se.Periodicity(3)),
                                se.total_potential(s, tight, se.Periodicity(3)))
    print(f"cfg1_tol total vs converged: {err:.3e}")
    assert err <= 1e-8  # measured with the reference itself: 3.7e-9


def test_cfg3_full_size_kspace_vs_direct_sum():
    # D = 2 at full size (N = 2e5): the tolerance-meeting parameter set (P = 10,
    # s0 = s = 4, nI = 48; 8.6e-10 on a probe) against the
    # closed-form doubly periodic direct sum at sampled targets
    import workloads

    w = workloads.ALL["cfg3_tol"]()
    p = se.SEParams(**w["prm"])
    s = se.ParticleSystem(w["pos"], w["q"], w["L"])
    phik = se.se_kspace(s, p, se.Periodicity(2))
    sel = np.random.default_rng(13).choice(s.N, 48, replace=False)
    kmax = direct.OracleConfig.for_accuracy(p.xi, s.L, 1e-13).kmax
    ref = direct.kspace_direct_2p(s, p.xi, kmax, targets=sel)
    err = se.relative_rms_error(phik[sel], ref)
    print(f"cfg3_tol SE k-space vs direct 2p sum (kmax={kmax}): rel RMS {err:.3e}")
    assert err < 1e-9  # measured 2.5e-10


def test_cfg4_full_size_kspace_vs_direct_sum():
    # D = 1 at full size (N = 2e5, cubic embedding L = 8): incomplete-Bessel
    # direct sum at sampled targets
    import workloads

    w = workloads.ALL["cfg4"]()
    p = se.SEParams(**w["prm"])
    s = se.ParticleSystem(w["pos"], w["q"], w["L"])
    phik = se.se_kspace(s, p, se.Periodicity(1))
    sel = np.random.default_rng(14).choice(s.N, 24, replace=False)
    kmax = direct.OracleConfig.for_accuracy(p.xi, s.L, 1e-13).kmax
    ref = direct.kspace_direct_1p(s, p.xi, kmax, targets=sel)
    err = se.relative_rms_error(phik[sel], ref)
    print(f"cfg4 SE k-space vs direct 1p sum (kmax={kmax}): rel RMS {err:.3e}")
    # measured 3.5e-8: the Gaussian P = 12 window limits this parameter set
    # (cfg4_tol below widens it to P = 16)
    assert err < 1e-7


def test_cfg4_tol_full_size_kspace_vs_direct_sum():
    # the tolerance-meeting D = 1 set: Gaussian P = 16 (tools/workloads.py;
    # probe with the reference: 4.6e-10) against the requested 1e-9
    import workloads

    w = workloads.ALL["cfg4_tol"]()
    p = se.SEParams(**w["prm"])
    s = se.ParticleSystem(w["pos"], w["q"], w["L"])
    phik = se.se_kspace(s, p, se.Periodicity(1))
    sel = np.random.default_rng(14).choice(s.N, 24, replace=False)
    kmax = direct.OracleConfig.for_accuracy(p.xi, s.L, 1e-13).kmax
    ref = direct.kspace_direct_1p(s, p.xi, kmax, targets=sel)
    err = se.relative_rms_error(phik[sel], ref)
    print(f"cfg4_tol SE k-space vs direct 1p sum (kmax={kmax}): rel RMS {err:.3e}")
    assert err <= p.eps


def test_cfg5_full_size_kspace_vs_direct_sum():
    import workloads

    w = workloads.ALL["cfg5"]()
    p = se.SEParams(**w["prm"])
    s = se.ParticleSystem(w["pos"], w["q"], w["L"])
    phik = se.se_kspace(s, p, se.Periodicity(0))
    sel = np.random.default_rng(12).choice(s.N, 512, replace=False)
    ref = direct.kspace_direct_0p(s, p.xi, targets=sel)
    err = se.relative_rms_error(phik[sel], ref)
    print(f"cfg5 SE k-space vs direct erf sum: rel RMS {err:.3e}")
    assert err < 1e-9  # measured 1.0e-10
