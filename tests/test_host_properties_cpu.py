"""Analytic properties of the host-side planning routines (CPU, no GPU).

The windows, truncated Green's functions, parameter selectors and core
helpers of the package are exercised against closed forms and limits the
method defines (the same invariants the reference's own test files check for
pmewald.windows / greens / params / core), evaluated through the library's
planning entry points.  Expected values are derived here from the formulas
of arXiv 1712.04732, not from reference outputs (those are covered by
tests/golden and test_host_cpu.py).
"""

import math
import warnings

import numpy as np
import pytest

import paper_1712_04732_b200 as se
from paper_1712_04732_b200 import greens, params as pm, windows
from paper_1712_04732_b200.core import ConfigurationError, Periodicity
from paper_1712_04732_b200.greens import GreensSpec, greens_hat, zero_mode_values, zero_point_value
from paper_1712_04732_b200.windows import WindowSpec


def _spec(kind, P=16, h=1.0 / 28, shape=None):
    return WindowSpec(kind, P, h, windows.default_shape(kind, P) if shape is None else shape)


def _i0(x):
    # modified Bessel I0 by its (positive-term) power series
    s, t, k = 1.0, 1.0, 0
    while t > 1e-18 * s:
        k += 1
        t *= (0.5 * x) ** 2 / (k * k)
        s += t
    return s


# --------------------------------------------------------------- Gaussian

def test_gaussian_peak_and_edge():
    sp = _spec("gaussian", P=12)
    xi = 4.7
    eta = sp.eta(xi)
    peak = float(windows.eval_gaussian(0.0, sp))
    assert peak == pytest.approx(math.sqrt(2.0 * xi * xi / (math.pi * eta)), rel=1e-14)
    edge = float(windows.eval_gaussian(sp.w, sp))
    assert edge / peak == pytest.approx(math.exp(-0.5 * sp.shape ** 2), rel=1e-12)
    assert windows.eval_gaussian(sp.w * (1 + 1e-9), sp) == 0.0
    assert windows.eval_gaussian(-3.0 * sp.w, sp) == 0.0


def test_gaussian_transform_dc_symmetry_and_decay_scale():
    sp = _spec("gaussian")
    assert windows.gaussian_fourier(0.0, sp) == 1.0
    k = np.linspace(-55.0, 55.0, 23)
    v = windows.gaussian_fourier(k, sp)
    assert np.array_equal(v, v[::-1])
    xi = 3.1
    k1 = 2.0 * xi * math.sqrt(2.0 / sp.eta(xi))   # eta k^2 / (8 xi^2) = 1
    assert float(windows.gaussian_fourier(k1, sp)) == pytest.approx(math.exp(-1.0), rel=1e-13)


def test_gaussian_transform_is_integral_of_window():
    # the truncated window integrates to ~1 (the transform at k=0 of the
    # untruncated Gaussian); the truncation tail is erfc(m/sqrt 2)
    sp = _spec("gaussian", P=16)
    x = np.linspace(-sp.w, sp.w, 40001)
    mass = np.trapezoid(windows.eval_gaussian(x, sp), x)
    assert mass == pytest.approx(1.0 - math.erfc(sp.shape / math.sqrt(2.0)), rel=1e-8)


# --------------------------------------------------------------- B-spline

def test_bspline_hat_and_partition_of_unity():
    assert windows.eval_bspline(1.0, 2) == 1.0
    assert windows.eval_bspline(0.0, 2) == 0.0 and windows.eval_bspline(2.0, 2) == 0.0
    with pytest.raises(ValueError):
        windows.eval_bspline(0.5, 1)
    for p in (3, 4, 6, 9):
        for x in (0.3, 0.77):
            total = sum(windows.eval_bspline(x - j, p) for j in range(-p - 2, p + 3))
            assert total == pytest.approx(1.0, abs=1e-13)
    # M_4 at its center is 2/3
    assert windows.eval_bspline(2.0, 4) == pytest.approx(2.0 / 3.0, rel=1e-15)
    xs = np.linspace(-1, 7, 33)
    assert np.allclose(windows.eval_bspline(xs, 6), windows.eval_bspline(6.0 - xs, 6), atol=1e-15)


# --------------------------------------------------------------- Kaiser-Bessel

def test_kaiser_center_edge_support():
    sp = _spec("kb", P=12)
    assert float(windows.eval_kaiser(0.0, sp)) == pytest.approx(1.0, rel=1e-14)
    assert float(windows.eval_kaiser(sp.w, sp)) == pytest.approx(1.0 / _i0(sp.shape), rel=1e-12)
    assert windows.eval_kaiser(-sp.w, sp) == windows.eval_kaiser(sp.w, sp)
    assert windows.eval_kaiser(1.001 * sp.w, sp) == 0.0


def test_kaiser_transform_dc_and_quadrature():
    sp = _spec("kb", P=8)
    beta, w = sp.shape, sp.w
    assert float(windows.kaiser_fourier(0.0, sp)) == pytest.approx(
        2.0 * w * math.sinh(beta) / (beta * _i0(beta)), rel=1e-13)
    x = np.linspace(-w, w, 40001)
    f = windows.eval_kaiser(x, sp)
    for k in (0.9, 23.0, 1.6 * beta / w):   # both sides of the sinh/sin seam
        num = np.trapezoid(f * np.cos(k * x), x)
        assert float(windows.kaiser_fourier(k, sp)) == pytest.approx(num, rel=1e-7)


def test_kaiser_transform_continuous_at_seam():
    sp = WindowSpec("kb", 4, 0.05, 0.1)
    k0 = sp.shape / sp.w
    lo, hi = windows.kaiser_fourier(np.array([k0 * (1 - 1e-6), k0 * (1 + 1e-6)]), sp)
    assert abs(lo - hi) < 1e-8 * abs(lo)


def test_sinhc_series_branch_agrees_with_closed_forms():
    r2 = np.array([0.999e-6, -0.999e-6, 0.4e-6, -0.4e-6, 3e-6, -3e-6])
    got = windows._sinhc(r2)
    want = np.where(r2 > 0, np.sinh(np.sqrt(np.abs(r2))) / np.sqrt(np.abs(r2)),
                    np.sin(np.sqrt(np.abs(r2))) / np.sqrt(np.abs(r2)))
    assert np.max(np.abs(got - want) / np.abs(want)) < 1e-13
    assert float(windows._sinhc(0.0)) == 1.0


# --------------------------------------------------------------- BM (ES)

def test_bm_center_edge_and_evenness():
    sp = _spec("bm", P=10)
    assert windows.eval_bm(0.0, sp) == 1.0
    assert float(windows.eval_bm(sp.w, sp)) == pytest.approx(math.exp(-sp.shape), rel=1e-12)
    assert windows.eval_bm(1.0001 * sp.w, sp) == 0.0
    x = np.linspace(0.0, sp.w, 37)
    assert np.array_equal(windows.eval_bm(x, sp), windows.eval_bm(-x, sp))


def test_bm_larger_beta_is_lower():
    w, x = 4.0, 1.7
    vals = [float(windows.eval_bm(x, WindowSpec("bm", 8, w / 4.0, b))) for b in (1.0, 4.0, 9.0, 20.0, 33.0)]
    assert all(a > b for a, b in zip(vals, vals[1:]))
    assert vals[2] == pytest.approx(math.exp(9.0 * (math.sqrt(1.0 - (x / w) ** 2) - 1.0)), rel=1e-14)


def test_bm_transform_box_limit():
    sp = WindowSpec("bm", 6, 1.0 / 12, 1e-12)
    k = np.linspace(0.3, 70.0, 31)
    t = windows.bm_fourier_precompute(sp, k)
    assert np.allclose(t.values, 2.0 * np.sin(k * sp.w) / k, rtol=1e-9, atol=1e-15)


def test_bm_transform_dc_is_mass_and_matches_quadrature():
    sp = _spec("bm", P=12, shape=30.0)
    x = np.linspace(-sp.w, sp.w, 2 ** 16 + 1)
    mass = (x[1] - x[0]) * np.sum(windows.eval_bm(x, sp))
    assert windows.bm_fourier_precompute(sp, np.array([0.0])).values[0] == pytest.approx(mass, rel=1e-9)
    k = np.array([3.0, 41.0, 180.0])
    f = windows.eval_bm(x, sp)
    num = np.array([np.trapezoid(f * np.cos(kk * x), x) for kk in k])
    assert np.allclose(windows.fourier(k, sp), num, rtol=1e-7, atol=1e-12 * mass)


def test_bm_quadrature_node_doubling_converges():
    sp = _spec("bm", P=16, shape=40.0)
    k = 2.0 * np.pi * np.fft.fftfreq(88, d=1.0 / 28)
    a = windows._bm_quadrature(sp.w, sp.shape, k, 200)
    b = windows._bm_quadrature(sp.w, sp.shape, k, 400)
    assert np.max(np.abs(a - b)) < 1e-14 * np.max(np.abs(b))


def test_bm_table_cached_even_and_real():
    sp = _spec("bm", P=12)
    k = 2.0 * np.pi * np.fft.fftfreq(64, d=1.0 / 28)
    t1 = windows.bm_fourier_precompute(sp, k)
    assert windows.bm_fourier_precompute(sp, k.copy()) is t1
    assert t1.values.dtype == np.float64 and t1.kind == "bm" and t1.w == sp.w
    lookup = dict(zip(np.round(k, 12), t1.values))
    peak = np.max(np.abs(t1.values))
    for kk, v in lookup.items():
        if -kk in lookup:
            assert abs(v - lookup[-kk]) < 1e-13 * peak
    with pytest.raises(ValueError):
        windows.bm_fourier_precompute(_spec("kb"), k)


def test_default_shapes():
    assert windows.default_shape("bm", 10) == 25.0
    assert windows.default_shape("kb", 6) == 15.0
    assert windows.default_shape("gaussian", 9) == pytest.approx(math.sqrt(9 * math.pi), rel=1e-15)
    with pytest.raises(ValueError):
        windows.default_shape("box", 8)


# --------------------------------------------------------------- Green's functions

def test_d3_kernel():
    assert greens_hat(np.zeros(3), GreensSpec(3)) == 0.0
    k = np.array([1.5, -2.0, 0.25])
    assert greens_hat(k, GreensSpec(3)) == pytest.approx(1.0 / (k @ k), rel=1e-15)


def test_d0_kernel_closed_form_null_and_zero():
    R = 1.9
    assert greens_hat(np.zeros(3), GreensSpec(0, R)) == pytest.approx(0.5 * R * R, rel=1e-15)
    assert abs(greens_hat(np.array([0.0, 0.0, 2 * math.pi / R]), GreensSpec(0, R))) < 1e-15
    for kap in (0.4, 6.0, 47.0):
        want = 2.0 * (math.sin(0.5 * R * kap) / kap) ** 2     # (1 - cos(R k)) / k^2
        assert greens_hat(np.array([kap, 0.0, 0.0]), GreensSpec(0, R)) == pytest.approx(want, rel=1e-13)


def test_d1_kernel_against_bessel_series():
    def j(nu, t):
        s, term, m = 0.0, (0.5 * t) ** nu / math.factorial(nu), 0
        while True:
            s += term
            m += 1
            term *= -(0.25 * t * t) / (m * (m + nu))
            if abs(term) < 1e-30:
                return s
    for R, kap in ((1.0, 3.0), (1.7, 2.2), (0.8, 11.0)):
        t = R * kap
        want = (1.0 - j(0, t)) / kap ** 2 - R * math.log(R) * j(1, t) / kap
        got = greens_hat(np.array([0.0, 0.0, kap]), GreensSpec(1, R))
        assert got == pytest.approx(want, rel=1e-12)
    R = 2.2
    assert greens_hat(np.zeros(3), GreensSpec(1, R)) == pytest.approx(R * R * (1 - 2 * math.log(R)) / 4, rel=1e-14)


def test_d2_kernel_small_and_large_argument():
    R = 1.3
    kap = 2e-4 / R
    t = R * kap
    got = greens_hat(np.array([0.0, 0.0, kap]), GreensSpec(2, R))
    assert got == pytest.approx(R * R * (-0.5 + t * t / 8 - t ** 4 / 144), rel=1e-12)
    kap = 5.9
    t = R * kap
    want = (1.0 - math.cos(t) - t * math.sin(t)) / kap ** 2
    assert greens_hat(np.array([0.0, 0.0, kap]), GreensSpec(2, R)) == pytest.approx(want, rel=1e-13)


@pytest.mark.parametrize("D", [0, 1, 2])
def test_zero_mode_continuous_at_origin_and_series_seam(D):
    R = 1.4
    kv = np.zeros(3)
    kv[2] = 1e-6 / R
    v0 = zero_point_value(D, R)
    assert abs(greens_hat(kv, GreensSpec(D, R)) - v0) < 1e-9 * abs(v0)
    # across the t = 1e-2 switch between the series and the closed form the
    # change must match the leading Taylor slope (d/d(t^2) of the kernel)
    slope = {0: -1.0 / 24.0, 1: -(1.0 / 64.0 - math.log(1.0) / 16.0), 2: 1.0 / 8.0}[D]
    Rn = 1.0
    a, b = zero_mode_values(D, Rn, np.array([0.99e-2, 1.01e-2]))
    assert abs((b - a) - slope * (1.01e-2 ** 2 - 0.99e-2 ** 2)) < 1e-10 * abs(b)


def test_periodic_modes_use_inverse_square_and_free_block_is_radial():
    R = 1.1
    k = np.array([2 * math.pi, 0.4, -0.9])
    for D in (1, 2):
        assert greens_hat(k, GreensSpec(D, R)) == pytest.approx(1.0 / (k @ k), rel=1e-15)
    a = greens_hat(np.array([0.0, 0.6, 0.8]), GreensSpec(1, R))
    b = greens_hat(np.array([0.0, 0.0, 1.0]), GreensSpec(1, R))
    assert a == pytest.approx(b, rel=1e-13)
    a = greens_hat(np.array([0.3, 0.4, 1.2]), GreensSpec(0, R))
    b = greens_hat(np.array([1.3, 0.0, 0.0]), GreensSpec(0, R))
    assert a == pytest.approx(b, rel=1e-13)


def test_default_truncation_radius_and_spec_validation():
    assert greens.default_truncation_radius(0, 2.0) == pytest.approx(2.0 * math.sqrt(3))
    assert greens.default_truncation_radius(1, 2.0) == pytest.approx(2.0 * math.sqrt(2))
    assert greens.default_truncation_radius(3, 2.0) == 0.0
    with pytest.raises(ValueError):
        GreensSpec(1, 0.0)
    with pytest.raises(ValueError):
        zero_mode_values(3, 1.0, [1.0])


def test_d0_kernel_reconstructs_coulomb_inside_ball():
    # radial inverse transform of the truncated kernel, band-limited at K:
    # G(r) = (1/(2 pi^2 r)) int_0^K k Ghat(k) sin(k r) dk = 1/(4 pi r) for r < R
    R = 2.0
    K, dk = 4.0e6, 0.1
    r = np.array([0.15, 0.4, 0.7]) * R
    acc = np.zeros_like(r)
    n = int(K / dk)
    for lo in range(0, n, 1_000_000):
        k = (np.arange(lo, min(lo + 1_000_000, n)) + 0.5) * dk
        acc += (k * zero_mode_values(0, R, k)) @ np.sin(np.outer(k, r))
    recon = acc * dk / (2 * math.pi ** 2 * r)
    assert np.max(np.abs(recon * 4 * math.pi * r - 1.0)) < 2e-6


# --------------------------------------------------------------- parameter selection

def test_select_cutoff():
    e16 = math.exp(-16.0)
    assert pm.select_cutoff(1.0, e16) == pytest.approx(4.0, rel=1e-14)
    assert pm.select_cutoff(4.0, e16) == pytest.approx(1.0, rel=1e-14)
    with pytest.warns(UserWarning):
        pm.select_cutoff(1.0, 1e-10, L=2.0)
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        pm.select_cutoff(10.0, 1e-10, L=2.0)
    for bad in (0.0, 1.0, 2.0, -1e-3):
        with pytest.raises(ValueError):
            pm.select_cutoff(1.0, bad)


def test_select_kinf():
    assert pm.select_kinf(math.pi, 1.0, math.exp(-16.0)) == (4, 8)
    kinf, M = pm.select_kinf(math.pi, 2.0, math.exp(-9.0))    # ceil(2*3) = 6 -> M = 12
    assert (kinf, M) == (6, 12)
    assert [pm.select_kinf(xi, 1.0, 1e-8)[0] for xi in (1.0, 3.0, 9.0)] == sorted(
        pm.select_kinf(xi, 1.0, 1e-8)[0] for xi in (1.0, 3.0, 9.0))
    for xi in (2.0, 5.5, 13.0):
        kinf, M = pm.select_kinf(xi, 1.0, 1e-10)
        assert M >= 2 * kinf and M % 2 == 0
        f = M
        for p in (2, 3, 5, 7):
            while f % p == 0:
                f //= p
        assert f == 1


def test_select_P_and_upsampling():
    assert pm.select_P("bm", 0.5, 1.0) == 1
    # smallest P with e^{-sqrt(2 pi) P} <= eps
    eps = 1e-10
    P = pm.select_P("bm", eps, 1.0)
    assert math.exp(-math.sqrt(2 * math.pi) * P) <= eps < math.exp(-math.sqrt(2 * math.pi) * (P - 1))
    Pg = pm.select_P("gaussian", eps, 1.0)
    assert math.exp(-math.pi / 2 * Pg) <= eps < math.exp(-math.pi / 2 * (Pg - 1))
    assert [pm.select_P("kb", e, 1.0) for e in (1e-3, 1e-7, 1e-11)] == sorted(
        pm.select_P("kb", e, 1.0) for e in (1e-3, 1e-7, 1e-11))
    assert pm.select_upsampling(3, 1e-6, 30) == (1.0, 1.0, 15)
    s0, s, nI = pm.select_upsampling(0, 1e-6, 30)
    assert (s0, s, nI) == (pytest.approx(1 + math.sqrt(3)), 1.0, 15)
    s0, s, nI = pm.select_upsampling(1, 1e-10, 64)
    assert s0 == pytest.approx(1 + math.sqrt(2)) and nI == 7
    assert s == pytest.approx(math.log(1e10) / (2 * math.pi), rel=1e-12)
    assert pm.select_upsampling(2, 0.5, 64)[1] == 1.0


def test_estimate_approx_error_shapes():
    for P in (6, 10, 14):
        m = math.sqrt(math.pi * P)
        est = pm.estimate_approx_error("gaussian", P, m)
        assert est == pytest.approx(math.exp(-math.pi * P / 2) + math.erfc(m / math.sqrt(2)), rel=1e-14)
        betas = np.linspace(0.5 * P, 5.0 * P, 300)
        vals = np.array([pm.estimate_approx_error("bm", P, b) for b in betas])
        i = int(np.argmin(vals))
        assert 0 < i < len(betas) - 1
        assert 0.6 * 2.5 * P < betas[i] < 1.1 * 2.5 * P
    with pytest.raises(ValueError):
        pm.estimate_approx_error("bm", 8, 0.0)


def test_auto_params_structure():
    s = se.generate_random_system(40, 1.0, seed=3)
    for D in (0, 1, 2, 3):
        for window in ("bm", "gaussian", "kb"):
            prm, budget = pm.auto_params(s, Periodicity(D), 6.0, 1e-8, window=window)
            assert (prm.M + prm.P) % 2 == 0 and prm.P <= prm.M
            assert budget.contributions["approximation"] <= 1e-8
            assert budget.contributions["real_truncation"] == pytest.approx(1e-8, rel=1e-12)
            if D == 3:
                assert prm.R == 0.0 and prm.s0 == 1.0
            else:
                assert prm.R > 0.0 and prm.s0 > 1.0
            if D in (1, 2):
                assert 1 <= prm.nI <= prm.M // 2


def test_auto_params_rejects_window_wider_than_grid():
    s = se.generate_random_system(10, 1.0, seed=1)
    with pytest.raises(ConfigurationError):
        pm.auto_params(s, Periodicity(3), 1.0, 1e-12, window="gaussian")


def test_amplitude():
    s = se.generate_random_system(64, 3.0, seed=9)
    Q = float(np.sum(s.charges ** 2))
    assert pm.amplitude(s, 2.5) == pytest.approx(math.sqrt(Q * 2.5 * 3.0) / 3.0, rel=1e-14)


# --------------------------------------------------------------- core helpers

def test_random_system_generation():
    s = se.generate_random_system(2, 1.0, seed=0)
    assert np.array_equal(s.charges, [1.0, -1.0])
    a = se.generate_random_system(51, 2.0, seed=7)
    b = se.generate_random_system(51, 2.0, seed=7)
    assert np.array_equal(a.positions, b.positions) and np.array_equal(a.charges, b.charges)
    assert abs(a.charges.sum()) < 1e-13 and a.is_neutral()
    assert a.positions.min() >= 0.0 and a.positions.max() < 2.0
    with pytest.raises(ValueError):
        se.generate_random_system(1, 1.0, seed=0)
    with pytest.raises(ValueError):
        se.ParticleSystem(np.array([[0.5, 0.5, 1.0]]), np.array([1.0]), 1.0)


def test_relative_rms_and_energy():
    ref = np.array([1.0, -2.0, 3.0, 0.5])
    assert se.relative_rms_error(ref, ref) == 0.0
    assert se.relative_rms_error(2 * ref, ref) == pytest.approx(1.0, rel=1e-15)
    x = ref + np.array([0.1, 0.0, -0.2, 0.3])
    want = math.sqrt(np.mean((x - ref) ** 2) / np.mean(ref ** 2))
    assert se.relative_rms_error(x, ref) == pytest.approx(want, rel=1e-14)
    with pytest.raises(ValueError):
        se.relative_rms_error(ref, np.zeros(4))
    with pytest.raises(ValueError):
        se.relative_rms_error(ref, ref[:3])
    s = se.generate_random_system(4, 1.0, seed=2)
    assert se.energy(s, np.zeros(4)) == 0.0
    assert se.energy(s, np.full(4, 3.7)) == pytest.approx(0.0, abs=1e-14)   # neutral
    phi = np.array([0.3, -1.0, 2.0, 0.25])
    assert se.energy(s, phi) == pytest.approx(float(s.charges @ phi), rel=1e-15)
    with pytest.raises(ValueError):
        se.energy(s, phi[:3])


def test_periodicity_axes():
    assert Periodicity(2).mask == (True, True, False)
    assert Periodicity(1).periodic_axes == (0,) and Periodicity(1).free_axes == (1, 2)
    assert Periodicity(0).periodic_axes == () and Periodicity(3).free_axes == ()
    with pytest.raises(ValueError):
        Periodicity(4)


# --------------------------------------------------------------- cell list / engine

def test_cell_list_buckets_every_particle_once():
    from paper_1712_04732_b200 import realspace
    s = se.generate_random_system(300, 2.0, seed=11)
    cl = realspace.build_cell_list(s, 0.35, Periodicity(3))
    n = cl.ncells[0]
    assert n == 5 and cl.edge >= cl.rc and cl.periodic_mask == (True, True, True)
    seen = np.sort(np.concatenate([m for m in cl.members if m.size]))
    assert np.array_equal(seen, np.arange(300))
    for c, m in enumerate(cl.members):
        assert np.all(np.diff(m) > 0)
        for i in m:
            idx = np.minimum((s.positions[i] / cl.edge).astype(int), n - 1)
            assert cl.flat(*idx) == c
    one = se.ParticleSystem(np.array([[0.5, 0.5, 0.5]]), np.array([1.0]), 1.0)
    occ = [m for m in realspace.build_cell_list(one, 0.3, Periodicity(0)).members if m.size]
    assert len(occ) == 1 and occ[0].tolist() == [0]
    with pytest.raises(ValueError):
        realspace.build_cell_list(s, 1.01, Periodicity(1))
    assert realspace.build_cell_list(s, 1.5, Periodicity(0)).ncells == (1, 1, 1)


def test_reference_engine_name_is_available():
    from paper_1712_04732_b200 import aft
    assert hasattr(aft.NumpyFftEngine(), "rfftn") and hasattr(aft.NumpyFftEngine(), "irfftn")


def test_run_record_csv_round_trip():
    import io

    from paper_1712_04732_b200 import records

    s = se.generate_random_system(30, 1.0, seed=4)
    for D in (3, 2, 0):
        prm, _ = pm.auto_params(s, Periodicity(D), 6.0, 1e-8)
        rec = records.make_record(s, prm, Periodicity(D), {"spread": 1e-3, "realspace": 2e-3}, 5e-3,
                                  seed=4, rms_vs_oracle=1.5e-9)
        assert list(rec) == records.CSV_COLUMNS
        buf = io.StringIO()
        records.write_records(buf, [rec], threads=8)
        text = buf.getvalue()
        assert text.startswith("# pmewald run ") and "# threads 8\n" in text
        row = records.read_records(io.StringIO(text))[0]
        assert int(row["D"]) == D and int(row["M"]) == prm.M and float(row["t_total"]) == 5e-3
        assert float(row["s0_eff"]) >= (1.0 if D == 3 else prm.s0 - 1e-12)
    with pytest.raises(RuntimeError):
        records.write_records(io.StringIO(), [{"command": "compute"}])
