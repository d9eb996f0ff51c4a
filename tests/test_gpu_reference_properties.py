"""The reference's stage-level properties (its test_sekspace / test_aft /
test_realspace / test_acceptance invariants) checked on the device path of
this package.  Expected values come from the method's definitions, the
device direct Ewald sums (pinned to the reference's oracle in
test_gpu_direct.py) or the stage identities themselves; no reference code is
used.
"""

import math

import numpy as np
import pytest

import paper_1712_04732_b200 as se
from paper_1712_04732_b200 import aft, direct, greens, sekspace, windows
from paper_1712_04732_b200.core import ParticleSystem, Periodicity, SEParams
from paper_1712_04732_b200.sekspace import Grid, GridField

pytestmark = pytest.mark.gpu


def params(D, L=1.0, M=28, P=16, xi=6.3, window="bm", shape=None, nI=None, eps=1e-13):
    """A tight parameter set in the style of the reference's tests."""
    h = L / M
    d = 3.0 - D
    rc = min(math.sqrt(-math.log(eps)) / xi, L)
    if D < 3:
        s0 = max(1.0 + math.sqrt(d), ((1.0 + math.sqrt(d)) * L + 2 * rc) / (L + P * h))
        R = 0.5 * (aft.padded_size(s0, M + P) * h - L + math.sqrt(d) * L)
    else:
        s0, R = 1.0, 0.0
    s = max(1.0, math.log(1.0 / eps) / (2 * math.pi)) if D in (1, 2) else 1.0
    nI = nI if nI is not None else (M // 2 if D in (1, 2) else 0)
    shape = windows.default_shape(window, P) if shape is None else shape
    return SEParams(xi=xi, rc=rc, M=M, P=P, window=window, shape=shape, s0=s0, s=s, nI=nI, R=R, eps=eps)


def rand_system(N, L, seed):
    rng = np.random.default_rng(seed)
    q = rng.uniform(-1, 1, N)
    return ParticleSystem(rng.random((N, 3)) * L, q - q.mean(), L)


# ---------------------------------------------------------------- spreading

def test_spread_empty_system_and_gather_zero_field():
    p = params(3, M=16, P=8)
    g = Grid.build(1.0, p, Periodicity(3))
    w = windows.WindowSpec("bm", 8, g.h, 20.0)
    empty = ParticleSystem(np.zeros((0, 3)), np.zeros(0), 1.0)
    assert not np.any(sekspace.spread(empty, w, g, Periodicity(3)).values)
    s = rand_system(5, 1.0, 3)
    assert not np.any(sekspace.gather(GridField(np.zeros(g.shape), g), s, w, Periodicity(3)))


def test_spread_touches_p_cubed_points():
    p = params(3, M=20, P=6, xi=5.0)
    g = Grid.build(1.0, p, Periodicity(3))
    w = windows.WindowSpec("bm", 6, g.h, 15.0)
    s = ParticleSystem(np.array([[0.311, 0.77, 0.132]]), np.array([1.0]), 1.0)
    assert np.count_nonzero(sekspace.spread(s, w, g, Periodicity(3)).values) == 6 ** 3


@pytest.mark.parametrize("D", [0, 1, 2, 3])
def test_spread_mass_identity(D):
    # h^3 sum H = sum_n q_n prod_axis (h sum_t w(x_t - x_n)): the separable
    # stencil weights summed per axis (stencil points: first = floor(u/h -
    # P/2) + 1, u = x + offset on free axes)
    p = params(D, M=18, P=8, xi=5.0)
    g = Grid.build(1.0, p, Periodicity(D))
    w = windows.WindowSpec("bm", 8, g.h, 20.0)
    s = rand_system(10, 1.0, 12 + D)
    H = sekspace.spread(s, w, g, Periodicity(D))
    rhs = 0.0
    for x, qn in zip(s.positions, s.charges):
        prod = 1.0
        for ax in range(3):
            u = x[ax] + (0.0 if ax < D else 0.5 * 8 * g.h)
            first = math.floor(u / g.h - 4) + 1
            pts = (np.arange(first, first + 8) * g.h) - u
            prod *= g.h * float(np.sum(windows.evaluate(pts, w)))
        rhs += qn * prod
    assert g.h ** 3 * H.values.sum() == pytest.approx(rhs, rel=1e-12, abs=1e-15)


def test_spread_rejects_window_wider_than_grid():
    # a grid whose window support P = 18 exceeds M = 16 (Grid fields: L, M, P,
    # D, h, Lt, Mt, R, g0, gs)
    g = Grid(1.0, 16, 18, 3, 1.0 / 16, 1.0 + 18 / 16, 34, 0.0, 16, 34)
    w = windows.WindowSpec("bm", 18, g.h, 45.0)
    with pytest.raises(ValueError):
        sekspace.spread(rand_system(3, 1.0, 0), w, g, Periodicity(3))


# ---------------------------------------------------------------- scaling

def test_scale_d3_zero_mode_zero_and_single_mode_constant():
    L, M, P, xi = 2.0, 8, 4, 3.0
    p = SEParams(xi=xi, rc=0.5, M=M, P=P, window="bm", shape=10.0, eps=1e-6)
    g = Grid.build(L, p, Periodicity(3))
    w = windows.WindowSpec("bm", P, g.h, 10.0)
    F = aft.aft_forward(np.random.default_rng(1).normal(size=(M, M, M)), None, 1.0, 1.0, Periodicity(3))
    out = sekspace.scale(F, xi, w, greens.GreensSpec(3), g, Periodicity(3))
    assert out.full[0, 0, 0] == 0.0
    # impulse at k = (2 pi / L, 0, 0): multiplier 4 pi e^{-k^2/4xi^2} / (k^2 (w(k) w(0)^2)^2)
    F = aft.SpectralField(3, M, M, M, M, full=np.zeros((M, M, M), dtype=complex))
    F.full[1, 0, 0] = 1.0
    out = sekspace.scale(F, xi, w, greens.GreensSpec(3), g, Periodicity(3))
    k = 2 * math.pi / L
    wk = float(windows.fourier(np.array([k]), w)[0] * windows.fourier(np.array([0.0]), w)[0] ** 2)
    assert out.full[1, 0, 0].real == pytest.approx(4 * math.pi * math.exp(-k * k / (4 * xi * xi)) / (k * k * wk ** 2),
                                                  rel=1e-13)
    assert np.count_nonzero(out.full) == 1


def test_scale_zero_spectrum_mixed():
    p = params(2, M=8, P=4, xi=5.0, eps=1e-6)
    g = Grid.build(1.0, p, Periodicity(2))
    part = aft.ModePartition.build(8, 2, 2)
    F = aft.aft_forward(np.zeros(g.shape), part, p.s0, p.s, Periodicity(2))
    out = sekspace.scale(F, p.xi, windows.WindowSpec("bm", 4, g.h, 10.0), greens.GreensSpec(2, p.R), g,
                         Periodicity(2))
    assert not np.any(out.zero) and not np.any(out.Iblk) and not np.any(out.Jblk)


# ---------------------------------------------------------------- pipeline

@pytest.mark.parametrize("D", [0, 1, 2, 3])
def test_se_kspace_tight_params_equal_direct_sum(D):
    s = rand_system(20, 1.0, 3)
    p = params(D, nI=8 if D in (1, 2) else None)
    ref = direct.kspace_direct(s, p.xi, Periodicity(D), 16)
    assert se.relative_rms_error(sekspace.se_kspace(s, p, Periodicity(D)), ref) < 2e-13


def test_se_kspace_off_unit_box_pins_constants():
    s = rand_system(16, 2.0, 19)
    p = params(3, L=2.0, M=32, P=14, xi=4.0)
    ref = direct.kspace_direct_3p(s, 4.0, 18)
    assert se.relative_rms_error(sekspace.se_kspace(s, p, Periodicity(3)), ref) < 1e-12


def test_mirror_dipole_antisymmetry_and_permutation_invariance():
    s = ParticleSystem(np.array([[0.25, 0.5, 0.5], [0.75, 0.5, 0.5]]), np.array([1.0, -1.0]), 1.0)
    phi = sekspace.se_kspace(s, params(3), Periodicity(3))
    assert phi[0] == pytest.approx(-phi[1], rel=1e-12)
    s = rand_system(12, 1.0, 4)
    perm = np.random.default_rng(0).permutation(12)
    sp = ParticleSystem(s.positions[perm], s.charges[perm], 1.0)
    p = params(2, nI=8)
    a = sekspace.se_kspace(s, p, Periodicity(2))
    b = sekspace.se_kspace(sp, p, Periodicity(2))
    assert np.allclose(a[perm], b, rtol=1e-12, atol=1e-14)


def test_exponential_convergence_in_P():
    # BM at beta = 2.5 P: successive errors fall by ~e^{-sqrt(2 pi) dP}
    s = rand_system(20, 1.0, 3)
    ref = direct.kspace_direct_3p(s, 6.3, 16)
    errs = [se.relative_rms_error(sekspace.se_kspace(s, params(3, P=P), Periodicity(3)), ref) for P in (4, 6, 8, 10)]
    predicted = math.exp(-math.sqrt(2 * math.pi) * 2)
    for e1, e2 in zip(errs, errs[1:]):
        assert e2 < e1
        assert 0.2 * predicted < e2 / e1 < 5.0 * predicted


def test_precompute_kernel_requires_minimum_upsampling_and_is_cached():
    with pytest.raises(ValueError):
        sekspace.precompute_truncated_greens(1.0, 16, 8, 2.0, rc=0.5)
    k1 = sekspace.precompute_truncated_greens(1.0, 16, 8, 1.0 + math.sqrt(3.0), rc=0.5)
    k2 = sekspace.precompute_truncated_greens(1.0, 16, 8, 1.0 + math.sqrt(3.0), rc=0.5)
    assert k1 is k2
    assert np.all(np.isfinite(k1.ghat)) and k1.ghat.dtype == np.float64


def test_unknown_window_rejected():
    s = rand_system(4, 1.0, 0)
    with pytest.raises(ValueError):
        se.total_potential(s, SEParams(xi=6.0, rc=0.3, M=16, P=8, window="box", shape=10.0), Periodicity(3))


# ---------------------------------------------------------------- AFT

def test_aft_zero_field_parseval_and_rejections():
    p = params(2, M=8, P=4, xi=5.0, eps=1e-6)
    g = Grid.build(1.0, p, Periodicity(2))
    part = aft.ModePartition.build(8, 2, 2)
    F = aft.aft_forward(np.zeros(g.shape), part, p.s0, p.s, Periodicity(2))
    assert not np.any(F.zero) and not np.any(F.Iblk) and not np.any(F.Jblk)
    assert not np.any(aft.aft_inverse(F, part, 8, Periodicity(2)))
    # Parseval of the periodic stage: sum |H_k|^2 = n_periodic sum |H|^2
    H = np.random.default_rng(2).normal(size=g.shape)
    Hk = aft.periodic_stage(H, 2)
    assert np.sum(np.abs(Hk) ** 2) == pytest.approx(64 * np.sum(H ** 2), rel=1e-12)
    with pytest.raises(ValueError):  # odd free-axis size
        aft.aft_forward(np.zeros((8, 8, 11)), part, p.s0, p.s, Periodicity(2))


# ---------------------------------------------------------------- real space

def test_far_pair_with_large_xi_negligible_and_newton_symmetry():
    # erfc(xi r)/r below 1e-300 at xi r ~ 27: exactly zero contribution
    s = ParticleSystem(np.array([[0.1, 0.5, 0.5], [0.45, 0.5, 0.5]]), np.array([1.0, -1.0]), 1.0)
    phi = se.real_space_sum(s, 80.0, 0.4, Periodicity(0))
    assert np.all(np.abs(phi) < 1e-300)
    # pair kernel symmetry: phi_m / q_n == phi_n / q_m for an isolated pair
    s = ParticleSystem(np.array([[0.3, 0.3, 0.3], [0.45, 0.4, 0.35]]), np.array([2.0, -0.5]), 1.0)
    phi = se.real_space_sum(s, 5.0, 0.45, Periodicity(3))
    assert phi[0] / -0.5 == pytest.approx(phi[1] / 2.0, rel=1e-15)


def test_cutoff_stability_at_selected_rc():
    # beyond the selected rc the sum changes by ~eps relative
    s = rand_system(400, 1.0, 21)
    xi, eps = 12.0, 1e-10
    rc = math.sqrt(-math.log(eps)) / xi
    a = se.real_space_sum(s, xi, rc, Periodicity(3))
    b = se.real_space_sum(s, xi, min(1.3 * rc, 0.5), Periodicity(3))
    assert se.relative_rms_error(a, b) < 100 * eps
