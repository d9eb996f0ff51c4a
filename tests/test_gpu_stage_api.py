"""GPU tests of the reference's stage-level API on the cuFFT engine:
aft.periodic_stage / free_stage / aft_forward / aft_inverse, set_engine,
and sekspace.scale -- mirroring the reference's test_aft.py and the scale
tests of test_sekspace.py, checked against numpy FFTs / direct DFTs and the
CPU oracle."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import se_oracle as orc  # noqa: E402

import paper_1712_04732_b200 as se  # noqa: E402
from paper_1712_04732_b200 import aft, greens, sekspace, windows  # noqa: E402
from paper_1712_04732_b200.aft import ModePartition, aft_forward, aft_inverse  # noqa: E402


def grid_rand(shape, seed):
    return np.random.default_rng(seed).normal(size=shape)


class DftEngine:
    """O(n^2) DFT with numpy-fft semantics (the reference's test fake)."""

    @staticmethod
    def _along(a, ax, inv):
        n = a.shape[ax]
        j = np.arange(n)
        W = np.exp((1j if inv else -1j) * 2 * np.pi * np.outer(j, j) / n)
        if inv:
            W = W / n
        return np.moveaxis(np.tensordot(W, np.moveaxis(a, ax, 0), axes=(1, 0)), 0, ax)

    def fftn(self, a, axes):
        out = np.asarray(a, dtype=complex)
        for ax in axes:
            out = self._along(out, ax, False)
        return out

    def ifftn(self, a, axes):
        out = np.asarray(a, dtype=complex)
        for ax in axes:
            out = self._along(out, ax, True)
        return out


def test_engine_matches_numpy():
    eng = aft.current_engine()
    a = grid_rand((6, 10, 8), 1) + 1j * grid_rand((6, 10, 8), 2)
    for axes in ((0, 1, 2), (0,), (1, 2), (0, 1), (2,), (0, 2)):
        assert np.allclose(eng.fftn(a, axes), np.fft.fftn(a, axes=axes), rtol=1e-13, atol=1e-12)
        assert np.allclose(eng.ifftn(a, axes), np.fft.ifftn(a, axes=axes), rtol=1e-13, atol=1e-14)
    r = grid_rand((12, 12, 12), 3)
    s = (16, 16, 16)
    assert np.allclose(eng.rfftn(r, s, (0, 1, 2)), np.fft.rfftn(r, s=s, axes=(0, 1, 2)), atol=1e-12)
    c = np.fft.rfftn(r, axes=(0, 1, 2))
    assert np.allclose(eng.irfftn(c, (12, 12, 12), (0, 1, 2)), r, atol=1e-13)


def test_forward_matches_direct_dft_d2():
    M, Mt = 8, 12
    part = ModePartition.build(M, 2, 2)
    H = grid_rand((M, M, Mt), 1)
    F = aft_forward(H, part, 2.0, 1.5, se.Periodicity(2))
    Hk = np.fft.fftn(H, axes=(0, 1))

    def padded(row, g):
        out = np.zeros(g, dtype=complex)
        out[:Mt] = row
        return np.fft.fft(out)

    assert np.allclose(F.zero, padded(Hk[0, 0], F.g0), atol=1e-12)
    for r, (i, j) in enumerate(part.I_idx):
        assert np.allclose(F.Iblk[r], padded(Hk[i, j], F.gs), atol=1e-12)
    for r, (i, j) in enumerate(part.J_idx):
        assert np.allclose(F.Jblk[r], np.fft.fft(Hk[i, j]), atol=1e-12)


def test_roundtrips_all_periodicities():
    M, Mt = 8, 12
    part = ModePartition.build(M, 2, 2)
    H = grid_rand((M, M, Mt), 3)
    back = aft_inverse(aft_forward(H, part, 2.0, 3.0, se.Periodicity(2)), part, M, se.Periodicity(2))
    assert np.max(np.abs(back - H)) < 1e-13 * np.max(np.abs(H))
    part1 = ModePartition.build(6, 1, 2)
    H1 = grid_rand((6, 10, 10), 4)
    back = aft_inverse(aft_forward(H1, part1, 2.5, 1.8, se.Periodicity(1)), part1, 6, se.Periodicity(1))
    assert np.max(np.abs(back - H1)) < 1e-13 * np.max(np.abs(H1))
    H3 = grid_rand((8, 8, 8), 5)
    assert np.max(np.abs(aft_inverse(aft_forward(H3, None, 1.0, 1.0, se.Periodicity(3)), None, 8,
                                     se.Periodicity(3)) - H3)) < 1e-13
    H0 = grid_rand((10, 10, 10), 6)
    assert np.max(np.abs(aft_inverse(aft_forward(H0, None, 2.8, 1.0, se.Periodicity(0)), None, 0,
                                     se.Periodicity(0)) - H0)) < 1e-13


def test_j_only_spectrum_matches_direct_inverse():
    M, Mt = 8, 10
    part = ModePartition.build(M, 1, 2)
    rng = np.random.default_rng(7)
    F = aft_forward(np.zeros((M, Mt, Mt)), part, 2.5, 1.5, se.Periodicity(1))
    F.Jblk = rng.normal(size=F.Jblk.shape) + 1j * rng.normal(size=F.Jblk.shape)
    got = aft_inverse(F, part, M, se.Periodicity(1))
    Hk = np.zeros((M, Mt, Mt), dtype=complex)
    for r, (i,) in enumerate(part.J_idx):
        Hk[i] = np.fft.ifftn(F.Jblk[r])
    want = np.fft.ifft(Hk, axis=0)
    assert np.max(np.abs(got - want)) < 1e-12 * np.max(np.abs(want))


def test_block_independence_bit_exact():
    M, Mt = 8, 12
    part = ModePartition.build(M, 2, 2)
    rng = np.random.default_rng(9)
    Hk = rng.normal(size=(M, M, Mt)) + 1j * rng.normal(size=(M, M, Mt))
    z1, I1, J1 = aft.free_stage(Hk, part, 24, 18)
    Hk2 = Hk.copy()
    for (i, j) in part.J_idx:
        Hk2[i, j] += rng.normal(size=Mt)
    z2, I2, J2 = aft.free_stage(Hk2, part, 24, 18)
    assert np.array_equal(z1, z2) and np.array_equal(I1, I2) and not np.array_equal(J1, J2)


def test_engine_swap_matches_default():
    M, Mt = 6, 8
    part = ModePartition.build(M, 2, 1)
    H = grid_rand((M, M, Mt), 10)
    F = aft_forward(H, part, 2.0, 1.5, se.Periodicity(2))
    old = aft.current_engine()
    aft.set_engine(DftEngine())
    try:
        G = aft_forward(H, part, 2.0, 1.5, se.Periodicity(2))
    finally:
        aft.set_engine(old)
    for a, b in ((F.zero, G.zero), (F.Iblk, G.Iblk), (F.Jblk, G.Jblk)):
        assert np.allclose(a, b, atol=1e-12)


def test_scale_single_mode_composed_constant():
    L, M, P, xi = 2.0, 8, 4, 3.0
    prm = se.SEParams(xi=xi, rc=0.5, M=M, P=P, window="bm", shape=10.0, eps=1e-6)
    grid = sekspace.Grid.build(L, prm, se.Periodicity(3))
    wspec = windows.WindowSpec("bm", P, grid.h, 10.0)
    F = aft.SpectralField(3, M, M, M, M, full=np.zeros((M, M, M), dtype=complex))
    F.full[1, 0, 0] = 1.0
    out = sekspace.scale(F, xi, wspec, greens.GreensSpec(3), grid, se.Periodicity(3))
    k = 2.0 * math.pi / L
    what = float(windows.fourier(np.array([k]), wspec)[0] * windows.fourier(np.array([0.0]), wspec)[0] ** 2)
    want = 4.0 * math.pi * math.exp(-k * k / (4 * xi * xi)) / (k * k * what ** 2)
    assert out.full[1, 0, 0].real == pytest.approx(want, rel=1e-13)
    assert np.count_nonzero(out.full) == 1


def test_scale_zero_spectrum_and_zero_mode():
    prm = se.SEParams(xi=5.0, rc=0.4, M=8, P=4, window="bm", shape=10.0, s0=3.0, s=2.0, nI=2, R=2.0, eps=1e-6)
    grid = sekspace.Grid.build(1.0, prm, se.Periodicity(2))
    part = ModePartition.build(8, 2, 2)
    F = aft_forward(np.zeros(grid.shape), part, prm.s0, prm.s, se.Periodicity(2))
    wspec = windows.WindowSpec("bm", 4, grid.h, 10.0)
    out = sekspace.scale(F, prm.xi, wspec, greens.GreensSpec(2, prm.R), grid, se.Periodicity(2))
    assert not np.any(out.zero) and not np.any(out.Iblk) and not np.any(out.Jblk)
    p3 = se.SEParams(xi=5.0, rc=0.4, M=8, P=4, window="bm", shape=10.0, eps=1e-6)
    g3 = sekspace.Grid.build(1.0, p3, se.Periodicity(3))
    F3 = aft_forward(grid_rand((8, 8, 8), 1), None, 1.0, 1.0, se.Periodicity(3))
    out3 = sekspace.scale(F3, 5.0, wspec, greens.GreensSpec(3), g3, se.Periodicity(3))
    assert out3.full[0, 0, 0] == 0.0


def test_scale_underflow_guard():
    prm = se.SEParams(xi=2.0, rc=0.4, M=64, P=4, window="gaussian", shape=0.1, eps=1e-8)
    grid = sekspace.Grid.build(1.0, prm, se.Periodicity(3))
    wspec = windows.WindowSpec("gaussian", 4, grid.h, 0.1)
    F = aft_forward(np.ones((64, 64, 64)), None, 1.0, 1.0, se.Periodicity(3))
    with pytest.raises(AssertionError):
        sekspace.scale(F, prm.xi, wspec, greens.GreensSpec(3), grid, se.Periodicity(3))


@pytest.mark.parametrize("D", [0, 1, 2, 3])
def test_stage_pipeline_equals_fused_and_oracle(D):
    # spread -> aft_forward -> scale -> aft_inverse -> gather == se_kspace (sekspace.py:340-389)
    s = se.generate_random_system(40, 1.0, seed=30 + D)
    M, P = 16, 8
    if D == 3:
        p = se.SEParams(xi=6.0, rc=0.4, M=M, P=P, window="bm", shape=20.0, eps=1e-8)
    else:
        s0 = 3.0 if D == 0 else 2.6
        p = se.SEParams(xi=6.0, rc=0.4, M=M, P=P, window="bm", shape=20.0, s0=s0, s=2.0,
                        nI=3 if D in (1, 2) else 0, R=2.2, eps=1e-8)
    peri = se.Periodicity(D)
    grid = sekspace.Grid.build(1.0, p, peri)
    wspec = windows.WindowSpec("bm", P, grid.h, 20.0)
    gspec = greens.GreensSpec(D, grid.R) if D < 3 else greens.GreensSpec(3)
    part = ModePartition.build(M, D, p.nI) if D in (1, 2) else None
    H = sekspace.spread(s, wspec, grid, peri)
    F = sekspace.scale(aft_forward(H.values, part, p.s0, p.s, peri), p.xi, wspec, gspec, grid, peri)
    Ht = aft_inverse(F, part, M, peri)
    phi = sekspace.gather(sekspace.GridField(np.ascontiguousarray(Ht.real), grid), s, wspec, peri)
    fused = se.se_kspace(s, p, peri, use_kernel=False if D == 0 else None)
    ref = orc.se_kspace(s.positions, s.charges, 1.0, D, dict(p.__dict__), use_kernel=False if D == 0 else None)
    assert se.relative_rms_error(phi, fused) < 1e-13
    assert se.relative_rms_error(phi, ref) < 1e-12
