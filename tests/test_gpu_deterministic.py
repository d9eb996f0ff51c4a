"""Deterministic mode (se_plan_set_deterministic / SE_B200_DETERMINISTIC):
repeated evaluations are bitwise identical -- the reference's
thread-count independence (test_core.py:139-145, test_realspace.py:129-133)
-- and agree with the default (atomic, Newton) mode to rounding.  Covers the
full-shell real-space path (periodic and free axes), the per-unit tile
spreading with its ordered reduction, and the whole pipeline."""

import numpy as np
import pytest

import paper_1712_04732_b200 as se

pytestmark = pytest.mark.gpu


def _system(N, L, seed):
    rng = np.random.default_rng(seed)
    pos = rng.random((N, 3)) * L
    q = rng.uniform(-1, 1, N)
    q -= q.mean()
    return se.ParticleSystem(pos, q, L)


@pytest.fixture
def det():
    se.set_deterministic(True)
    yield
    se.set_deterministic(False)


@pytest.mark.parametrize("D", [3, 2, 1, 0])
def test_total_potential_bitwise_reproducible(det, D):
    s = _system(30000, 3.0, 40 + D)
    prm = se.SEParams(xi=6.0, rc=0.5, M=32, P=8, window="bm", shape=20.0, s0=4.0, s=2.0, nI=4, R=3.0)
    peri = se.Periodicity(D)
    a = se.total_potential(s, prm, peri)
    b = se.total_potential(s, prm, peri, threads=4)
    c = se.total_potential(s, prm, peri)
    assert np.array_equal(a, b) and np.array_equal(a, c)
    r1 = se.real_space_sum(s, 6.0, 0.5, peri)
    r2 = se.real_space_sum(s, 6.0, 0.5, peri, threads=8)
    assert np.array_equal(r1, r2)
    se.set_deterministic(False)
    ref = se.total_potential(s, prm, peri)
    err = se.relative_rms_error(a, ref)
    print(f"D={D}: deterministic vs default {err:.2e}")
    assert err < 1e-13


def test_spread_grid_bitwise_reproducible(det):
    from paper_1712_04732_b200 import sekspace, windows

    s = _system(50000, 2.0, 7)
    prm = se.SEParams(xi=6.0, rc=0.5, M=40, P=8, window="bm", shape=20.0)
    grid = sekspace.Grid.build(2.0, prm, se.Periodicity(3))
    ws = windows.WindowSpec("bm", 8, grid.h, 20.0)
    g1 = sekspace.spread(s, ws, grid, se.Periodicity(3)).values
    g2 = sekspace.spread(s, ws, grid, se.Periodicity(3)).values
    assert np.array_equal(g1, g2)
    se.set_deterministic(False)
    g3 = sekspace.spread(s, ws, grid, se.Periodicity(3)).values
    assert np.max(np.abs(g1 - g3)) <= 1e-13 * np.max(np.abs(g3))


def test_coincident_z_layer(det):
    # every particle at the same z: whole columns fall into one fine bin of
    # the counting sort (the large-bin path); still bitwise reproducible and
    # equal to the oracle
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import se_oracle as orc

    rng = np.random.default_rng(9)
    N, L = 6000, 2.0
    pos = rng.random((N, 3)) * L
    pos[:, 2] = 0.7
    q = rng.uniform(-1, 1, N)
    q -= q.mean()
    s = se.ParticleSystem(pos, q, L)
    a = se.real_space_sum(s, 6.0, 0.5, se.Periodicity(2))
    b = se.real_space_sum(s, 6.0, 0.5, se.Periodicity(2))
    assert np.array_equal(a, b)
    ref = orc.realspace(pos, q, L, 2, 6.0, 0.5)
    assert se.relative_rms_error(a, ref) < 1e-13
    se.set_deterministic(False)
    c = se.real_space_sum(s, 6.0, 0.5, se.Periodicity(2))
    assert se.relative_rms_error(c, ref) < 1e-13


@pytest.mark.parametrize("D", [3, 1, 0])
def test_dense_full_shell_matches_newton_and_oracle(det, D):
    # ~2000 partners per particle: most batches of the deterministic mode's
    # full shell take the dense path (dense_batch_poly without Newton: the
    # self pair dropped by its index, no source side), the rest the
    # compacted path with the polynomial pair term
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import se_oracle as orc

    s = _system(30000, 1.0, 90 + D)
    xi, rc = 14.0, 0.25
    peri = se.Periodicity(D)
    a = se.real_space_sum(s, xi, rc, peri)
    b = se.real_space_sum(s, xi, rc, peri)
    assert np.array_equal(a, b)
    se.set_deterministic(False)
    ref = se.real_space_sum(s, xi, rc, peri)
    assert se.relative_rms_error(a, ref) < 1e-14
    sel = np.random.default_rng(6).choice(s.N, 40, replace=False)
    want = orc.realspace(s.positions, s.charges, s.L, D, xi, rc, targets=sel)
    assert se.relative_rms_error(a[sel], want) < 1e-13
