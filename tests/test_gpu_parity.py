"""GPU parity: the sm_100a pipeline through the public API (C ABI) against
the reference's golden vectors and the CPU oracle (oracle/se_oracle.py).

Tolerances: every comparison is fp64; the north-star bar is relative RMS
<= 1e-10 against the reference CPU implementation.  Stage comparisons use
tighter bounds (1e-12 .. 1e-13) because the only differences are rounding
(fp64 atomics in spreading, cuFFT vs pocketfft, CUDA vs cephes erfc).
"""

import math
import os
import warnings

import numpy as np
import pytest

from conftest import GOLDEN, PIPELINE_CASES, load_case

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import se_oracle as orc  # noqa: E402

import paper_1712_04732_b200 as se  # noqa: E402
from paper_1712_04732_b200 import device as sedev  # noqa: E402
from paper_1712_04732_b200 import sekspace, windows  # noqa: E402

FIELDS = ("xi", "rc", "M", "P", "window", "shape", "s0", "s", "nI", "R", "eps")
PARITY = 1e-10  # north_star bar (relative RMS vs the reference CPU path)


def params_of(c):
    return se.SEParams(**{k: c["prm"][k] for k in FIELDS})


def system_of(c):
    return se.ParticleSystem(c["pos"], c["q"], c["L"])


def rand_system(N, L, seed):
    rng = np.random.default_rng(seed)
    pos = rng.random((N, 3)) * L
    q = rng.uniform(-1, 1, N)
    q -= q.mean()
    return se.ParticleSystem(pos, q, L)


# ------------------------------------------------------------ golden vectors

@pytest.mark.parametrize("name", PIPELINE_CASES)
def test_golden_stages(name):
    c = load_case(name)
    s, p, peri = system_of(c), params_of(c), se.Periodicity(c["D"])
    grid = sekspace.Grid.build(s.L, p, peri)
    wspec = windows.WindowSpec(p.window, p.P, grid.h, p.shape)
    H = sekspace.spread(s, wspec, grid, peri).values
    assert np.max(np.abs(H - c["H"])) <= 1e-13 * np.max(np.abs(c["H"]))
    uk = None if c["use_kernel"] < 0 else bool(c["use_kernel"])
    phik = se.se_kspace(s, p, peri, use_kernel=uk)
    assert se.relative_rms_error(phik, c["phi_k"]) < 1e-12
    if "phi_r" in c:
        phir = se.real_space_sum(s, p.xi, p.rc, peri)
        assert np.allclose(phir, c["phi_r"], rtol=1e-12, atol=1e-13)
        assert np.allclose(se.self_term(s.charges, p.xi), c["phi_s"], rtol=1e-15, atol=0)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            phi = se.total_potential(s, p, peri) if uk is None else phir + phik + se.self_term(s.charges, p.xi)
        assert se.relative_rms_error(phi, c["phi"]) < PARITY
        assert se.relative_rms_error(phi, c["phi"]) < 1e-12


def test_golden_realspace_paths():
    z = np.load(os.path.join(GOLDEN, "realspace.npz"))
    s = se.ParticleSystem(z["img_pos"], z["img_q"], 1.0)
    for D, rc in ((3, 1.2), (2, 0.8), (1, 0.7)):
        assert np.allclose(se.real_space_sum(s, 4.0, rc, se.Periodicity(D)), z[f"img_d{D}"], rtol=1e-12, atol=1e-13)
    s = se.ParticleSystem(z["cell_pos"], z["cell_q"], 1.0)
    for D in (0, 1, 2, 3):
        assert np.allclose(se.real_space_sum(s, 7.0, 0.23, se.Periodicity(D)), z[f"cell_d{D}"], rtol=1e-12, atol=1e-13)
        assert np.allclose(se.real_space_sum(s, 5.0, 0.45, se.Periodicity(D)), z[f"cell2_d{D}"], rtol=1e-12, atol=1e-13)


def test_golden_d0_kernel_table():
    z = np.load(os.path.join(GOLDEN, "d0_kernel.npz"))
    k = sekspace.precompute_truncated_greens(1.0, 16, 8, 1 + math.sqrt(3.0), rc=0.5)
    assert k.nconv == int(z["nconv"]) and k.g0 == int(z["g0"])
    assert np.max(np.abs(k.ghat - z["ghat"])) <= 1e-12 * np.max(np.abs(z["ghat"]))
    assert sekspace.precompute_truncated_greens(1.0, 16, 8, 1 + math.sqrt(3.0), rc=0.5) is k


# ------------------------------------------------------- oracle, larger sizes

CFG_SMALL = {
    # cfg1 exactly (N=2000, Gaussian P=16, M=32, rc=0.3, xi=12.94)
    "cfg1": (3, 2000, 1.0, dict(xi=12.94, rc=0.3, M=32, P=16, window="gaussian",
                                shape=math.sqrt(16 * math.pi), eps=1e-8)),
    # cfg2 shape at 1/100 of the particles (same density: L = 10 * 0.1^(2/3))
    "cfg2_small": (3, 10000, 10.0 * 0.01 ** (1 / 3), dict(xi=4.2919, rc=1.0, M=28, P=8, window="bm",
                                                          shape=20.0, eps=1e-8)),
}


@pytest.mark.parametrize("name", sorted(CFG_SMALL))
def test_oracle_parity_configs(name):
    D, N, L, prm = CFG_SMALL[name]
    s = rand_system(N, L, 11)
    p = se.SEParams(**prm)
    phi = se.total_potential(s, p, se.Periodicity(D))
    ref = orc.total_potential(s.positions, s.charges, L, D, dict(p.__dict__))
    assert se.relative_rms_error(phi, ref) < PARITY


@pytest.mark.parametrize("D", [0, 1, 2])
def test_oracle_parity_mixed(D):
    # cfg3/4/5 shapes at reduced N and grids
    s = rand_system(3000, 2.0, 20 + D)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        p, _ = se.auto_params(s, se.Periodicity(D), 4.0, 1e-8,
                              window="gaussian" if D == 1 else "bm")
    phi = se.total_potential(s, p, se.Periodicity(D))
    ref = orc.total_potential(s.positions, s.charges, s.L, D, dict(p.__dict__))
    assert se.relative_rms_error(phi, ref) < PARITY


def test_d0_full_path_matches_oracle_and_kernel():
    s = rand_system(200, 1.0, 5)
    p = se.SEParams(xi=8.0, rc=0.43, M=24, P=16, window="bm", shape=40.0, s0=3.0, R=2.9, eps=1e-12)
    full = se.se_kspace(s, p, se.Periodicity(0), use_kernel=False)
    kern = se.se_kspace(s, p, se.Periodicity(0), use_kernel=True)
    ref = orc.se_kspace(s.positions, s.charges, 1.0, 0, dict(p.__dict__), use_kernel=False)
    assert se.relative_rms_error(full, ref) < 1e-12
    assert se.relative_rms_error(kern, full) < 1e-10


@pytest.mark.parametrize("D", [1, 2])
def test_degenerate_aft_equals_global_padding(D):
    s = rand_system(60, 1.0, 6 + D)
    M, P = 16, 8
    rc = 0.5
    s0 = max(1 + math.sqrt(3 - D), ((1 + math.sqrt(3 - D)) + 2 * rc) / 1.5)
    from paper_1712_04732_b200 import aft
    R = 0.5 * (aft.padded_size(s0, M + P) / M - 1 + math.sqrt(3 - D))
    p = se.SEParams(xi=5.0, rc=rc, M=M, P=P, window="bm", shape=20.0, s0=s0, s=s0, nI=M // 2, R=R, eps=1e-8)
    a = se.se_kspace(s, p, se.Periodicity(D))
    b = sekspace.global_upsampled_kspace(s, p, se.Periodicity(D))
    ref = orc.se_kspace(s.positions, s.charges, 1.0, D, dict(p.__dict__))
    assert se.relative_rms_error(a, b) < 1e-13
    assert se.relative_rms_error(a, ref) < 1e-12


def test_large_support_direct_path():
    # P=34 > shared-memory tile capacity: direct global-atomic spreading path
    s = rand_system(80, 1.0, 9)
    p = se.SEParams(xi=12.0, rc=0.4, M=64, P=34, window="bm", shape=85.0, eps=1e-12)
    phi = se.se_kspace(s, p, se.Periodicity(3))
    ref = orc.se_kspace(s.positions, s.charges, 1.0, 3, dict(p.__dict__))
    assert se.relative_rms_error(phi, ref) < 1e-12


# ----------------------------------------------------------- reference tests

def test_spread_gather_adjoint_all_periodicities():
    rng = np.random.default_rng(15)
    for D in (0, 1, 2, 3):
        for window in ("bm", "gaussian", "kb"):
            p = se.SEParams(xi=5.0, rc=0.4, M=14, P=6, window=window,
                            shape=windows.default_shape(window, 6), s0=3.0, R=2.0)
            grid = sekspace.Grid.build(1.0, p, se.Periodicity(D))
            wspec = windows.WindowSpec(window, 6, grid.h, p.shape)
            s = se.generate_random_system(9, 1.0, seed=D)
            H = sekspace.spread(s, wspec, grid, se.Periodicity(D))
            G = rng.normal(size=grid.shape)
            lhs = grid.h ** 3 * float(np.sum(H.values * G))
            rhs = float(s.charges @ sekspace.gather(sekspace.GridField(G, grid), s, wspec, se.Periodicity(D)))
            assert lhs == pytest.approx(rhs, rel=1e-13)


@pytest.mark.parametrize("P", list(range(2, 19)) + [20, 24])
def test_spread_gather_tile_geometry_sweep(P):
    # every window width against the oracle's stencils: anisotropic 17-deep
    # tiles (P <= 12), cubic ones above, compile-time and runtime P, tiles
    # clipped at the free-axis ends and wrapped on periodic axes, a cluster
    # that splits one tile into several work units
    rng = np.random.default_rng(300 + P)
    for D in ((0, 3) if P % 2 else (0, 1, 2, 3)):
        M = max(P + 2, 38) + (P % 2 if D in (1, 2) else 0)
        N = 2500
        pos = rng.random((N, 3))
        pos[:1200] = np.mod(0.37 + rng.normal(scale=0.01, size=(1200, 3)), 1.0)
        pos[pos >= 1.0] = 0.0
        q = rng.uniform(-1, 1, N)
        window = ("bm", "gaussian", "kb")[P % 3]
        shape = windows.default_shape(window, P)
        p = se.SEParams(xi=6.0, rc=0.4, M=M, P=P, window=window, shape=shape, s0=3.0, R=2.0)
        peri = se.Periodicity(D)
        grid = sekspace.Grid.build(1.0, p, peri)
        wspec = windows.WindowSpec(window, P, grid.h, shape)
        s = se.ParticleSystem(pos, q, 1.0)
        H = sekspace.spread(s, wspec, grid, peri).values
        g = orc.geometry(1.0, D, M, P, 3.0, 1.0, 2.0)
        ref = orc.spread(pos, q, g, window, shape)
        assert np.max(np.abs(H - ref)) <= 1e-13 * np.max(np.abs(ref)), (P, D)
        G = rng.normal(size=grid.shape)
        phi = sekspace.gather(sekspace.GridField(G, grid), s, wspec, peri)
        rphi = orc.gather(G, pos, g, window, shape)
        assert np.max(np.abs(phi - rphi)) <= 1e-13 * np.max(np.abs(rphi)), (P, D)


def test_spread_on_node_tensor_window_and_count():
    M, P = 16, 6
    p = se.SEParams(xi=5.0, rc=0.4, M=M, P=P, window="bm", shape=15.0, s0=3.0, R=2.0)
    grid = sekspace.Grid.build(1.0, p, se.Periodicity(0))
    wspec = windows.WindowSpec("bm", P, grid.h, 15.0)
    x = 5 * grid.h
    H = sekspace.spread(se.ParticleSystem(np.array([[x, x, x]]), np.array([1.0]), 1.0), wspec, grid,
                        se.Periodicity(0)).values
    ref = orc.spread(np.array([[x, x, x]]), np.array([1.0]), orc.geometry(1.0, 0, M, P, 3.0, 1.0, 2.0), "bm", 15.0)
    assert np.array_equal(H != 0, ref != 0)
    assert np.allclose(H, ref, rtol=1e-14, atol=1e-300)
    p3 = se.SEParams(xi=5.0, rc=0.4, M=20, P=6, window="bm", shape=15.0)
    g3 = sekspace.Grid.build(1.0, p3, se.Periodicity(3))
    H3 = sekspace.spread(se.ParticleSystem(np.array([[0.311, 0.77, 0.132]]), np.array([1.0]), 1.0),
                         windows.WindowSpec("bm", 6, g3.h, 15.0), g3, se.Periodicity(3)).values
    assert np.count_nonzero(H3) == 6 ** 3


def test_empty_and_zero_charge_systems():
    p = se.SEParams(xi=6.0, rc=0.4, M=16, P=8, window="bm", shape=20.0, eps=1e-8)
    grid = sekspace.Grid.build(1.0, p, se.Periodicity(3))
    wspec = windows.WindowSpec("bm", 8, grid.h, 20.0)
    empty = se.ParticleSystem(np.empty((0, 3)), np.empty(0), 1.0)
    assert not np.any(sekspace.spread(empty, wspec, grid, se.Periodicity(3)).values)
    assert se.se_kspace(empty, p, se.Periodicity(3)).shape == (0,)
    s = se.generate_random_system(6, 1.0, seed=4)
    s0 = se.ParticleSystem(s.positions, np.zeros(6), 1.0)
    assert np.all(se.total_potential(s0, p, se.Periodicity(3)) == 0.0)


def test_error_conventions():
    p = se.SEParams(xi=5.0, rc=0.4, M=16, P=8, window="bm", shape=20.0, eps=1e-8)
    pos = np.array([[0.5, 0.5, 0.5], [0.5, 0.5, 0.5]])
    s = se.ParticleSystem(pos, np.array([1.0, -1.0]), 1.0)
    with pytest.raises(se.SingularConfigurationError):
        se.real_space_sum(s, 5.0, 0.4, se.Periodicity(0))
    with pytest.raises(se.SingularConfigurationError):
        se.total_potential(s, p, se.Periodicity(3))
    charged = se.ParticleSystem(np.array([[0.1, 0.2, 0.3], [0.6, 0.5, 0.4]]), np.array([1.0, 0.5]), 1.0)
    with pytest.raises(ValueError, match="charge-neutral"):
        se.total_potential(charged, p, se.Periodicity(3))
    pd0 = se.SEParams(xi=5.0, rc=0.4, M=16, P=8, window="bm", shape=20.0, s0=3.0, R=2.0, eps=1e-8)
    with pytest.warns(UserWarning):
        se.total_potential(charged, pd0, se.Periodicity(0))
    with pytest.raises(ValueError):
        se.real_space_sum(s, -1.0, 0.4, se.Periodicity(3))


@pytest.mark.parametrize("D", [3, 0])
def test_invalid_coordinates_are_reported_after_the_device_work(D):
    """core.py:65-77: coordinates outside [0, L) are a ValueError.  The fused
    device call reports them after its device work (no host round trip up
    front); the binning kernels read coordinates through sane_coord, so a
    NaN, a negative value, x >= L or a whole batch of unwrapped coordinates
    neither faults nor piles up -- and the next valid call is untouched."""
    dev = torch.device("cuda", 0)
    L, N = 2.0, 20000
    p = se.SEParams(xi=6.0, rc=0.5, M=32, P=8, window="bm", shape=20.0, eps=1e-8,
                    **({"s0": 3.0, "R": 3.5} if D == 0 else {}))
    peri = se.Periodicity(D)
    s = rand_system(N, L, 11)
    pos = torch.from_numpy(s.positions).to(dev)
    q = torch.from_numpy(s.charges).to(dev)
    good = sedev.total_potential(pos, q, L, p, peri).cpu().numpy()
    ref = se.total_potential(s, p, peri)
    assert np.linalg.norm(good - ref) <= 1e-12 * np.linalg.norm(ref)
    for kind in ("nan", "negative", "at_L", "far", "half_unwrapped"):
        bad = pos.clone()
        if kind == "nan":
            bad[7, 1] = float("nan")
        elif kind == "negative":
            bad[3, 0] = -1e-9
        elif kind == "at_L":
            bad[N - 1, 2] = L
        elif kind == "far":
            bad[5] = torch.tensor([1e300, -1e300, float("inf")], dtype=torch.float64)
        else:
            bad[: N // 2] += L  # unwrapped MD coordinates
        for _ in range(3):  # eager, graph capture, graph replay
            with pytest.raises(ValueError, match=r"\[0, L\)"):
                sedev.total_potential(bad, q, L, p, peri)
    again = sedev.total_potential(pos, q, L, p, peri).cpu().numpy()
    assert np.max(np.abs(again - good)) <= 1e-13 * np.max(np.abs(good))


def test_two_particle_single_term_and_cutoff():
    from scipy.special import erfc
    r = 0.2
    s = se.ParticleSystem(np.array([[0.3, 0.5, 0.5], [0.5, 0.5, 0.5]]), np.array([2.0, -1.0]), 1.0)
    phi = se.real_space_sum(s, 5.0, 0.45, se.Periodicity(0))
    assert phi[0] == pytest.approx(-1.0 * erfc(5.0 * r) / r, rel=1e-15)
    assert phi[1] == pytest.approx(2.0 * erfc(5.0 * r) / r, rel=1e-15)
    rc = 0.25
    far = se.ParticleSystem(np.array([[0.1, 0.5, 0.5], [0.1 + rc + 1 / 28, 0.5, 0.5]]), np.array([1.0, -1.0]), 1.0)
    assert np.all(se.real_space_sum(far, 5.0, rc, se.Periodicity(0)) == 0.0)


# xi rc covers every degree of the polynomial pair term (se_pair_poly_coefficients:
# 20 for xi rc <= 2.5, 24, 28, 32) and the erfc fallback (xi rc > ~5)
@pytest.mark.parametrize("xi,rc", [(4.2919, 1.0), (12.0, 0.45), (2.0, 1.0), (8.0, 0.4), (4.0, 1.0), (4.8, 1.0),
                                   (5.4, 1.0)])
def test_isolated_pairs_sweep_pair_kernel(xi, rc):
    # K isolated +-1 pairs at separations spanning (0, rc): each potential is
    # one kernel term q erfc(xi r)/r, checked against 30-digit values.  The
    # bound is on the absolute error of erfc (the pair term carries the 1/r
    # rounding anyway): 4 ulp of 1/r.
    import mpmath as mp
    mp.mp.dps = 30
    K = 400
    d = np.linspace(1e-3, 0.999, K) * rc
    d[-1] = rc * (1 - 1e-9)
    L = 4.0 * rc * K ** (1 / 3) + 10 * rc
    g = int(np.ceil(K ** (1 / 3)))
    ij = np.array([(i, j, k) for i in range(g) for j in range(g) for k in range(g)][:K], dtype=float)
    base = 2.0 * rc + ij * 3.0 * rc
    pos = np.concatenate([base, base + np.stack([d, np.zeros(K), np.zeros(K)], 1)])
    q = np.concatenate([np.ones(K), -np.ones(K)])
    s = se.ParticleSystem(pos, q, L)
    phi = se.real_space_sum(s, xi, rc, se.Periodicity(0))
    r = np.linalg.norm(pos[K:] - pos[:K], axis=1)
    want = np.array([float(mp.erfc(mp.mpf(xi) * mp.mpf(v)) / mp.mpf(v)) for v in r])
    err = np.abs(-phi[:K] - want) * r
    assert np.max(err) < 4.5e-16, np.max(err)
    assert np.max(np.abs(phi[K:] - want) * r) < 4.5e-16
    # both pair-term forms are accurate in ABSOLUTE terms (the 1/r rounding):
    # erfc_fast's erfc fit keeps tiny tail terms to ~1e-9 relative, the
    # polynomial form 1/r - Q(r^2) (pair_poly, cancelling towards the
    # cutoff) to ~ulp(1/rc) / term -- < 5e-6 for terms >= 1e-10 / rc
    big = want * rc >= 1e-10
    rel = np.abs(-phi[:K] - want)[big] / want[big]
    assert np.max(rel) < 5e-6


def test_threads_argument_and_determinism():
    s = rand_system(4000, 1.0, 8)
    p = se.SEParams(xi=8.0, rc=0.4, M=32, P=8, window="bm", shape=20.0, eps=1e-8)
    a = se.total_potential(s, p, se.Periodicity(3), threads=1)
    b = se.total_potential(s, p, se.Periodicity(3), threads=8)
    # fp64 atomics (spreading-tile flush, Newton-symmetric real-space pair
    # sums) add in nondeterministic order: the only run-to-run difference is
    # final-bit rounding, far below the 1e-10 parity bar.  The reference's
    # bit-identity across thread counts (test_core.py:139-145) becomes this
    # bound.
    assert se.relative_rms_error(a, b) < 1e-14
    ra = se.real_space_sum(s, 8.0, 0.4, se.Periodicity(3), threads=1)
    rb = se.real_space_sum(s, 8.0, 0.4, se.Periodicity(3), threads=4)
    assert se.relative_rms_error(ra, rb) < 1e-14


def test_xi_invariance_all_periodicities():
    s = rand_system(60, 1.0, 11)
    worst = 0.0
    for D in (0, 1, 2, 3):
        phis = []
        for xi in (4.0, 6.3, 8.0):
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                p, _ = se.auto_params(s, se.Periodicity(D), xi, 1e-10)
            phis.append(se.total_potential(s, p, se.Periodicity(D)))
        for i in range(3):
            for j in range(i + 1, 3):
                worst = max(worst, se.relative_rms_error(phis[i], phis[j]))
    assert worst <= 1e-9


def test_timings_keys():
    s = rand_system(500, 1.0, 3)
    p = se.SEParams(xi=8.0, rc=0.4, M=24, P=8, window="bm", shape=20.0, eps=1e-8)
    t = {}
    se.total_potential(s, p, se.Periodicity(3), timings=t)
    for k in ("realspace", "spread", "aft", "scale", "aift", "gather", "precompute"):
        assert k in t and t[k] >= 0.0


# ----------------------------------------------------------- device API

def test_device_api_matches_host_api():
    s = rand_system(5000, 2.0, 31)
    p = se.SEParams(xi=5.0, rc=0.6, M=32, P=8, window="bm", shape=20.0, eps=1e-8)
    host = se.total_potential(s, p, se.Periodicity(3))
    pos = torch.from_numpy(s.positions).cuda()
    q = torch.from_numpy(s.charges).cuda()
    dev = sedev.total_potential(pos, q, s.L, p, se.Periodicity(3)).cpu().numpy()
    assert se.relative_rms_error(dev, host) < 1e-14


def test_sharded_pipeline_single_process_world_splits():
    # the shard entry points, summed over ranks, reproduce the full potential
    from paper_1712_04732_b200 import _native
    s = rand_system(3000, 1.0, 41)
    p = se.SEParams(xi=8.0, rc=0.4, M=24, P=8, window="bm", shape=20.0, eps=1e-8)
    full = se.total_potential(s, p, se.Periodicity(3))
    pos = torch.from_numpy(s.positions).cuda()
    q = torch.from_numpy(s.charges).cuda()
    from paper_1712_04732_b200.distributed import NativeBackend
    be = NativeBackend(s.L, p, se.Periodicity(3), pos.device)
    world = 3
    grid = torch.zeros(be.shape, dtype=torch.float64, device=pos.device)
    for r in range(world):
        g = be.empty_grid()
        be.spread_shard(pos, q, r, world, g)
        grid += g
    be.kspace_apply(grid)
    phi = torch.zeros(3000, dtype=torch.float64, device=pos.device)
    for r in range(world):
        ph = be.empty_phi(3000)
        be.realspace_shard(pos, q, r, world, ph)
        be.gather_shard(grid, pos, r, world, ph)
        phi += ph
    assert se.relative_rms_error(phi.cpu().numpy(), full) < 1e-13


# --------------------------------------------- full-size (cfg2) properties

@pytest.fixture(scope="module")
def cfg2_full():
    rng = np.random.default_rng(2)
    N, L = 1_000_000, 10.0
    pos = rng.random((N, 3)) * L
    q = rng.uniform(-1, 1, N)
    q -= q.mean()
    p = se.SEParams(xi=4.2919, rc=1.0, M=128, P=8, window="bm", shape=20.0, eps=1e-8)
    return pos, q, L, p


def test_cfg2_full_size_realspace_sample_vs_oracle(cfg2_full):
    pos, q, L, p = cfg2_full
    s = se.ParticleSystem(pos, q, L)
    phir = se.real_space_sum(s, p.xi, p.rc, se.Periodicity(3))
    sel = np.random.default_rng(0).choice(len(q), 200, replace=False)
    ref = orc.realspace(pos, q, L, 3, p.xi, p.rc, targets=sel)
    assert se.relative_rms_error(phir[sel], ref) < 1e-13


def test_cfg2_full_size_linearity_and_translation(cfg2_full):
    pos, q, L, p = cfg2_full
    phi = se.total_potential(se.ParticleSystem(pos, q, L), p, se.Periodicity(3))
    phi2 = se.total_potential(se.ParticleSystem(pos, -2.0 * q, L), p, se.Periodicity(3))
    assert se.relative_rms_error(phi2, -2.0 * phi) < 1e-13
    # a shift by exactly 3 grid spacings (h = L/M) is a symmetry of the grid
    h = L / p.M
    sh = np.mod(pos + 3 * h, L)
    sh[sh >= L] = 0.0
    phi3 = se.total_potential(se.ParticleSystem(sh, q, L), p, se.Periodicity(3))
    assert se.relative_rms_error(phi3, phi) < 1e-11


# ------------------------------------------ BASELINE configs at full size

@pytest.mark.parametrize("name", ["cfg1", "cfg3", "cfg3_tol", "cfg4", "cfg5"])
def test_baseline_config_full_size(name):
    import sys as _sys
    _sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import workloads

    w = workloads.ALL[name]()
    pos, q, L, D = w["pos"], w["q"], w["L"], w["D"]
    p = se.SEParams(**w["prm"])
    peri = se.Periodicity(D)
    s = se.ParticleSystem(pos, q, L)
    t = {}
    phi = se.total_potential(s, p, peri, timings=t)
    assert np.all(np.isfinite(phi))
    phir = se.real_space_sum(s, p.xi, p.rc, peri)
    phik = se.se_kspace(s, p, peri)
    assert se.relative_rms_error(phi, phir + phik + se.self_term(q, p.xi)) < 1e-13
    rng = np.random.default_rng(7)
    sel = rng.choice(len(q), 64, replace=False)
    ref = orc.realspace(pos, q, L, D, p.xi, p.rc, targets=sel)
    assert se.relative_rms_error(phir[sel], ref) < 1e-12
    # k-space parity on a neutral subset with the same grid geometry
    sub = rng.choice(len(q), min(3000, len(q)), replace=False)
    qs = q[sub] - q[sub].mean()
    gk = se.se_kspace(se.ParticleSystem(pos[sub], qs, L), p, peri)
    rk = orc.se_kspace(pos[sub], qs, L, D, dict(p.__dict__))
    assert se.relative_rms_error(gk, rk) < 1e-11


def test_sharded_pipeline_nccl_single_rank():
    # the torch.distributed orchestration with a real NCCL communicator (1 rank)
    import socket

    import torch.distributed as dist
    from paper_1712_04732_b200.distributed import NativeBackend, total_potential_sharded

    s = rand_system(4000, 1.0, 43)
    p = se.SEParams(xi=8.0, rc=0.4, M=24, P=8, window="bm", shape=20.0, eps=1e-8)
    full = se.total_potential(s, p, se.Periodicity(3))
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        dev = torch.device("cuda", 0)
        pos = torch.from_numpy(s.positions).to(dev)
        q = torch.from_numpy(s.charges).to(dev)
        be = NativeBackend(s.L, p, se.Periodicity(3), dev)
        for mode in ("replicated", "slab"):
            phi = total_potential_sharded(pos, q, be, kspace=mode)
            assert se.relative_rms_error(phi.cpu().numpy(), full) < 1e-13, mode
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_slab_kspace_stages_virtual_ranks(world):
    # the slab-decomposed D = 3 k-space stage for `world` ranks, driven in one
    # process: each virtual rank's forward / x-pass / inverse run on the device
    # and the two all-to-all transposes are done by indexing (send block s of
    # rank r -> recv block r of rank s).  The assembled grid must equal the
    # replicated stage (se_kspace_apply_dev) on the same spread grid.
    from paper_1712_04732_b200.distributed import NativeBackend

    s = rand_system(6000, 2.0, 47)
    p = se.SEParams(xi=6.0, rc=0.5, M=32, P=8, window="bm", shape=20.0, eps=1e-8)
    dev = torch.device("cuda", 0)
    pos = torch.from_numpy(s.positions).to(dev)
    q = torch.from_numpy(s.charges).to(dev)
    be = NativeBackend(s.L, p, se.Periodicity(3), dev)
    grid = be.empty_grid()
    be.spread_shard(pos, q, 0, 1, grid)
    ref = grid.clone()
    be.kspace_apply(ref)
    nx, nky, nkz = be.slab_geometry(world)
    assert (nx, nky, nkz) == (32 // world, 32 // world, 17)
    send = [be.empty_spectrum(world) for _ in range(world)]
    for r in range(world):
        be.slab_forward(grid[r * nx:(r + 1) * nx].contiguous(), world, send[r])
    recv = [torch.stack([send[src][r] for src in range(world)]) for r in range(world)]
    for r in range(world):
        be.slab_xpass(recv[r], r, world)
    back = [torch.stack([recv[src][r] for src in range(world)]) for r in range(world)]
    out = torch.empty_like(grid)
    for r in range(world):
        slab = torch.empty((nx,) + tuple(grid.shape[1:]), dtype=torch.float64, device=dev)
        be.slab_inverse(back[r], world, slab)
        out[r * nx:(r + 1) * nx] = slab
    assert torch.max(torch.abs(out - ref)).item() <= 1e-13 * torch.max(torch.abs(ref)).item()


def test_slab_kspace_rejections():
    from paper_1712_04732_b200.distributed import NativeBackend

    dev = torch.device("cuda", 0)
    p = se.SEParams(xi=6.0, rc=0.5, M=24, P=8, window="bm", shape=20.0, eps=1e-8)
    be = NativeBackend(2.0, p, se.Periodicity(3), dev)
    with pytest.raises(ValueError):
        be.slab_geometry(5)  # 24 % 5 != 0
    p2 = se.SEParams(xi=6.0, rc=0.5, M=24, P=8, window="bm", shape=20.0, eps=1e-8, R=3.0)
    be2 = NativeBackend(2.0, p2, se.Periodicity(2), dev)
    with pytest.raises(ValueError):
        be2.slab_geometry(2)  # D = 2


def test_cuda_graph_replay_matches_eager_and_tracks_inputs():
    # repeated device-API calls with the same buffers replay a captured CUDA
    # graph (first call eager, second captured); results must equal the eager
    # path, follow in-place input changes, and re-capture on new buffers
    import torch

    s = rand_system(3000, 1.0, 31)
    p = se.SEParams(xi=8.0, rc=0.4, M=32, P=8, window="bm", shape=20.0, eps=1e-8)
    peri = se.Periodicity(3)
    dev = torch.device("cuda", 0)
    pos = torch.from_numpy(s.positions.copy()).to(dev)
    q = torch.from_numpy(s.charges.copy()).to(dev)
    out = torch.empty(s.N, dtype=torch.float64, device=dev)
    plan = sedev.plan(1.0, p, peri, dev)
    plan.set_graphs(False)
    eager = sedev.total_potential(pos, q, 1.0, p, peri, out=out).cpu().numpy().copy()
    plan.set_graphs(True)
    for _ in range(4):
        g = sedev.total_potential(pos, q, 1.0, p, peri, out=out).cpu().numpy()
        assert se.relative_rms_error(g, eager) < 1e-14
    q.mul_(-0.5)  # same buffers, new values: the replay must read them
    g = sedev.total_potential(pos, q, 1.0, p, peri, out=out).cpu().numpy()
    assert se.relative_rms_error(g, -0.5 * eager) < 1e-14
    out2 = torch.empty_like(out)  # new output buffer: re-warm, then capture again
    for _ in range(3):
        g2 = sedev.total_potential(pos, q, 1.0, p, peri, out=out2).cpu().numpy()
        assert se.relative_rms_error(g2, -0.5 * eager) < 1e-14
    plan.set_graphs(False)


# ------------------------------------ real-space geometry sweep vs the oracle

@pytest.mark.parametrize("D", [0, 1, 2, 3])
@pytest.mark.parametrize("L_over_rc,N", [(2.05, 400), (2.6, 900), (3.4, 1500), (6.9, 2500), (12.5, 6000),
                                          (12.5, 60000)])
def test_realspace_geometry_sweep(D, L_over_rc, N):
    # column binning edge cases: minimum-image columns (< 7 per axis), reach 2
    # / reach 3 columns, short and long columns, periodic z windows wrapping
    # on both sides, free axes clipped; plus a clustered case (tight cluster
    # straddling the periodic seam)
    rc = 0.37
    L = L_over_rc * rc
    rng = np.random.default_rng(int(100 * L_over_rc) + D + N)
    pos = rng.random((N, 3)) * L
    k = N // 5
    pos[:k] = np.mod(np.array([0.02, 0.5, 0.99]) * L + rng.normal(scale=0.05 * rc, size=(k, 3)), L)
    pos[pos >= L] = 0.0
    q = rng.uniform(-1, 1, N)
    q -= q.mean()
    s = se.ParticleSystem(pos, q, L)
    xi = 3.1 / rc
    phi = se.real_space_sum(s, xi, rc, se.Periodicity(D))
    sel = rng.choice(N, min(N, 300), replace=False)
    ref = orc.realspace(pos, q, L, D, xi, rc, targets=sel)
    assert se.relative_rms_error(phi[sel], ref) < 1e-12


@pytest.mark.parametrize("D", [3, 0])
@pytest.mark.parametrize("xi_rc", [2.0, 3.5, 4.2919, 4.6, 5.5])
def test_realspace_pair_term_every_degree_vs_oracle(D, xi_rc):
    # a dense system (dense and compacted batches both) at xi rc values that
    # select each degree of the polynomial pair term (20, 24, 28, 32) and the
    # erfc fallback (5.5): the device real-space sum against the oracle's
    # scipy-erfc evaluation of the reference's loop (realspace.py:100-126)
    rc = 0.5
    L = 8.0 * rc
    N = 40000
    rng = np.random.default_rng(int(10 * xi_rc) + D)
    pos = rng.random((N, 3)) * L
    q = rng.uniform(-1, 1, N)
    q -= q.mean()
    s = se.ParticleSystem(pos, q, L)
    xi = xi_rc / rc
    phi = se.real_space_sum(s, xi, rc, se.Periodicity(D))
    sel = rng.choice(N, 400, replace=False)
    ref = orc.realspace(pos, q, L, D, xi, rc, targets=sel)
    assert se.relative_rms_error(phi[sel], ref) < 1e-14


# ----------------------------------------------- randomized configurations

@pytest.mark.parametrize("case", range(24))
def test_randomized_configurations_vs_oracle(case):
    # seeded random (D, window, P incl. odd -- allowed for D = 0, 3 -- and
    # > 16, M, xi, L, N, clustering): the full device pipeline against the
    # CPU oracle
    rng = np.random.default_rng(1000 + case)
    D = int(rng.integers(0, 4))
    window = ["bm", "gaussian", "kb"][int(rng.integers(0, 3))]
    Ps = [4, 6, 8, 10, 12, 14, 18, 20] if D in (1, 2) else [3, 4, 5, 6, 7, 8, 10, 12, 17, 20]
    P = int(rng.choice(Ps))
    M = max(int(rng.choice([16, 18, 20, 24, 28])), P + P % 2)
    L = float(rng.choice([0.7, 1.0, 2.3]))
    N = int(rng.integers(40, 600))
    xi = float(rng.uniform(4.0, 9.0)) / L
    eps = 1e-10
    rc = math.sqrt(-math.log(eps)) / xi
    h = L / M
    d = 3.0 - D
    if D < 3:
        s0 = max(1.0 + math.sqrt(d), ((1.0 + math.sqrt(d)) * L + 2.0 * rc) / (L + P * h))
        R = 0.5 * (se.aft.padded_size(s0, M + P) * h - L + math.sqrt(d) * L)
    else:
        s0, R = 1.0, 0.0
    s_up = max(1.0, math.log(1.0 / eps) / (2 * math.pi)) if D in (1, 2) else 1.0
    nI = int(rng.integers(1, M // 2 + 1)) if D in (1, 2) else 0
    prm = se.SEParams(xi=xi, rc=rc, M=M, P=P, window=window, shape=windows.default_shape(window, P),
                      s0=s0, s=s_up, nI=nI, R=R, eps=eps)
    s = rand_system(N, L, 2000 + case)
    if case % 4 == 3:  # a tight cluster
        pos = s.positions.copy()
        pos[: N // 3] = np.mod(0.5 * L + rng.normal(scale=0.03 * L, size=(N // 3, 3)), L)
        pos[pos >= L] = 0.0
        s = se.ParticleSystem(pos, s.charges, L)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        phi = se.total_potential(s, prm, se.Periodicity(D))
    ref = orc.total_potential(s.positions, s.charges, L, D, dict(prm.__dict__))
    assert se.relative_rms_error(phi, ref) < 1e-11, (D, window, P, M, L, N)


@pytest.mark.parametrize("D", [0, 1, 2, 3])
def test_realspace_rank_shards_sum_to_full(D):
    # rank shards of the real-space path (contiguous ranges of the column
    # order, Newton source sides included, only the shard's units launched):
    # for any rank count their sum must equal the one-rank result
    from paper_1712_04732_b200.distributed import NativeBackend

    s = rand_system(120000, 4.0, 71 + D)
    p = se.SEParams(xi=6.0, rc=0.5, M=32, P=8, window="bm", shape=20.0, eps=1e-8,
                    R=0.0 if D == 3 else 9.0, s0=1.0 if D == 3 else 3.5)
    dev = torch.device("cuda", 0)
    pos = torch.from_numpy(s.positions).to(dev)
    q = torch.from_numpy(s.charges).to(dev)
    be = NativeBackend(s.L, p, se.Periodicity(D), dev)
    full = be.empty_phi(len(s.charges))
    be.realspace_shard(pos, q, 0, 1, full)
    be.finish()
    for world in (2, 3, 8):
        tot = torch.zeros_like(full)
        for r in range(world):
            ph = be.empty_phi(len(s.charges))
            be.realspace_shard(pos, q, r, world, ph)
            be.finish()
            tot += ph
        assert se.relative_rms_error(tot.cpu().numpy(), full.cpu().numpy()) < 1e-13, (D, world)
