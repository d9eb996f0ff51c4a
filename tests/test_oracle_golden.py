"""Pin the CPU oracle (oracle/se_oracle.py) against the reference's own outputs.

The golden vectors were produced by the unmodified reference
(tests/golden/make_golden.py); these tests prove the restatement before it
is trusted as the GPU parity checker.  CPU only.
"""

import math
import os

import numpy as np
import pytest

import se_oracle as orc
from conftest import GOLDEN, load_case


def rms(a, b):
    return orc.relative_rms(a, b)


def test_pipeline_stages_match_reference(golden_case):
    name, c = golden_case
    prm, D, L = c["prm"], c["D"], c["L"]
    g = orc.geometry(L, D, prm["M"], prm["P"], prm["s0"], prm["s"], prm["R"])
    assert (g["g0"], g["gs"], g["Mt"]) == (int(c["g0"]), int(c["gs"]), int(c["Mt"]))
    H = orc.spread(c["pos"], c["q"], g, prm["window"], prm["shape"])
    assert H.shape == c["H"].shape
    assert np.max(np.abs(H - c["H"])) <= 1e-13 * np.max(np.abs(c["H"]))
    uk = None if c["use_kernel"] < 0 else bool(c["use_kernel"])
    phik = orc.se_kspace(c["pos"], c["q"], L, D, prm, use_kernel=uk)
    assert rms(phik, c["phi_k"]) < 1e-12
    if "phi_r" in c:
        phir = orc.realspace(c["pos"], c["q"], L, D, prm["xi"], prm["rc"])
        assert np.allclose(phir, c["phi_r"], rtol=1e-13, atol=1e-13)
        phis = orc.self_term(c["q"], prm["xi"])
        assert np.array_equal(phis, c["phi_s"])
        assert rms(phir + phik + phis, c["phi"]) < 1e-12


def test_realspace_paths_match_reference():
    z = np.load(os.path.join(GOLDEN, "realspace.npz"))
    for D, rc in ((3, 1.2), (2, 0.8), (1, 0.7)):
        got = orc.realspace(z["img_pos"], z["img_q"], 1.0, D, 4.0, rc)
        assert np.allclose(got, z[f"img_d{D}"], rtol=1e-13, atol=1e-14)
    for D in (0, 1, 2, 3):
        got = orc.realspace(z["cell_pos"], z["cell_q"], 1.0, D, 7.0, 0.23)
        assert np.allclose(got, z[f"cell_d{D}"], rtol=1e-13, atol=1e-14)
        got = orc.realspace(z["cell_pos"], z["cell_q"], 1.0, D, 5.0, 0.45)
        assert np.allclose(got, z[f"cell2_d{D}"], rtol=1e-13, atol=1e-14)


def test_realspace_target_subset():
    z = np.load(os.path.join(GOLDEN, "realspace.npz"))
    sel = np.arange(0, 600, 7)
    got = orc.realspace(z["cell_pos"], z["cell_q"], 1.0, 3, 7.0, 0.23, targets=sel)
    assert np.allclose(got, z["cell_d3"][sel], rtol=1e-13, atol=1e-14)


def test_window_and_greens_tables():
    z = np.load(os.path.join(GOLDEN, "tables.npz"))
    h = 1.0 / 24
    for kind, P, shape in (("bm", 8, 20.0), ("bm", 10, 25.0), ("bm", 16, 40.0),
                           ("gaussian", 12, math.sqrt(12 * math.pi)), ("kb", 8, 20.0)):
        w = 0.5 * P * h
        for n in (24, 70, 210):
            got = orc.window_fourier(kind, shape, w, orc.wavenumbers(n, h))
            want = z[f"wf_{kind}_{P}_{n}"]
            assert np.max(np.abs(got - want)) <= 1e-15 * np.max(np.abs(want))
        x = np.linspace(-w * 1.1, w * 1.1, 101)
        assert np.array_equal(orc.window_eval(kind, shape, w, x), z[f"we_{kind}_{P}"])
    for D in (0, 1, 2):
        for R in (1.7, 3.2):
            assert np.array_equal(orc.greens_zero_block(D, R, z["kappa"]), z[f"g_{D}_{R}"])


def test_d0_kernel_table():
    z = np.load(os.path.join(GOLDEN, "d0_kernel.npz"))
    tab, kg = orc.d0_kernel_table(1.0, 16, 8, 1 + math.sqrt(3.0), 0.5)
    assert kg["nconv"] == int(z["nconv"]) and kg["g0"] == int(z["g0"])
    assert kg["R"] == float(z["R"])
    assert np.max(np.abs(tab - z["ghat"])) <= 1e-13 * np.max(np.abs(z["ghat"]))


def test_padded_size_and_partition_known_answers():
    # aft.py:76-84 known answers (test_aft.py:16-26)
    assert orc.padded_size(1.0, 44) == 44
    assert orc.padded_size(2.0, 44) == 90
    I_idx, J_idx = orc.mode_partition(64, 2, 7)
    assert len(I_idx) == 15 * 15 - 1 and len(J_idx) == 64 * 64 - 15 * 15
    with pytest.raises(ValueError):
        orc.padded_size(0.5, 10)


def test_direct_sums_match_reference():
    z = np.load(os.path.join(GOLDEN, "direct.npz"))
    for i in range(2):
        N, L, xi, kmax, _ = z[f"d3_{i}_in"]
        phi = orc.direct_kspace_3p(z[f"d3_{i}_pos"], z[f"d3_{i}_q"], L, xi, int(kmax))
        assert rms(phi, z[f"d3_{i}_phi"]) < 1e-13
        sub = np.array([0, 3, 7])
        part = orc.direct_kspace_3p(z[f"d3_{i}_pos"], z[f"d3_{i}_q"], L, xi, int(kmax), targets=sub)
        assert np.allclose(part, z[f"d3_{i}_phi"][sub], rtol=1e-12, atol=1e-13)
        N, L, xi, _ = z[f"d0_{i}_in"]
        phi = orc.direct_kspace_0p(z[f"d0_{i}_pos"], z[f"d0_{i}_q"], xi)
        assert rms(phi, z[f"d0_{i}_phi"]) < 1e-14
        N, L, xi, kmax, _ = z[f"d2_{i}_in"]
        phi = orc.direct_kspace_2p(z[f"d2_{i}_pos"], z[f"d2_{i}_q"], L, xi, int(kmax))
        assert rms(phi, z[f"d2_{i}_phi"]) < 1e-12
