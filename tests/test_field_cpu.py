"""The field (forces) oracle against the reference: central differences of
the reference's own real_space_sum and oracle.kspace_direct_3p
(tests/golden/make_field_golden.py -> field.npz).  CPU only."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import se_oracle as orc  # noqa: E402

G = np.load(os.path.join(ROOT, "tests", "golden", "field.npz"))


def _rel(a, b):
    return np.sqrt(np.mean((a - b) ** 2)) / np.sqrt(np.mean(b ** 2))


def test_realspace_field_matches_reference_differences():
    E = orc.realspace_field(G["pos"], G["q"], float(G["L"]), 3, float(G["xi"]), float(G["rc"]))
    assert _rel(E, G["E_real_fd"]) < 1e-8


def test_direct_field_matches_reference_differences():
    E = orc.direct_field_3p(G["pos"], G["q"], float(G["L"]), float(G["xi"]), int(G["kmax"]))
    assert _rel(E, G["E_kspace_direct_fd"]) < 1e-8


def test_se_kspace_field_converges_to_direct():
    prm = dict(xi=float(G["xi"]), rc=float(G["rc"]), M=32, P=16, window="gaussian", shape=np.sqrt(16 * np.pi))
    E = orc.kspace_field_d3(G["pos"], G["q"], float(G["L"]), prm)
    assert _rel(E, G["E_kspace_direct_fd"]) < 1e-7


G3 = np.load(os.path.join(ROOT, "tests", "golden", "field_dlt3.npz"))


def _tight(D, pos, q, L, xi, window):
    import paper_1712_04732_b200 as se
    s = se.ParticleSystem(pos, q, L)
    p, _ = se.auto_params(s, se.Periodicity(D), xi, 1e-13, window=window)
    return dict(p.__dict__), p


@pytest.mark.parametrize("D", [2, 1, 0])
def test_realspace_field_dlt3_matches_reference_differences(D):
    L, xi, rc, kmax, delta = G3[f"D{D}_prm"]
    E = orc.realspace_field(G3[f"D{D}_pos"], G3[f"D{D}_q"], L, D, xi, rc)
    assert _rel(E, G3[f"D{D}_E_real_fd"]) < 1e-7


@pytest.mark.parametrize("D,window", [(2, "gaussian"), (1, "gaussian"), (0, "gaussian"), (2, "kb"), (0, "kb")])
def test_gradient_gather_field_dlt3_converges_to_direct(D, window):
    # E_F by the gradient of the gather (any D) with tight parameters against
    # central differences of the reference's own direct Fourier-space sums
    L, xi, rc, kmax, delta = G3[f"D{D}_prm"]
    pos, q = G3[f"D{D}_pos"], G3[f"D{D}_q"]
    prm, _ = _tight(D, pos, q, L, xi, window)
    E = orc.kspace_field_grad(pos, q, L, D, prm)
    err = _rel(E, G3[f"D{D}_E_kspace_direct_fd"])
    print(f"D={D} {window}: gradient-gather field vs reference differences {err:.2e}")
    assert err < 1e-6
