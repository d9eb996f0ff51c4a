"""The field (forces) oracle against the reference: central differences of
the reference's own real_space_sum and oracle.kspace_direct_3p
(tests/golden/make_field_golden.py -> field.npz).  CPU only."""

import os
import sys

import numpy as np

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
