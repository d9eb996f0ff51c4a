"""Adaptive-FFT planning (mirror of the planning half of pmewald.aft).

The transforms themselves run inside the SE B200 library's k-space stage
(csrc/se_kspace.cu: batched cuFFT over the zero / I / J blocks).  This
module keeps the reference's integer planning API -- padded sizes, signed
mode integers, the max-norm mode partition and the transformed-point
accounting -- with the padded-size rules evaluated by the same library
routine the device plan uses (aft.py:61-84).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native


def mode_integers(M: int) -> np.ndarray:
    """Signed FFT-order mode indices 0..M/2-1, -M/2..-1 (aft.py:56-58)."""
    j = np.arange(M)
    return np.where(j < (M + 1) // 2, j, j - M)


def next_even_smooth(n: int) -> int:
    """Smallest even 7-smooth integer >= n (aft.py:68-73)."""
    out = ctypes.c_int32()
    _native.call("se_next_even_smooth", int(n), ctypes.byref(out))
    return int(out.value)


def padded_size(s: float, n: int) -> int:
    """Even 7-smooth size >= s*n, or n when no padding is needed (aft.py:76-84)."""
    out = ctypes.c_int32()
    _native.call("se_padded_size", float(s), int(n), ctypes.byref(out))
    return int(out.value)


@dataclass(frozen=True)
class ModePartition:
    """Zero / I / J split of the periodic modes by max-norm (aft.py:87-121)."""

    M: int
    D: int
    nI: int
    I_idx: np.ndarray
    J_idx: np.ndarray

    @classmethod
    def build(cls, M: int, D: int, nI: int) -> "ModePartition":
        if D not in (1, 2):
            raise ValueError("mode partitions apply to D in {1,2}")
        if not 0 <= nI <= M // 2:
            raise ValueError("nI must lie in [0, M/2]")
        a = np.abs(mode_integers(M))
        mu = a if D == 1 else np.maximum.outer(a, a)
        part = cls(M, D, nI, np.argwhere((mu > 0) & (mu <= nI)), np.argwhere(mu > nI))
        assert 1 + len(part.I_idx) + len(part.J_idx) == M ** D, "mode partition must be exact"
        return part

    @property
    def counts(self) -> tuple[int, int, int]:
        return 1, len(self.I_idx), len(self.J_idx)


@dataclass
class SpectralField:
    """Fourier coefficients grouped by upsampling block (aft.py:124-152)."""

    D: int
    M: int
    Mt: int
    g0: int
    gs: int
    zero: np.ndarray | None = None
    Iblk: np.ndarray | None = None
    Jblk: np.ndarray | None = None
    I_idx: np.ndarray | None = None
    J_idx: np.ndarray | None = None
    full: np.ndarray | None = None

    @property
    def s0_eff(self) -> float:
        return self.g0 / self.Mt

    @property
    def s_eff(self) -> float:
        return self.gs / self.Mt


def transformed_points(partition: ModePartition, Mt: int, g0: int, gs: int) -> dict:
    """Free-axis transform sizes, adaptive vs fully upsampled (aft.py:268-275)."""
    f = 3 - partition.D
    _, ni, nj = partition.counts
    zero, I, J = g0 ** f, ni * gs ** f, nj * Mt ** f
    return {"zero": zero, "I": I, "J": J, "adaptive": zero + I + J,
            "full_upsampled": partition.M ** partition.D * gs ** f}
