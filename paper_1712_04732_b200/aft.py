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


# ------------------------------------------------------------------ FFT engine
class CuFftEngine:
    """The reference's FFT-engine plugin interface (aft.py:24-53: fftn, ifftn,
    rfftn, irfftn with numpy semantics -- unnormalised forward, 1/n inverse)
    on cuFFT through the C ABI.  Default engine of this package."""

    def __init__(self, device: int = 0):
        self.device = int(device)

    @staticmethod
    def _axes(ndim, axes):
        ax = sorted({a % ndim for a in (range(ndim) if axes is None else axes)})
        return ax

    def _c2c(self, a, axes, inverse):
        a = np.ascontiguousarray(a, dtype=np.complex128)
        ax = self._axes(a.ndim, axes)
        if not ax or a.size == 0:
            return a.copy()
        if ax != list(range(ax[0], ax[-1] + 1)):  # non-contiguous: one axis at a time
            for x in ax:
                a = self._c2c(a, (x,), inverse)
            return a
        out = np.empty_like(a)
        shape = (ctypes.c_int64 * a.ndim)(*a.shape)
        _native.call("se_fft_c2c_host", self.device, a.ndim, shape, ax[0], ax[-1], int(inverse),
                     _native.ptr(a), _native.ptr(out))
        return out

    def fftn(self, a, axes):
        return self._c2c(a, axes, False)

    def ifftn(self, a, axes):
        return self._c2c(a, axes, True)

    def rfftn(self, a, s, axes):
        a = np.asarray(a, dtype=np.float64)
        ax = self._axes(a.ndim, axes)
        if ax != list(range(ax[0], a.ndim)):
            raise NotImplementedError("rfftn over a trailing block of axes only")
        s = tuple(a.shape[x] for x in ax) if s is None else tuple(s)
        src = np.zeros(a.shape[:ax[0]] + s)
        cut = tuple(slice(0, min(a.shape[x], n)) for x, n in zip(ax, s))
        src[(Ellipsis,) + cut] = a[(Ellipsis,) + cut]
        out = np.empty(src.shape[:-1] + (src.shape[-1] // 2 + 1,), dtype=np.complex128)
        shape = (ctypes.c_int64 * src.ndim)(*src.shape)
        _native.call("se_fft_r2c_host", self.device, src.ndim, shape, ax[0], ax[-1], _native.ptr(src),
                     _native.ptr(out))
        return out

    def irfftn(self, a, s, axes):
        a = np.asarray(a, dtype=np.complex128)
        ax = self._axes(a.ndim, axes)
        if ax != list(range(ax[0], a.ndim)):
            raise NotImplementedError("irfftn over a trailing block of axes only")
        if s is None:
            s = tuple(a.shape[x] for x in ax[:-1]) + (2 * (a.shape[-1] - 1),)
        s = tuple(s)
        want = s[:-1] + (s[-1] // 2 + 1,)
        src = np.zeros(a.shape[:ax[0]] + want, dtype=np.complex128)
        cut = tuple(slice(0, min(a.shape[x], n)) for x, n in zip(ax, want))
        src[(Ellipsis,) + cut] = a[(Ellipsis,) + cut]
        out = np.empty(a.shape[:ax[0]] + s)
        shape = (ctypes.c_int64 * out.ndim)(*out.shape)
        _native.call("se_fft_c2r_host", self.device, out.ndim, shape, ax[0], ax[-1], _native.ptr(src),
                     _native.ptr(out))
        return out



# The reference's default engine (aft.py:24-41) by name.  Its contract is
# numpy's FFT semantics, which the cuFFT engine above implements.
NumpyFftEngine = CuFftEngine

_ENGINE = CuFftEngine()


def set_engine(engine) -> None:
    """Swap the FFT engine used by the stage functions below (aft.py:47-49)."""
    global _ENGINE
    _ENGINE = engine


def current_engine():
    return _ENGINE


# ------------------------------------------------------- stage functions
def _pad_to(arr, g, axes):
    if all(arr.shape[a] == g for a in axes):
        return arr
    shp = list(arr.shape)
    for a in axes:
        shp[a] = g
    out = np.zeros(shp, dtype=np.complex128)
    out[tuple(slice(0, arr.shape[i]) for i in range(arr.ndim))] = arr
    return out


def _rows(Hk, idx, D):
    return Hk[idx[:, 0], idx[:, 1]] if D == 2 else Hk[idx[:, 0]]


def periodic_stage(H, D: int):
    """Transform along the periodic axes only (aft.py:168-170)."""
    return _ENGINE.fftn(np.asarray(H, dtype=np.complex128), axes=tuple(range(D)))


def free_stage(Hk, partition: ModePartition, g0: int, gs: int):
    """Per-block padded transforms along the free axes (aft.py:173-190)."""
    D = partition.D
    faxes = tuple(range(1, 4 - D))
    zero = _ENGINE.fftn(_pad_to(Hk[(0,) * D][None], g0, faxes), axes=faxes)[0]
    Iblk = _ENGINE.fftn(_pad_to(_rows(Hk, partition.I_idx, D), gs, faxes), axes=faxes)
    Jblk = _ENGINE.fftn(np.ascontiguousarray(_rows(Hk, partition.J_idx, D)), axes=faxes)
    return zero, Iblk, Jblk


def aft_forward(H, partition, s0: float, s: float, periodicity) -> SpectralField:
    """Adaptive Fourier transform of a grid field (aft.py:193-223)."""
    D = periodicity.D
    H = np.asarray(H)
    if D == 3:
        M = H.shape[0]
        return SpectralField(D, M, M, M, M, full=_ENGINE.fftn(H.astype(np.complex128), axes=(0, 1, 2)))
    Mt = H.shape[-1]
    if D == 0:
        g0 = padded_size(s0, Mt)
        return SpectralField(D, 0, Mt, g0, Mt,
                             zero=_ENGINE.fftn(_pad_to(H.astype(np.complex128), g0, (0, 1, 2)), axes=(0, 1, 2)))
    if partition is None:
        raise ValueError("D in {1,2} requires a mode partition")
    if Mt % 2:
        raise ValueError("free-axis grid size must be even")
    g0, gs = padded_size(s0, Mt), padded_size(s, Mt)
    zero, Iblk, Jblk = free_stage(periodic_stage(H, D), partition, g0, gs)
    return SpectralField(D, partition.M, Mt, g0, gs, zero=zero, Iblk=Iblk, Jblk=Jblk,
                         I_idx=partition.I_idx, J_idx=partition.J_idx)


def aft_inverse(F: SpectralField, partition, M: int, periodicity) -> np.ndarray:
    """Inverse of aft_forward; returns the complex grid field (aft.py:226-265)."""
    D = periodicity.D
    if D == 3:
        return _ENGINE.ifftn(F.full, axes=(0, 1, 2))
    Mt = F.Mt
    if D == 0:
        return _ENGINE.ifftn(F.zero, axes=(0, 1, 2))[:Mt, :Mt, :Mt]
    if partition is None:
        raise ValueError("D in {1,2} requires a mode partition")
    if F.Iblk.shape[0] != len(partition.I_idx) or F.Jblk.shape[0] != len(partition.J_idx):
        raise ValueError("spectral blocks do not match the mode partition")
    nfree = 3 - D
    faxes = tuple(range(1, 1 + nfree))
    cut = (slice(None),) + (slice(0, Mt),) * nfree
    out = np.zeros((M,) * D + (Mt,) * nfree, dtype=np.complex128)
    out[(0,) * D] = _ENGINE.ifftn(F.zero[None], axes=faxes)[cut][0]
    Ib = _ENGINE.ifftn(F.Iblk, axes=faxes)[cut]
    Jb = _ENGINE.ifftn(F.Jblk, axes=faxes)[cut]
    if D == 2:
        out[partition.I_idx[:, 0], partition.I_idx[:, 1]] = Ib
        out[partition.J_idx[:, 0], partition.J_idx[:, 1]] = Jb
    else:
        out[partition.I_idx[:, 0]] = Ib
        out[partition.J_idx[:, 0]] = Jb
    return _ENGINE.ifftn(out, axes=tuple(range(D)))


def transformed_points(partition: ModePartition, Mt: int, g0: int, gs: int) -> dict:
    """Free-axis transform sizes, adaptive vs fully upsampled (aft.py:268-275)."""
    f = 3 - partition.D
    _, ni, nj = partition.counts
    zero, I, J = g0 ** f, ni * gs ** f, nj * Mt ** f
    return {"zero": zero, "I": I, "J": J, "adaptive": zero + I + J,
            "full_upsampled": partition.M ** partition.D * gs ** f}
