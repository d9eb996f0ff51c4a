"""Window functions and their Fourier transforms (mirror of pmewald.windows).

The hot path evaluates windows inside the spreading / gathering kernels on
the device.  The functions here expose the same values to callers and tests
through the library's planning routines (`se_window_eval`,
`se_window_fourier`, the latter with the long-double Gauss-Legendre BM
transform of windows.py:175-239), i.e. exactly the tables the device
multiplier uses.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native

GAUSSIAN = "gaussian"
KAISER = "kb"
BM = "bm"
KINDS = (GAUSSIAN, KAISER, BM)


@dataclass(frozen=True)
class WindowSpec:
    """1-D window on a grid of spacing h: half width w = P h / 2 (windows.py:30-61)."""

    kind: str
    P: int
    h: float
    shape: float

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"unknown window kind {self.kind!r}")
        if self.P < 1 or self.h <= 0 or self.shape <= 0:
            raise ValueError("invalid window parameters")

    @property
    def w(self) -> float:
        return 0.5 * self.P * self.h

    def eta(self, xi: float) -> float:
        if self.kind != GAUSSIAN:
            raise ValueError("eta is defined for the Gaussian window only")
        return (2.0 * self.w * xi / self.shape) ** 2


def default_shape(kind: str, P: int) -> float:
    """sqrt(pi P) for the Gaussian, 2.5 P for KB / BM (windows.py:63-71)."""
    if P < 1:
        raise ValueError("P must be >= 1")
    if kind == GAUSSIAN:
        return math.sqrt(math.pi * P)
    if kind in (KAISER, BM):
        return 2.5 * P
    raise ValueError(f"unknown window kind {kind!r}")


def _apply(fn: str, values, spec: WindowSpec) -> np.ndarray:
    arr = np.asarray(values, dtype=float)
    flat = np.ascontiguousarray(arr.ravel())
    out = np.empty_like(flat)
    _native.call(fn, _native.WINDOWS[spec.kind], int(spec.P), float(spec.h), float(spec.shape),
                 _native.ptr(flat), flat.size, _native.ptr(out))
    return out.reshape(arr.shape)


def evaluate(x, spec: WindowSpec) -> np.ndarray:
    """Real-space window values at offsets x (windows.py:242-248)."""
    return _apply("se_window_eval", x, spec)


def fourier(k, spec: WindowSpec) -> np.ndarray:
    """Window Fourier transform at wavenumbers k (windows.py:251-257)."""
    return _apply("se_window_fourier", k, spec)


def eval_gaussian(x, spec: WindowSpec):
    return evaluate(x, WindowSpec(GAUSSIAN, spec.P, spec.h, spec.shape))


def eval_kaiser(x, spec: WindowSpec):
    return evaluate(x, WindowSpec(KAISER, spec.P, spec.h, spec.shape))


def eval_bm(x, spec: WindowSpec):
    return evaluate(x, WindowSpec(BM, spec.P, spec.h, spec.shape))
