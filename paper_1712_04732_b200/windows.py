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


def gaussian_fourier(k, spec: WindowSpec):
    """exp(-(w k)^2 / (2 m^2)): the untruncated Gaussian transform (windows.py:87-91)."""
    return fourier(k, WindowSpec(GAUSSIAN, spec.P, spec.h, spec.shape))


def kaiser_fourier(k, spec: WindowSpec):
    """2w sinhc(beta^2 - (k w)^2) / I0(beta) (windows.py:135-145)."""
    return fourier(k, WindowSpec(KAISER, spec.P, spec.h, spec.shape))


def _sinhc(rho2) -> np.ndarray:
    """sinh(sqrt(rho2))/sqrt(rho2), continued to rho2 < 0 (windows.py:115-132)."""
    arr = np.ascontiguousarray(np.asarray(rho2, dtype=float).ravel())
    out = np.empty_like(arr)
    _native.call("se_kb_sinhc", _native.ptr(arr), arr.size, _native.ptr(out))
    return out.reshape(np.shape(rho2))


def _bm_quadrature(w: float, beta: float, k, nodes: int) -> np.ndarray:
    """BM transform by an n-node long-double Gauss-Legendre rule (windows.py:202-211)."""
    kk = np.ascontiguousarray(np.asarray(k, dtype=float).ravel())
    out = np.empty_like(kk)
    _native.call("se_bm_quadrature", float(w), float(beta), _native.ptr(kk), kk.size, int(nodes),
                 _native.ptr(out))
    return out


def eval_bspline(x, p: int):
    """Cardinal B-spline M_p supported on [0, p] (windows.py:94-103).

    Not a spreading window of this package (the reference's pipeline never
    selects it); kept for API completeness.  Evaluated piecewise from the
    order-2 hat by the Cox-de Boor recursion, iteratively over the order.
    """
    if p < 2:
        raise ValueError("B-spline order must be >= 2")
    x = np.asarray(x, dtype=float)
    # values of M_2(x - j) for the shifts the recursion needs, j = 0..p-2
    layers = [np.where((x - j >= 0.0) & (x - j <= 2.0), 1.0 - np.abs(x - j - 1.0), 0.0)
              for j in range(p - 1)]
    for order in range(3, p + 1):
        layers = [((x - j) * layers[j] + (order - (x - j)) * layers[j + 1]) / (order - 1)
                  for j in range(len(layers) - 1)]
    out = layers[0]
    return float(out) if out.ndim == 0 else out


@dataclass(frozen=True)
class TabulatedTransform:
    """A window transform sampled on one mode set (windows.py:158-166)."""

    kind: str
    P: int
    shape: float
    w: float
    k: np.ndarray
    values: np.ndarray


_BM_TABLES: dict[tuple, TabulatedTransform] = {}


def bm_fourier_precompute(spec: WindowSpec, k) -> TabulatedTransform:
    """BM transform tabulated at exactly the modes k, quadrature self-checked by
    node doubling inside the library; cached per (beta, w, mode set)
    (windows.py:214-239)."""
    if spec.kind != BM:
        raise ValueError("spec.kind must be 'bm'")
    k = np.ascontiguousarray(k, dtype=float)
    key = (float(spec.shape), float(spec.w), k.tobytes())
    hit = _BM_TABLES.get(key)
    if hit is not None:
        return hit
    table = TabulatedTransform(BM, spec.P, spec.shape, spec.w, k.copy(), fourier(k, spec))
    _BM_TABLES[key] = table
    return table
