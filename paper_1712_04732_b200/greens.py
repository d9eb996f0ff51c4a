"""Truncated free-space Green's functions on the zero periodic-mode block
(mirror of pmewald.greens).  Values come from the library routine the
device multiplier mirrors (`se_greens_zero_mode`, greens.py:48-85),
including the reference's D=2 sign convention (greens.py:75-82).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native


@dataclass(frozen=True)
class GreensSpec:
    D: int
    R: float = 0.0

    def __post_init__(self):
        if self.D not in (0, 1, 2, 3):
            raise ValueError("D must be in {0,1,2,3}")
        if self.D < 3 and self.R <= 0:
            raise ValueError("R must be positive for D < 3")


def default_truncation_radius(D: int, Lt: float) -> float:
    """sqrt(3 - D) Lt (greens.py:41-45)."""
    if D not in (0, 1, 2, 3):
        raise ValueError("D must be in {0,1,2,3}")
    return math.sqrt(3.0 - D) * Lt


def zero_mode_values(D: int, R: float, kappa) -> np.ndarray:
    """Kernel on the zero periodic-mode block as a function of |kappa|."""
    if D not in (0, 1, 2):
        raise ValueError("zero-mode kernel is defined for D < 3")
    arr = np.asarray(kappa, dtype=float)
    flat = np.ascontiguousarray(arr.ravel())
    out = np.empty_like(flat)
    _native.call("se_greens_zero_mode", int(D), float(R), _native.ptr(flat), flat.size, _native.ptr(out))
    return out.reshape(arr.shape)


def zero_point_value(D: int, R: float) -> float:
    """Exact k = 0 limits (greens.py:88-96)."""
    return {3: 0.0, 0: 0.5 * R * R, 1: 0.25 * R * R * (1.0 - 2.0 * math.log(R)),
            2: -0.5 * R * R}[D]


def greens_hat(kvec, spec: GreensSpec) -> float:
    """Scalar kernel value at one wavevector (greens.py:99-118)."""
    k = np.asarray(kvec, dtype=float)
    if k.shape != (3,):
        raise ValueError("kvec must be a 3-vector")
    k2 = float(k @ k)
    if np.any(k[: spec.D] != 0.0):
        return 1.0 / k2
    if spec.D == 3:
        return 0.0
    kappa = math.sqrt(float(k[spec.D:] @ k[spec.D:]))
    if kappa == 0.0:
        return zero_point_value(spec.D, spec.R)
    return float(zero_mode_values(spec.D, spec.R, np.array([kappa]))[0])
