"""Direct Ewald sums on the device (mirror of the evaluators in pmewald.oracle).

The reference ships independently coded, slow evaluators for validating the
SE method (oracle.py).  Its direct Fourier-space sums for every periodicity
are the natural large-N checks of this package's SE path and run here as
CUDA kernels of the SE B200 library (csrc/se_direct.cu):

  * kspace_direct_3p  (oracle.py:109-118): the Ewald Fourier sum over all
    integer modes |n_a| <= kmax (structure factors + per-target mode sum);
  * kspace_direct_2p  (oracle.py:120-153): the closed-form doubly periodic
    sum (per-mode erfc form in its overflow-safe erfcx variant + zero mode);
  * kspace_direct_1p  (oracle.py:156-178): the singly periodic sum
    (incomplete Bessel K0 by Gauss-Legendre quadrature, log + E1 zero mode);
  * kspace_direct_0p  (oracle.py:181-192): the free-space complement
    sum q erf(xi r)/r plus the self limit.

All accept `targets` (indices into the system) so that a full-size system
(all N sources) can be checked at a sample of targets.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native
from .core import ParticleSystem, Periodicity


@dataclass(frozen=True)
class OracleConfig:
    """kmax per periodic axis for a target accuracy (oracle.py:25-36)."""

    kmax: int
    image_layers: int = 32
    quad_tol: float = 1e-13

    @classmethod
    def for_accuracy(cls, xi: float, L: float, eps: float) -> "OracleConfig":
        kmax = int(np.ceil(xi * L * np.sqrt(-np.log(eps)) / np.pi)) + 1
        return cls(kmax=kmax, quad_tol=min(1e-13, eps / 100.0))


def _targets(system: ParticleSystem, targets):
    if targets is None:
        return None, system.N
    t = np.ascontiguousarray(np.asarray(targets, dtype=np.int64).ravel())
    return t, t.size


def kspace_direct_3p(system: ParticleSystem, xi: float, kmax: int, targets=None) -> np.ndarray:
    """(4 pi / L^3) sum_{0 < |n|_inf <= kmax} e^{-k^2/4xi^2}/k^2 Re(e^{i k.x_m} S_k)."""
    t, T = _targets(system, targets)
    phi = np.empty(T)
    _native.call("se_direct_kspace_3p_host", _native.ptr(system.positions), _native.ptr(system.charges),
                 system.N, float(system.L), float(xi), int(kmax),
                 _native.ptr(t) if t is not None else None, T, _native.ptr(phi))
    return phi


def kspace_direct_2p(system: ParticleSystem, xi: float, kmax: int, targets=None) -> np.ndarray:
    """Closed-form doubly periodic Fourier sum (per-mode erfc form + zero mode),
    oracle.py:134-153; periodic axes x, y."""
    t, T = _targets(system, targets)
    phi = np.empty(T)
    _native.call("se_direct_kspace_2p_host", _native.ptr(system.positions), _native.ptr(system.charges),
                 system.N, float(system.L), float(xi), int(kmax),
                 _native.ptr(t) if t is not None else None, T, _native.ptr(phi))
    return phi


def kspace_direct_1p(system: ParticleSystem, xi: float, kmax: int, targets=None) -> np.ndarray:
    """Singly periodic Fourier sum (oracle.py:156-178): incomplete Bessel K0
    per mode (quadrature on the device), log + E1 zero mode; periodic axis x.
    SingularConfigurationError if two charges share transverse coordinates."""
    t, T = _targets(system, targets)
    phi = np.empty(T)
    _native.call("se_direct_kspace_1p_host", _native.ptr(system.positions), _native.ptr(system.charges),
                 system.N, float(system.L), float(xi), int(kmax),
                 _native.ptr(t) if t is not None else None, T, _native.ptr(phi))
    return phi


def kspace_direct_0p(system: ParticleSystem, xi: float, targets=None) -> np.ndarray:
    """sum_{n != m} q_n erf(xi r)/r + q_m 2 xi / sqrt(pi); SingularConfigurationError
    for coincident distinct particles."""
    t, T = _targets(system, targets)
    phi = np.empty(T)
    _native.call("se_direct_kspace_0p_host", _native.ptr(system.positions), _native.ptr(system.charges),
                 system.N, float(xi), _native.ptr(t) if t is not None else None, T, _native.ptr(phi))
    return phi


def kspace_direct(system: ParticleSystem, xi: float, periodicity: Periodicity, kmax: int,
                  targets=None) -> np.ndarray:
    """Dispatch by periodicity (oracle.py:195-204)."""
    if periodicity.D == 3:
        return kspace_direct_3p(system, xi, kmax, targets)
    if periodicity.D == 2:
        return kspace_direct_2p(system, xi, kmax, targets)
    if periodicity.D == 1:
        return kspace_direct_1p(system, xi, kmax, targets)
    return kspace_direct_0p(system, xi, targets)


def self_limit(q, xi: float) -> np.ndarray:
    """q 2 xi / sqrt(pi): the r -> 0 limit of q erf(xi r)/r (oracle.py:191)."""
    return np.asarray(q, dtype=float) * (2.0 * xi / math.sqrt(math.pi))
