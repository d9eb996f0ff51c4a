"""Real-space Ewald sum and self term (mirror of pmewald.realspace).

real_space_sum runs the library's cell-list erfc kernel
(csrc/se_realspace.cu; explicit images when rc > L/2 on a periodic axis,
realspace.py:138-165); self_term runs the library's elementwise kernel.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .core import ParticleSystem, Periodicity, SEParams


def _real_params(xi: float, rc: float) -> SEParams:
    # only xi and rc enter the real-space sum; the grid fields are placeholders
    return SEParams(xi=float(xi), rc=float(rc), M=2, P=2, window="bm", shape=5.0,
                    s0=1.0, s=1.0, nI=0, R=1.0)


def real_space_sum(system: ParticleSystem, xi: float, rc: float, periodicity: Periodicity,
                   threads: int = 1) -> np.ndarray:
    """sum over pairs / images within rc of q_n erfc(xi r)/r (realspace.py:168-180)."""
    if xi <= 0 or rc <= 0:
        raise ValueError("xi and rc must be positive")
    plan = _native.plan_for(periodicity.D, system.L, _real_params(xi, rc))
    phi = np.empty(system.N)
    _native.call("se_realspace_host", plan.handle, _native.ptr(system.positions),
                 _native.ptr(system.charges), system.N, _native.ptr(phi), 0)
    return phi


def self_term(q, xi: float) -> np.ndarray:
    """-2 xi q / sqrt(pi) (realspace.py:183-185)."""
    qa = np.ascontiguousarray(np.asarray(q, dtype=float))
    out = np.empty_like(qa)
    _native.call("se_self_term_host", _native.ptr(qa), qa.size, float(xi), _native.ptr(out))
    return out
