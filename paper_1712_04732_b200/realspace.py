"""Real-space Ewald sum and self term (mirror of pmewald.realspace).

real_space_sum runs the library's cell-list erfc kernel
(csrc/se_realspace.cu; explicit images when rc > L/2 on a periodic axis,
realspace.py:138-165); self_term runs the library's elementwise kernel.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .core import ParticleSystem, Periodicity, SEParams


@dataclass(frozen=True)
class CellList:
    """Particles bucketed into n^3 cells of edge >= rc (realspace.py:24-40);
    members[flat cell] lists each particle exactly once."""

    ncells: tuple[int, int, int]
    edge: float
    members: list[np.ndarray]
    periodic_mask: tuple[bool, bool, bool]
    rc: float

    def flat(self, cx: int, cy: int, cz: int) -> int:
        nx, ny, nz = self.ncells
        return (cx * ny + cy) * nz + cz


def build_cell_list(system: ParticleSystem, rc: float, periodicity: Periodicity) -> CellList:
    """Cell list with edge L / floor(L / rc) (realspace.py:43-59), built by the
    library's counting sort (se_cell_list_host).  An inspection utility: the
    device real-space kernel bins into z-sorted columns of edge rc/3."""
    if rc <= 0:
        raise ValueError("rc must be positive")
    if periodicity.D >= 1 and rc > system.L / 2 + 1e-12:
        raise ValueError("cell list requires rc <= L/2 on periodic axes (minimum image)")
    n = max(1, int(np.floor(system.L / rc)))
    order = np.empty(system.N, dtype=np.int64)
    bounds = np.empty(n ** 3 + 1, dtype=np.int64)
    _native.call("se_cell_list_host", _native.ptr(system.positions), system.N, float(system.L), n,
                 _native.ptr(order), _native.ptr(bounds))
    members = [order[bounds[c]:bounds[c + 1]] for c in range(n ** 3)]
    return CellList((n, n, n), system.L / n, members, periodicity.mask, float(rc))


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
    phi = _native.host_out(system.N)
    _native.call("se_realspace_host", plan.handle, _native.ptr(system.positions),
                 _native.ptr(system.charges), system.N, _native.ptr(phi), 0)
    return phi


def real_space_field(system: ParticleSystem, xi: float, rc: float, periodicity: Periodicity,
                     threads: int = 1) -> np.ndarray:
    """Real-space part of E = -grad phi, (N, 3): sum over the pairs / images
    of real_space_sum of q_n (erfc(xi r)/r + 2 xi/sqrt(pi) e^{-xi^2 r^2})
    (x_m - x_n)/r^2.  Beyond the reference (forces)."""
    if xi <= 0 or rc <= 0:
        raise ValueError("xi and rc must be positive")
    plan = _native.plan_for(periodicity.D, system.L, _real_params(xi, rc))
    E = _native.host_out((system.N, 3))
    _native.call("se_realspace_field_host", plan.handle, _native.ptr(system.positions),
                 _native.ptr(system.charges), system.N, _native.ptr(E))
    return E


def self_term(q, xi: float) -> np.ndarray:
    """-2 xi q / sqrt(pi) (realspace.py:183-185)."""
    qa = np.ascontiguousarray(np.asarray(q, dtype=float))
    out = np.empty_like(qa)
    _native.call("se_self_term_host", _native.ptr(qa), qa.size, float(xi), _native.ptr(out))
    return out
