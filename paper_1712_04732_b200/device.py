"""Device-resident entry points: the same pipeline as core.total_potential /
sekspace.se_kspace / realspace.real_space_sum, on CUDA torch tensors that
already live in HBM (zero copy through the C ABI's _dev functions, ordered
on torch's current stream).  torch provides device memory and streams only.
"""

from __future__ import annotations

import torch

from . import _native
from .core import Periodicity, SEParams


def _check(t: torch.Tensor, shape, name):
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous float64 CUDA tensor")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}")


def plan(L: float, params: SEParams, periodicity: Periodicity, device: torch.device):
    pl = _native.plan_for(periodicity.D, L, params, device.index or 0)
    pl.set_stream(torch.cuda.current_stream(device).cuda_stream)
    return pl


def total_potential(positions: torch.Tensor, charges: torch.Tensor, L: float, params: SEParams,
                    periodicity: Periodicity, out: torch.Tensor | None = None,
                    timings: dict | None = None) -> torch.Tensor:
    """core.total_potential on device tensors: positions (N,3), charges (N,)."""
    N = charges.shape[0]
    _check(positions, (N, 3), "positions")
    _check(charges, (N,), "charges")
    params.validate(L, periodicity)
    pl = plan(L, params, periodicity, positions.device)
    if out is None:
        out = torch.empty(N, dtype=torch.float64, device=positions.device)
    tb = _native.timings_buffer() if timings is not None else None
    _native.call("se_total_potential_dev", pl.handle, _native.ptr(positions), _native.ptr(charges), N,
                 _native.ptr(out), _native.ptr(tb) if tb is not None else None)
    _native.fill_timings(timings, tb)
    if pl.warnings() & 1:
        import warnings
        warnings.warn("system is not charge neutral; free-space potentials are still "
                      "defined but the Ewald split assumes neutrality", stacklevel=2)
    return out


def total_field(positions: torch.Tensor, charges: torch.Tensor, L: float, params: SEParams,
                periodicity: Periodicity, out: torch.Tensor | None = None) -> torch.Tensor:
    """core.total_field on device tensors: E (N, 3)."""
    N = charges.shape[0]
    _check(positions, (N, 3), "positions")
    _check(charges, (N,), "charges")
    if periodicity.D != 3 and params.window == "bm":
        raise ValueError("forces for D < 3 need the Gaussian or Kaiser-Bessel window (the ES window's "
                         "derivative is singular at its support edge)")
    params.validate(L, periodicity)
    pl = plan(L, params, periodicity, positions.device)
    if out is None:
        out = torch.empty((N, 3), dtype=torch.float64, device=positions.device)
    _native.call("se_total_field_dev", pl.handle, _native.ptr(positions), _native.ptr(charges), N,
                 _native.ptr(out))
    return out


def kspace_potential(positions, charges, L, params, periodicity, use_kernel=None, out=None, timings=None):
    """sekspace.se_kspace on device tensors."""
    N = charges.shape[0]
    _check(positions, (N, 3), "positions")
    _check(charges, (N,), "charges")
    pl = plan(L, params, periodicity, positions.device)
    if out is None:
        out = torch.empty(N, dtype=torch.float64, device=positions.device)
    uk = 1 if (periodicity.D == 0 and (use_kernel or use_kernel is None)) else 0
    tb = _native.timings_buffer() if timings is not None else None
    _native.call("se_kspace_potential_dev", pl.handle, _native.ptr(positions), _native.ptr(charges), N,
                 _native.ptr(out), uk, _native.ptr(tb) if tb is not None else None)
    _native.fill_timings(timings, tb, ("spread", "aft", "scale", "aift", "gather", "precompute"))
    return out


def real_space_sum(positions, charges, L, xi, rc, periodicity, add_self=False, out=None):
    """realspace.real_space_sum (+ self_term) on device tensors."""
    from .realspace import _real_params

    N = charges.shape[0]
    _check(positions, (N, 3), "positions")
    _check(charges, (N,), "charges")
    pl = plan(L, _real_params(xi, rc), periodicity, positions.device)
    if out is None:
        out = torch.empty(N, dtype=torch.float64, device=positions.device)
    _native.call("se_realspace_dev", pl.handle, _native.ptr(positions), _native.ptr(charges), N,
                 _native.ptr(out), int(bool(add_self)))
    return out


def spread(positions, charges, L, params, periodicity, out=None):
    """sekspace.spread on device tensors (grid in the reference's layout)."""
    N = charges.shape[0]
    pl = plan(L, params, periodicity, positions.device)
    g = pl.grid()
    if out is None:
        out = torch.empty(tuple(g.shape), dtype=torch.float64, device=positions.device)
    _native.call("se_spread_dev", pl.handle, _native.ptr(positions), _native.ptr(charges), N, _native.ptr(out))
    return out


def apply_kspace(grid, L, params, periodicity, use_kernel=None):
    """In-place k-space stage on a device grid."""
    pl = plan(L, params, periodicity, grid.device)
    uk = 1 if (periodicity.D == 0 and (use_kernel or use_kernel is None)) else 0
    _native.call("se_kspace_apply_dev", pl.handle, _native.ptr(grid), uk, None)
    return grid


def gather(grid, positions, L, params, periodicity, out=None, accumulate=False):
    """sekspace.gather on device tensors."""
    N = positions.shape[0]
    pl = plan(L, params, periodicity, positions.device)
    if out is None:
        out = torch.empty(N, dtype=torch.float64, device=positions.device)
    _native.call("se_gather_dev", pl.handle, _native.ptr(grid), _native.ptr(positions), N, _native.ptr(out),
                 int(bool(accumulate)))
    return out


def launch_count(L, params, periodicity, device) -> int:
    return _native.plan_for(periodicity.D, L, params, device.index or 0).launches()
