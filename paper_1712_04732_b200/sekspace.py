"""Fourier-space pipeline (mirror of pmewald.sekspace) on the SE B200 library.

Stage calls map onto the C ABI (include/se_b200.h):

    spread                      -> se_spread_host      (tile-binned smem spreading kernel)
    gather                      -> se_gather_host      (tile-staged gather kernel)
    apply_kspace                -> se_kspace_apply_host (cuFFT + fused multiplier)
    se_kspace                   -> se_kspace_potential_host (spread, k-space, gather)
    precompute_truncated_greens -> se_d0_kernel_table_host (device precompute)

Grid geometry and the D=0 kernel geometry come from the library's planning
routines (sekspace.py:53-70, 266-279 of the reference).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _native, aft, windows  # noqa: F401  (aft: reachable as sekspace.aft, as in the reference)
from .core import ParticleSystem, Periodicity, SEParams


@dataclass(frozen=True)
class Grid:
    """Grid geometry (sekspace.py:36-70): M per periodic axis, Mt = M + P per
    free axis, spacing h = L/M, free-axis offsets P h / 2."""

    L: float
    M: int
    P: int
    D: int
    h: float
    Lt: float
    Mt: int
    R: float
    g0: int
    gs: int

    @classmethod
    def build(cls, L: float, params: SEParams, periodicity: Periodicity) -> "Grid":
        g = _native.se_grid_t()
        _native.call("se_grid_build", int(periodicity.D), float(L),
                     _native.params_struct(params), ctypes.byref(g))
        return cls(g.L, g.M, g.P, g.D, g.h, g.Lt, g.Mt, g.R, g.g0, g.gs)

    @property
    def shape(self) -> tuple[int, int, int]:
        return tuple(self.M if a < self.D else self.Mt for a in range(3))

    @property
    def offsets(self) -> np.ndarray:
        return np.array([0.0 if a < self.D else 0.5 * self.P * self.h for a in range(3)])


@dataclass(frozen=True)
class GridField:
    values: np.ndarray
    grid: Grid


@dataclass(frozen=True)
class PrecomputedKernel:
    """Truncated free-space kernel on the convolution grid (sekspace.py:73-94)."""

    Mt: int
    g0: int
    nconv: int
    R: float
    h: float
    ghat: np.ndarray


_KERNEL_CACHE: dict = {}


def mode_values(n: int, h: float) -> np.ndarray:
    """2 pi fftfreq(n, d=h) (sekspace.py:100-102)."""
    return 2.0 * np.pi * np.fft.fftfreq(n, d=h)


def _stage_params(grid: Grid, wspec: windows.WindowSpec) -> SEParams:
    """Parameters that pin a library plan to (grid, window) for the stage calls;
    xi / rc / upsampling do not enter spreading or gathering."""
    s0 = max(1.0, grid.g0 / grid.Mt) if grid.D < 3 else 1.0
    return SEParams(xi=1.0, rc=1.0, M=grid.M, P=grid.P, window=wspec.kind, shape=wspec.shape,
                    s0=s0, s=1.0, nI=0, R=grid.R if grid.R > 0 else 1.0, eps=1e-12)


def _stage_plan(grid: Grid, wspec: windows.WindowSpec):
    if grid.P > grid.M:
        raise ValueError("window support P must not exceed M")
    return _native.plan_for(grid.D, grid.L, _stage_params(grid, wspec))


def _stencil(system: ParticleSystem, wspec: windows.WindowSpec, grid: Grid, sel) -> tuple[list, list]:
    """Per-axis stencil indices (n, P) and window weights of a particle
    selection (sekspace.py:105-121): first = floor(u / h - P / 2) + 1 with
    u = x + the free-axis offset, idx = first + t (mod M on periodic axes),
    weights = window(idx h - u).  The host-side view of what the spreading
    and gathering kernels compute per particle (the reference's tests use it
    for the mass identity); the weights come from the library's window
    evaluation."""
    P, h = grid.P, grid.h
    t = np.arange(P)
    idxs, wts = [], []
    offs = grid.offsets
    for a in range(3):
        u = np.asarray(system.positions[sel, a]) + offs[a]
        first = np.floor(u / h - 0.5 * P).astype(np.int64) + 1
        idx = first[:, None] + t[None, :]
        delta = idx * h - u[:, None]
        if a < grid.D:
            idx = np.mod(idx, grid.M)
        wts.append(windows.evaluate(delta, wspec))
        idxs.append(idx)
    return idxs, wts


def spread(system: ParticleSystem, wspec: windows.WindowSpec, grid: Grid,
           periodicity: Periodicity, threads: int = 1) -> GridField:
    """H = sum_n q_n w (x) w (x) w on the grid (sekspace.py:130-156)."""
    plan = _stage_plan(grid, wspec)
    out = np.empty(grid.shape)
    _native.call("se_spread_host", plan.handle, _native.ptr(system.positions),
                 _native.ptr(system.charges), system.N, _native.ptr(out))
    return GridField(out, grid)


def gather(field: GridField, system: ParticleSystem, wspec: windows.WindowSpec,
           periodicity: Periodicity, threads: int = 1) -> np.ndarray:
    """phi_m = h^3 sum H~ w (x) w (x) w, the adjoint of spread (sekspace.py:159-178)."""
    grid = field.grid
    plan = _stage_plan(grid, wspec)
    H = np.ascontiguousarray(field.values, dtype=np.float64)
    if H.shape != grid.shape:
        raise ValueError("grid values do not match the grid shape")
    phi = _native.host_out(system.N)
    _native.call("se_gather_host", plan.handle, _native.ptr(H), _native.ptr(system.positions),
                 system.N, _native.ptr(phi))
    return phi


def _window_table(wspec: windows.WindowSpec, k) -> np.ndarray:
    """Window transform on a mode set with the underflow guard (sekspace.py:181-185)."""
    vals = np.ascontiguousarray(windows.fourier(k, wspec), dtype=np.float64)
    if vals.size and np.min(np.abs(vals)) < 1e-30:
        raise AssertionError("window transform underflow: P/M misconfigured")
    return vals


def scale(F, xi: float, wspec: windows.WindowSpec, gspec, grid: Grid, periodicity: Periodicity):
    """Multiply every retained mode by 4 pi e^{-k^2/4 xi^2} G_hat / w_hat^2
    (sekspace.py:192-254), on the device (se_scale_blocks_host); returns a
    new SpectralField."""
    from . import aft

    D, h = periodicity.D, grid.h

    def tab(n):
        k = np.ascontiguousarray(mode_values(n, h))
        return k, _window_table(wspec, k)

    def c(a):
        return np.array(a, dtype=np.complex128, order="C", copy=True)

    kp, wp = tab(grid.M)
    R = float(getattr(gspec, "R", 0.0))
    args = dict(full=None, zero=None, Iblk=None, Jblk=None)
    if D == 3:
        cube = c(F.full)
        _native.call("se_scale_blocks_host", 0, 3, grid.M, grid.Mt, F.g0, F.gs, float(xi), R,
                     _native.ptr(kp), _native.ptr(wp), None, None, None, None, None, None,
                     _native.ptr(cube), None, None, 0, None, None, 0)
        args["full"] = cube
        return aft.SpectralField(D, F.M, F.Mt, F.g0, F.gs, **args)
    k0, w0 = tab(F.g0)
    zero = c(F.zero)
    if D == 0:
        _native.call("se_scale_blocks_host", 0, 0, grid.M, grid.Mt, F.g0, F.gs, float(xi), R,
                     _native.ptr(kp), _native.ptr(wp), _native.ptr(k0), _native.ptr(w0), None, None, None, None,
                     _native.ptr(zero), None, None, 0, None, None, 0)
        return aft.SpectralField(D, F.M, F.Mt, F.g0, F.gs, zero=zero)
    ks, ws = tab(F.gs)
    kt, wt = tab(F.Mt)
    Ib, Jb = c(F.Iblk), c(F.Jblk)
    Ii = np.ascontiguousarray(F.I_idx, dtype=np.int32)
    Ji = np.ascontiguousarray(F.J_idx, dtype=np.int32)
    _native.call("se_scale_blocks_host", 0, D, grid.M, F.Mt, F.g0, F.gs, float(xi), R,
                 _native.ptr(kp), _native.ptr(wp), _native.ptr(k0), _native.ptr(w0), _native.ptr(ks),
                 _native.ptr(ws), _native.ptr(kt), _native.ptr(wt), _native.ptr(zero),
                 _native.ptr(Ib) if Ib.size else None, _native.ptr(Ii) if Ii.size else None, len(Ii),
                 _native.ptr(Jb) if Jb.size else None, _native.ptr(Ji) if Ji.size else None, len(Ji))
    return aft.SpectralField(D, F.M, F.Mt, F.g0, F.gs, zero=zero, Iblk=Ib, Jblk=Jb, I_idx=F.I_idx, J_idx=F.J_idx)


def apply_kspace(field: GridField, params: SEParams, periodicity: Periodicity,
                 use_kernel: bool | None = None) -> GridField:
    """H -> H~: aft_forward, scale, aft_inverse, real part (sekspace.py:366-381),
    or the D=0 precomputed-kernel path (sekspace.py:301-337)."""
    plan = _native.plan_for(periodicity.D, field.grid.L, params)
    H = np.array(field.values, dtype=np.float64, order="C", copy=True)
    uk = 1 if (periodicity.D == 0 and (use_kernel or use_kernel is None)) else 0
    _native.call("se_kspace_apply_host", plan.handle, _native.ptr(H), uk)
    return GridField(H, field.grid)


def precompute_truncated_greens(L: float, M: int, P: int, s0: float,
                                rc: float | None = None) -> PrecomputedKernel:
    """Tabulate the truncated free-space kernel on the device (sekspace.py:257-298)."""
    if s0 < 1.0 + math.sqrt(3.0) - 1e-12:
        raise ValueError("free-space precompute requires s0 >= 1 + sqrt(3)")
    rcv = 1e-300 if rc is None else float(rc)  # margin = max(P h, min(rc, L))
    nconv, g0, R = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_double()
    _native.call("se_d0_kernel_geometry", float(L), int(M), int(P), float(s0), rcv,
                 ctypes.byref(nconv), ctypes.byref(g0), ctypes.byref(R))
    h = L / M
    key = (M + P, g0.value, nconv.value, round(R.value, 12), round(h, 12))
    hit = _KERNEL_CACHE.get(key)
    if hit is not None:
        return hit
    prm = SEParams(xi=1.0, rc=rcv, M=M, P=P, window="bm", shape=2.5 * P, s0=s0, R=1.0)
    plan = _native.Plan(0, L, prm)
    n = nconv.value
    tab = np.empty((n, n, n // 2 + 1))
    _native.call("se_d0_kernel_table_host", plan.handle, _native.ptr(tab))
    kern = PrecomputedKernel(M + P, g0.value, n, R.value, h, tab)
    _KERNEL_CACHE[key] = kern
    return kern


def se_kspace(system: ParticleSystem, params: SEParams, periodicity: Periodicity,
              threads: int = 1, timings: dict | None = None,
              use_kernel: bool | None = None) -> np.ndarray:
    """Fourier-space potential at every source (sekspace.py:340-389)."""
    params.validate(system.L, periodicity)
    plan = _native.plan_for(periodicity.D, system.L, params)
    uk = 1 if (periodicity.D == 0 and (use_kernel or use_kernel is None)) else 0
    phi = _native.host_out(system.N)
    tb = _native.timings_buffer() if timings is not None else None
    _native.call("se_kspace_potential_host", plan.handle, _native.ptr(system.positions),
                 _native.ptr(system.charges), system.N, _native.ptr(phi), uk,
                 _native.ptr(tb) if tb is not None else None)
    if timings is not None:
        _native.fill_timings(timings, tb, ("spread", "aft", "scale", "aift", "gather"))
        timings.setdefault("precompute", float(tb[_native.TIMING_KEYS.index("precompute")]))
    return phi


def se_kspace_field(system: ParticleSystem, params: SEParams, periodicity: Periodicity,
                    threads: int = 1) -> np.ndarray:
    """Fourier part of E = -grad phi at every source, (N, 3).  D = 3: the
    scaled spectrum of se_kspace times -i k per axis, three inverse
    transforms and three gathers; D < 3: the filtered grid of se_kspace and
    the gradient of the gather, h^3 sum H w'(delta_a) prod_{b != a} w(delta_b)
    (Gaussian / Kaiser-Bessel windows).  Beyond the reference (forces,
    SURVEY 8f item 4)."""
    if periodicity.D != 3 and params.window == "bm":
        raise ValueError("forces for D < 3 need the Gaussian or Kaiser-Bessel window (the ES window's "
                         "derivative is singular at its support edge)")
    params.validate(system.L, periodicity)
    plan = _native.plan_for(periodicity.D, system.L, params)
    E = _native.host_out((system.N, 3))
    _native.call("se_kspace_field_host", plan.handle, _native.ptr(system.positions),
                 _native.ptr(system.charges), system.N, _native.ptr(E))
    return E


def global_upsampled_kspace(system: ParticleSystem, params: SEParams,
                            periodicity: Periodicity) -> np.ndarray:
    """Validation path with every free axis padded at s0 (sekspace.py:392-435).

    With nI = M/2 and s = s0 the adaptive transform degenerates to exactly this
    single padded transform (the reference's own acceptance criterion,
    test_acceptance.py:134-147); D=0 is the use_kernel=False path.
    """
    D = periodicity.D
    params.validate(system.L, periodicity)
    if D == 3:
        return se_kspace(system, params, periodicity)
    if D == 0:
        return se_kspace(system, params, periodicity, use_kernel=False)
    degenerate = SEParams(**{**params.__dict__, "nI": params.M // 2, "s": params.s0})
    return se_kspace(system, degenerate, periodicity)
