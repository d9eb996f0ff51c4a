"""ctypes binding of the C ABI in include/se_b200.h (libse_b200.so).

The library is built in-tree (`paper_1712_04732_b200/_lib/libse_b200.so`,
see csrc/Makefile).  There is no Python or CPU fallback for any compute
entry point: if the library is missing, every call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SE_B200_LIB: an alternative build of the same library (A/B measurements)
LIB_PATH = os.environ.get("SE_B200_LIB") or os.path.join(_HERE, "_lib", "libse_b200.so")

SE_OK, SE_EINVAL, SE_ECONFIG, SE_ESINGULAR, SE_ENUMERIC, SE_EDEVICE = range(6)
WINDOWS = {"gaussian": 0, "kb": 1, "bm": 2}
TIMING_KEYS = ("realspace", "spread", "aft", "scale", "aift", "gather", "precompute")
KERNEL_SLOTS = ("realspace", "spread", "gather", "kspace", "sort")

c_double_p = ctypes.POINTER(ctypes.c_double)
c_int32_p = ctypes.POINTER(ctypes.c_int32)
c_int64_p = ctypes.POINTER(ctypes.c_int64)


class se_params_t(ctypes.Structure):
    _fields_ = [("xi", ctypes.c_double), ("rc", ctypes.c_double), ("M", ctypes.c_int32),
                ("P", ctypes.c_int32), ("window", ctypes.c_int32), ("nI", ctypes.c_int32),
                ("shape", ctypes.c_double), ("s0", ctypes.c_double), ("s", ctypes.c_double),
                ("R", ctypes.c_double), ("eps", ctypes.c_double)]


class se_grid_t(ctypes.Structure):
    _fields_ = [("D", ctypes.c_int32), ("M", ctypes.c_int32), ("P", ctypes.c_int32),
                ("Mt", ctypes.c_int32), ("g0", ctypes.c_int32), ("gs", ctypes.c_int32),
                ("shape", ctypes.c_int32 * 3), ("L", ctypes.c_double), ("h", ctypes.c_double),
                ("Lt", ctypes.c_double), ("R", ctypes.c_double), ("offsets", ctypes.c_double * 3)]


_P = ctypes.c_void_p
# name -> argtypes (restype is always c_int unless listed in _RESTYPES)
SIGNATURES = {
    "se_params_validate": [ctypes.POINTER(se_params_t), ctypes.c_double, ctypes.c_int],
    "se_grid_build": [ctypes.c_int, ctypes.c_double, ctypes.POINTER(se_params_t), ctypes.POINTER(se_grid_t)],
    "se_padded_size": [ctypes.c_double, ctypes.c_int32, c_int32_p],
    "se_next_even_smooth": [ctypes.c_int32, c_int32_p],
    "se_pair_poly_coefficients": [ctypes.c_double, ctypes.c_double, ctypes.c_int, _P, c_int32_p],
    "se_d0_kernel_geometry": [ctypes.c_double, ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                              ctypes.c_double, c_int32_p, c_int32_p, c_double_p],
    "se_mode_partition_counts": [ctypes.c_int32, ctypes.c_int, ctypes.c_int32, c_int64_p, c_int64_p],
    "se_window_eval": [ctypes.c_int, ctypes.c_int32, ctypes.c_double, ctypes.c_double, _P,
                       ctypes.c_int64, _P],
    "se_window_fourier": [ctypes.c_int, ctypes.c_int32, ctypes.c_double, ctypes.c_double, _P,
                          ctypes.c_int64, _P],
    "se_bm_quadrature": [ctypes.c_double, ctypes.c_double, _P, ctypes.c_int64, ctypes.c_int32, _P],
    "se_kb_sinhc": [_P, ctypes.c_int64, _P],
    "se_cell_list_host": [_P, ctypes.c_int64, ctypes.c_double, ctypes.c_int32, _P, _P],
    "se_greens_zero_mode": [ctypes.c_int, ctypes.c_double, _P, ctypes.c_int64, _P],
    "se_plan_create": [ctypes.POINTER(_P), ctypes.c_int, ctypes.c_double, ctypes.POINTER(se_params_t),
                       ctypes.c_int],
    "se_plan_destroy": [_P],
    "se_plan_set_stream": [_P, _P],
    "se_plan_grid": [_P, ctypes.POINTER(se_grid_t)],
    "se_plan_launch_count": [_P, c_int64_p],
    "se_plan_warnings": [_P, ctypes.POINTER(ctypes.c_int)],
    "se_plan_d0_geometry": [_P, c_int32_p, c_int32_p, c_double_p],
    "se_plan_set_profiling": [_P, ctypes.c_int],
    "se_plan_set_graphs": [_P, ctypes.c_int],
    "se_plan_set_deferred_checks": [_P, ctypes.c_int],
    "se_plan_set_deterministic": [_P, ctypes.c_int],
    "se_plan_finish": [_P],
    "se_plan_kernel_times": [_P, c_double_p, c_int64_p],
    "se_realspace_pair_count_dev": [_P, _P, _P, ctypes.c_int64, c_int64_p],
    "se_check_system_dev": [_P, _P, _P, ctypes.c_int64, ctypes.c_int],
    "se_spread_dev": [_P, _P, _P, ctypes.c_int64, _P],
    "se_kspace_apply_dev": [_P, _P, ctypes.c_int, _P],
    "se_gather_dev": [_P, _P, _P, ctypes.c_int64, _P, ctypes.c_int],
    "se_kspace_potential_dev": [_P, _P, _P, ctypes.c_int64, _P, ctypes.c_int, _P],
    "se_realspace_dev": [_P, _P, _P, ctypes.c_int64, _P, ctypes.c_int],
    "se_total_potential_dev": [_P, _P, _P, ctypes.c_int64, _P, _P],
    "se_realspace_domain_dev": [_P, _P, _P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                _P, ctypes.c_int],
    "se_spread_shard_dev": [_P, _P, _P, ctypes.c_int64, ctypes.c_int, ctypes.c_int, _P],
    "se_total_field_dev": [_P, _P, _P, ctypes.c_int64, _P],
    "se_total_field_host": [_P, _P, _P, ctypes.c_int64, _P],
    "se_realspace_field_host": [_P, _P, _P, ctypes.c_int64, _P],
    "se_kspace_field_host": [_P, _P, _P, ctypes.c_int64, _P],
    "se_slab_geometry": [_P, ctypes.c_int, c_int64_p, c_int64_p, c_int64_p],
    "se_zslab_geometry": [_P, ctypes.c_int, ctypes.c_int, c_int64_p],
    "se_zslab_forward_dev": [_P, ctypes.c_int, ctypes.c_int, _P, _P],
    "se_zslab_rows_dev": [_P, ctypes.c_int, ctypes.c_int, _P],
    "se_zslab_inverse_dev": [_P, ctypes.c_int, ctypes.c_int, _P, _P],
    "se_slab_forward_dev": [_P, ctypes.c_int, _P, _P],
    "se_slab_xpass_dev": [_P, ctypes.c_int, ctypes.c_int, _P],
    "se_slab_inverse_dev": [_P, ctypes.c_int, _P, _P],
    "se_gather_shard_dev": [_P, _P, _P, ctypes.c_int64, ctypes.c_int, ctypes.c_int, _P, ctypes.c_int],
    "se_realspace_shard_dev": [_P, _P, _P, ctypes.c_int64, ctypes.c_int, ctypes.c_int, _P, ctypes.c_int],
    "se_total_potential_host": [_P, _P, _P, ctypes.c_int64, _P, _P],
    "se_kspace_potential_host": [_P, _P, _P, ctypes.c_int64, _P, ctypes.c_int, _P],
    "se_spread_host": [_P, _P, _P, ctypes.c_int64, _P],
    "se_gather_host": [_P, _P, _P, ctypes.c_int64, _P],
    "se_kspace_apply_host": [_P, _P, ctypes.c_int],
    "se_realspace_host": [_P, _P, _P, ctypes.c_int64, _P, ctypes.c_int],
    "se_direct_kspace_3p_dev": [_P, _P, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_int32, _P,
                                ctypes.c_int64, _P, _P],
    "se_direct_kspace_3p_host": [_P, _P, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_int32, _P,
                                 ctypes.c_int64, _P],
    "se_direct_kspace_2p_dev": [_P, _P, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_int32, _P,
                                ctypes.c_int64, _P, _P],
    "se_direct_kspace_2p_host": [_P, _P, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_int32, _P,
                                 ctypes.c_int64, _P],
    "se_direct_kspace_1p_dev": [_P, _P, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_int32, _P,
                                ctypes.c_int64, _P, _P],
    "se_direct_kspace_1p_host": [_P, _P, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_int32, _P,
                                 ctypes.c_int64, _P],
    "se_direct_kspace_0p_dev": [_P, _P, ctypes.c_int64, ctypes.c_double, _P, ctypes.c_int64, _P, _P],
    "se_direct_kspace_0p_host": [_P, _P, ctypes.c_int64, ctypes.c_double, _P, ctypes.c_int64, _P],
    "se_self_term_host": [_P, ctypes.c_int64, ctypes.c_double, _P],
    "se_self_term_dev": [_P, ctypes.c_int64, ctypes.c_double, _P, _P],
    "se_d0_kernel_table_host": [_P, _P],
    "se_fft_c2c_host": [ctypes.c_int, ctypes.c_int, c_int64_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _P],
    "se_fft_r2c_host": [ctypes.c_int, ctypes.c_int, c_int64_p, ctypes.c_int, ctypes.c_int, _P, _P],
    "se_fft_c2r_host": [ctypes.c_int, ctypes.c_int, c_int64_p, ctypes.c_int, ctypes.c_int, _P, _P],
    "se_scale_blocks_host": [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                             ctypes.c_double, ctypes.c_double] + [_P] * 8 + [_P, _P, _P, ctypes.c_int64, _P, _P,
                                                                              ctypes.c_int64],
    "se_last_error": [],
    "se_version": [],
}
_RESTYPES = {"se_last_error": ctypes.c_char_p, "se_version": ctypes.c_char_p}

_lib = None
_lock = threading.Lock()


def load():
    """Load libse_b200.so (raises OSError if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise OSError(f"SE B200 library not built: {LIB_PATH} (run __graft_entry__.build())")
            lib = ctypes.CDLL(LIB_PATH)
            for name, args in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = _RESTYPES.get(name, ctypes.c_int)
            _lib = lib
    return _lib


def _errors():
    from . import core
    return {SE_EINVAL: ValueError, SE_ECONFIG: core.ConfigurationError,
            SE_ESINGULAR: core.SingularConfigurationError, SE_ENUMERIC: AssertionError,
            SE_EDEVICE: RuntimeError}


def call(name, *args):
    """Call a C-ABI function and map a non-zero status to the reference's exception."""
    lib = load()
    st = getattr(lib, name)(*args)
    if st != SE_OK:
        msg = lib.se_last_error().decode(errors="replace")
        raise _errors().get(st, RuntimeError)(msg)
    return st


def params_struct(p) -> se_params_t:
    """SEParams -> se_params_t (window kinds as in windows.py:24-27)."""
    if p.window not in WINDOWS:
        raise ValueError(f"unknown window {p.window!r}")
    return se_params_t(float(p.xi), float(p.rc), int(p.M), int(p.P), WINDOWS[p.window],
                       int(p.nI), float(p.shape), float(p.s0), float(p.s), float(p.R), float(p.eps))


def ptr(a) -> ctypes.c_void_p:
    """Data pointer of a C-contiguous numpy array or a CUDA torch tensor."""
    if isinstance(a, np.ndarray):
        return ctypes.c_void_p(a.ctypes.data)
    return ctypes.c_void_p(a.data_ptr())


# ----------------------------------------------------------------- plan cache
class Plan:
    """Owns one se_plan_t (device tables, cuFFT plans, buffers) for a
    (D, L, SEParams, device) key -- the analogue of the reference's
    module-level caches (sekspace.py:97, windows.py:169-172)."""

    def __init__(self, D: int, L: float, params, device: int = 0):
        self.D, self.L, self.device = int(D), float(L), int(device)
        self._p = params_struct(params)
        h = ctypes.c_void_p()
        call("se_plan_create", ctypes.byref(h), self.D, self.L, ctypes.byref(self._p), self.device)
        self.handle = h

    def grid(self) -> se_grid_t:
        g = se_grid_t()
        call("se_plan_grid", self.handle, ctypes.byref(g))
        return g

    def set_stream(self, stream_ptr: int):
        """Order subsequent calls on this cudaStream_t (0 = legacy default stream)."""
        call("se_plan_set_stream", self.handle, ctypes.c_void_p(int(stream_ptr)))

    def set_graphs(self, on: bool):
        """Replay repeated total-potential calls from a CUDA graph (default on)."""
        call("se_plan_set_graphs", self.handle, int(bool(on)))

    def set_profiling(self, on: bool):
        call("se_plan_set_profiling", self.handle, int(bool(on)))

    def kernel_times(self):
        """Accumulated (ms, launches) per SE_K_* slot since profiling was enabled."""
        ms = (ctypes.c_double * 5)()
        n = (ctypes.c_int64 * 5)()
        call("se_plan_kernel_times", self.handle, ms, n)
        return {k: (ms[i], n[i]) for i, k in enumerate(KERNEL_SLOTS)}

    def launches(self) -> int:
        n = ctypes.c_int64()
        call("se_plan_launch_count", self.handle, ctypes.byref(n))
        return int(n.value)

    def warnings(self) -> int:
        f = ctypes.c_int()
        call("se_plan_warnings", self.handle, ctypes.byref(f))
        return int(f.value)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and _lib is not None:
            try:
                _lib.se_plan_destroy(h)
            except Exception:
                pass
            self.handle = None


# A plan owns mutable device buffers and a stream binding, so it is not
# shared between host threads (one plan per host thread):
# the cache is per thread, and bounded -- a sweep over L / xi / rc / M
# evicts the least recently used plans (their device buffers and cuFFT
# plans are released when the Plan object is collected).
PLAN_CACHE_LIMIT = int(os.environ.get("SE_B200_PLAN_CACHE", "8"))
_tls = threading.local()


def _plan_cache():
    c = getattr(_tls, "plans", None)
    if c is None:
        from collections import OrderedDict
        c = _tls.plans = OrderedDict()
    return c


def plan_for(D, L, params, device: int = 0) -> Plan:
    key = (int(D), float(L), params_key(params), int(device))
    cache = _plan_cache()
    pl = cache.get(key)
    if pl is None:
        pl = Plan(D, L, params, device)
        cache[key] = pl
        while len(cache) > max(1, PLAN_CACHE_LIMIT):
            cache.popitem(last=False)
    else:
        cache.move_to_end(key)
    return pl


def params_key(p):
    return (float(p.xi), float(p.rc), int(p.M), int(p.P), p.window, float(p.shape), float(p.s0),
            float(p.s), int(p.nI), float(p.R), float(p.eps))


def clear_plans():
    """Drop this thread's cached plans (device memory is freed with them)."""
    _plan_cache().clear()


def set_deterministic(on: bool = True):
    """Bitwise reproducible results for the plans created from now on
    (se_plan_set_deterministic: real space without Newton's third law,
    spreading by per-unit tiles reduced in a fixed order).  The reference
    promises thread-count independent, bit-identical potentials
    (test_core.py:139-145); the default mode agrees with this one to
    rounding.  Drops this thread's cached plans."""
    os.environ["SE_B200_DETERMINISTIC"] = "1" if on else "0"
    clear_plans()


def host_out(shape):
    """A fresh float64 output array for a _host entry point, in page-locked
    memory when CUDA is up: the device-to-host copy then runs at full link
    speed without the driver's pageable staging and without first-touch page
    faults on a new array (~0.5 ms for 8 MB).  The array owns its memory
    like any numpy array (torch's caching host allocator takes the block back
    when it is collected)."""
    try:
        import torch
        if torch.cuda.is_available():
            return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()
    except Exception:  # noqa: BLE001 -- fall back to pageable memory
        pass
    return np.empty(shape)


def timings_buffer():
    return np.zeros(len(TIMING_KEYS))


def fill_timings(timings: dict | None, buf, keys=TIMING_KEYS):
    if timings is None:
        return
    for k in keys:
        timings[k] = float(buf[TIMING_KEYS.index(k)])
