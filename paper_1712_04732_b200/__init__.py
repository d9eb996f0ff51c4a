"""B200-native Spectral Ewald summation with 0-3 periodic directions.

Drop-in for the hot path of the reference package `pmewald`
(arXiv 1712.04732): the public names of its `__all__`
(reference __init__.py:20-36), with the same signatures, dataclasses and
exceptions.  All compute runs in the hand-written sm_100a kernels of
`_lib/libse_b200.so` (C ABI: include/se_b200.h); there is no CPU fallback.
Device-resident (torch CUDA tensor) entry points live in `.device`, the
one-process-per-GPU sharded pipeline in `.distributed`.
"""

from . import core, params, realspace, sekspace

_PUBLIC = {
    core: ("ConfigurationError", "ParticleSystem", "Periodicity", "SEParams",
           "SingularConfigurationError", "energy", "generate_random_system", "load_particles",
           "relative_rms_error", "save_particles", "total_potential",
           # beyond the reference: E = -grad phi and F = q E, D = 3
           "total_field", "forces"),
    params: ("auto_params",),
    realspace: ("real_space_sum", "self_term"),
    sekspace: ("se_kspace",),
}
for _mod, _names in _PUBLIC.items():
    for _n in _names:
        globals()[_n] = getattr(_mod, _n)

__all__ = sorted(n for names in _PUBLIC.values() for n in names)

from ._native import set_deterministic  # noqa: E402  (beyond the reference: opt-in bitwise reproducibility)
del _mod, _names, _n
