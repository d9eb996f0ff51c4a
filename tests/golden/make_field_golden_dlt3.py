"""Golden vectors for the electric field (forces) with D = 0, 1, 2 periodic
directions, from the UNMODIFIED reference by central differences of its own
potentials (it stops at potentials): the real-space sum
(realspace.real_space_sum, realspace.py:168-180) and the direct Fourier-space
sums (oracle.kspace_direct_2p / _1p / _0p, oracle.py:134-192).  Moving x_m
changes only the evaluation point of phi_m's terms (the particle's own term
is independent of x_m), so -(phi_m(x + delta) - phi_m(x - delta)) / (2 delta)
is the field at x_m.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_field_golden_dlt3.py

Writes tests/golden/field_dlt3.npz (D<d>_* arrays).
"""

from __future__ import annotations

import os

import numpy as np

from pmewald import oracle, realspace
from pmewald.core import ParticleSystem, Periodicity

HERE = os.path.dirname(os.path.abspath(__file__))


def fd(fun, pos, m, a, delta):
    p1, p2 = pos.copy(), pos.copy()
    p1[m, a] += delta
    p2[m, a] -= delta
    return -(fun(p1)[m] - fun(p2)[m]) / (2 * delta)


def main():
    out = {}
    for D, N in ((2, 24), (1, 12), (0, 24)):
        rng = np.random.default_rng(30 + D)
        L = 1.0
        pos = 0.1 + 0.8 * rng.random((N, 3))
        q = rng.uniform(-1.0, 1.0, N)
        q -= q.mean()
        xi, rc, kmax, delta = 6.0, 0.45, 12, 1e-6
        per = Periodicity(D)
        real = lambda p: realspace.real_space_sum(ParticleSystem(p, q, L), xi, rc, per)  # noqa: E731
        kdir = lambda p: oracle.kspace_direct(ParticleSystem(p, q, L), xi, per, kmax)  # noqa: E731
        Er = np.array([[fd(real, pos, m, a, delta) for a in range(3)] for m in range(N)])
        Ek = np.array([[fd(kdir, pos, m, a, delta) for a in range(3)] for m in range(N)])
        out.update({f"D{D}_pos": pos, f"D{D}_q": q, f"D{D}_prm": np.array([L, xi, rc, kmax, delta]),
                    f"D{D}_E_real_fd": Er, f"D{D}_E_kspace_direct_fd": Ek})
        print(f"D={D}: N {N} |E_R| max {np.abs(Er).max():.3f} |E_k| max {np.abs(Ek).max():.3f}", flush=True)
    np.savez(os.path.join(HERE, "field_dlt3.npz"), **out)


if __name__ == "__main__":
    main()
