"""Golden vectors for the electric field (forces), from the UNMODIFIED
reference by central differences of its own potentials: the reference stops
at potentials, so E = -grad phi is pinned through them.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_field_golden.py

For particle m and axis a, moving x_m by +-delta changes only the evaluation
point of phi_m's pair terms (real_space_sum, realspace.py:168-180) and of
its Fourier sum (oracle.kspace_direct_3p, oracle.py:109-118; the particle's
own term in S(k) contributes q_m independently of x_m), so
-(phi_m(x + delta) - phi_m(x - delta)) / (2 delta) is the field at x_m.
Writes tests/golden/field.npz.
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
    rng = np.random.default_rng(11)
    N, L = 48, 1.0
    pos = rng.random((N, 3)) * L
    q = rng.uniform(-1.0, 1.0, N)
    q -= q.mean()
    xi, rc, kmax, delta = 8.0, 0.45, 10, 1e-6
    per = Periodicity(3)
    real = lambda p: realspace.real_space_sum(ParticleSystem(p, q, L), xi, rc, per)  # noqa: E731
    kdir = lambda p: oracle.kspace_direct_3p(ParticleSystem(p, q, L), xi, kmax)  # noqa: E731
    Er = np.array([[fd(real, pos, m, a, delta) for a in range(3)] for m in range(N)])
    Ek = np.array([[fd(kdir, pos, m, a, delta) for a in range(3)] for m in range(N)])
    np.savez(os.path.join(HERE, "field.npz"), pos=pos, q=q, L=L, xi=xi, rc=rc, kmax=kmax, delta=delta,
             E_real_fd=Er, E_kspace_direct_fd=Ek)
    print("field.npz: N", N, "|E_R| max", np.abs(Er).max(), "|E_k| max", np.abs(Ek).max())


if __name__ == "__main__":
    main()
