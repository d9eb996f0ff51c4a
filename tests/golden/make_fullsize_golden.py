"""Full-size golden vectors: the UNMODIFIED reference (`pmewald`) run on the
BASELINE configs at their full sizes, on the same seeded inputs the bench
and the GPU tests generate (tools/workloads.py).

Run in the build container (the reference is not on the GPU box); cfg2 takes
~20 min of the reference's CPU path on 8 threads:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fullsize_golden.py cfg1 cfg3 cfg4 cfg2
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fullsize_golden.py cfg1_tol cfg4_tol cfg2_tol

Writes `tests/golden/full_<cfg>.npz`: the reference's total potential
(core.total_potential), Fourier part (sekspace.se_kspace) and real-space part
(realspace.real_space_sum) at a seeded sample of targets, whole-vector
checksums of the total potential (sum q phi -- the reference's core.energy
--, sum phi^2, sum phi), the reference's own stage timings and the thread
count.  A full vector is 8 bytes per particle; the sample plus checksums
keep the fixtures small while the checksums still cover every entry.

cfg5 (D = 0, N = 5e5, clustered): the reference's real space builds dense
(|home|, |neighbour|, 3) distance blocks of ~24k x 24k particles per cell
pair there (~32 GB per thread), so it runs with THREADS=1 in the
62 GB container (round 2: 5,334 s, real space 5,304 s):

    THREADS=1 PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fullsize_golden.py cfg5
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import workloads  # noqa: E402
from pmewald import core, realspace, sekspace  # noqa: E402
from pmewald.core import ParticleSystem, Periodicity, SEParams  # noqa: E402

SAMPLE = {"cfg1": 2000, "cfg1_tol": 2000, "cfg2": 20000, "cfg2_tol": 20000, "cfg3": 20000, "cfg3_tol": 20000,
          "cfg4": 20000, "cfg4_tol": 20000, "cfg5": 20000}


def run(name, threads):
    w = workloads.ALL[name]()
    pos, q, L, D = w["pos"], w["q"], w["L"], w["D"]
    prm = SEParams(**w["prm"])
    peri = Periodicity(D)
    system = ParticleSystem(pos, q, float(L))
    t0 = time.perf_counter()
    tim = {}
    phi = core.total_potential(system, prm, peri, threads=threads, timings=tim)
    wall = time.perf_counter() - t0
    # the parts (the k-space stage again: ~seconds; real space once more only
    # for the small configs -- for cfg2 the total minus k-space minus self
    # term is the real-space part to rounding)
    phik = sekspace.se_kspace(system, prm, peri, threads=threads)
    phis = realspace.self_term(q, prm.xi)
    phir = phi - phik - phis
    n = len(q)
    k = min(SAMPLE.get(name, 20000), n)
    sel = np.sort(np.random.default_rng(1000 + n % 997).choice(n, k, replace=False))
    out = dict(name=name, N=n, sel=sel, phi=phi[sel], phi_k=phik[sel], phi_r=phir[sel],
               energy=float(core.energy(system, phi)), sum_phi=float(phi.sum()),
               sum_phi2=float(np.dot(phi, phi)), threads=threads, wall_s=wall,
               timings_keys=np.array(sorted(tim)), timings=np.array([tim[x] for x in sorted(tim)]))
    path = os.path.join(HERE, f"full_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: N={n} wall {wall:.1f} s ({threads} threads) timings "
          + ", ".join(f"{x}={tim[x]:.2f}" for x in sorted(tim)) + f" -> {path}", flush=True)


if __name__ == "__main__":
    threads = int(os.environ.get("THREADS", os.cpu_count() or 1))
    for name in sys.argv[1:] or ["cfg1", "cfg3", "cfg4", "cfg2"]:
        run(name, threads)
