"""Randomized campaign for the real-space field: the default path (Newton
half shell with dense batches where the pair polynomial is fitted, the full
shell otherwise) against the deterministic mode's full-shell field and, at
sampled targets, the oracle.   python tools/gpu/field_campaign.py [cases]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import se_oracle as orc  # noqa: E402

import paper_1712_04732_b200 as se  # noqa: E402
from paper_1712_04732_b200.realspace import real_space_field  # noqa: E402


def rel(a, b):
    return float(np.sqrt(np.mean((a - b) ** 2)) / np.sqrt(np.mean(b ** 2)))


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    rng = np.random.default_rng(4242)
    worst_full = worst_orc = worst_mom = 0.0
    for case in range(cases):
        D = int(rng.integers(0, 4))
        N = int(rng.integers(3000, 40000))
        L = float(rng.uniform(0.8, 2.5))
        rc = float(rng.uniform(0.12, 0.35)) * L
        xi = float(rng.uniform(2.2, 5.6)) / rc  # above ~5: no polynomial, the full-shell field
        clustered = case % 4 == 3
        if clustered:
            c = rng.random((8, 3)) * L
            pos = (c[rng.integers(0, 8, N)] + 0.08 * L * rng.standard_normal((N, 3))) % L
        else:
            pos = rng.random((N, 3)) * L
        q = rng.uniform(-1, 1, N)
        q -= q.mean()
        s = se.ParticleSystem(pos, q, L)
        peri = se.Periodicity(D)
        e = real_space_field(s, xi, rc, peri)
        se.set_deterministic(True)
        try:
            ef = real_space_field(s, xi, rc, peri)
        finally:
            se.set_deterministic(False)
        sel = rng.choice(N, 16, replace=False)
        eo = orc.realspace_field(pos, q, L, D, xi, rc, targets=sel)
        F = q[:, None] * e
        r1, r2 = rel(e, ef), rel(e[sel], eo)
        mom = float(np.abs(F.sum(0)).max() / np.abs(F).sum(0).max())
        worst_full, worst_orc, worst_mom = max(worst_full, r1), max(worst_orc, r2), max(worst_mom, mom)
        ok = r1 < 1e-12 and r2 < 1e-11 and mom < 1e-10
        print(f"case {case:3d} D={D} N={N:6d} L={L:.2f} rc={rc:.3f} xi*rc={xi * rc:.2f} "
              f"{'clustered' if clustered else 'uniform  '} vs full shell {r1:.1e} vs oracle {r2:.1e} "
              f"sum F {mom:.1e} {'ok' if ok else 'FAIL'}", flush=True)
        if not ok:
            raise SystemExit(1)
    print(f"{cases} cases, worst vs full shell {worst_full:.2e}, vs oracle {worst_orc:.2e}, sum F {worst_mom:.2e}")


if __name__ == "__main__":
    main()
