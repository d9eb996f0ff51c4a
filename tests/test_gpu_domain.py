"""Domain decomposition on the B200 (se_realspace_domain_dev and
distributed.total_potential_domain), without a second GPU:

  * virtual ranks: for a world of 2, 4 or 8 ranks, each rank's own + halo
    particle set is formed on the host exactly as the orchestration forms
    it, the CUDA domain kernel runs per rank, and the own potentials plus
    the returned halo sums must reproduce the single-set real-space sum
    (every unordered pair once over all ranks) -- periodic and free x;
  * one rank (no process group): total_potential_domain through the native
    backend (migration / halo / plane exchange degenerate, slab k-space with
    one slab) equals the fused single-GPU total_potential.
"""

import numpy as np
import pytest
import torch

import paper_1712_04732_b200 as se
from paper_1712_04732_b200 import _native
from paper_1712_04732_b200 import device as sedev
from paper_1712_04732_b200.distributed import DomainPartition, NativeBackend, total_potential_domain

pytestmark = pytest.mark.gpu


def _system(D, N=60000, L=4.0, seed=21):
    rng = np.random.default_rng(seed)
    pos = rng.random((N, 3)) * L
    q = rng.uniform(-1, 1, N)
    q -= q.mean()
    return pos, q, L


@pytest.mark.parametrize("D", [3, 2, 1, 0])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_domain_realspace_virtual_ranks(D, world):
    pos, q, L = _system(D)
    xi, rc = 6.0, 0.4
    prm = se.SEParams(xi=xi, rc=rc, M=32, P=8, window="bm", shape=20.0, s0=4.0, s=2.0, nI=4, R=3.0)
    peri = se.Periodicity(D)
    dev = torch.device("cuda", 0)
    part = DomainPartition(L, prm, peri, world, len(q))
    pl = _native.Plan(D, L, prm, 0)
    cols = part.columns(torch.from_numpy(pos[:, 0])).numpy()
    owner = np.asarray(part.owner_of_col)[cols]
    halo_tab = np.asarray(part.halo_to)
    phi = np.zeros(len(q))
    for r in range(world):
        own = np.nonzero(owner == r)[0]
        halo = np.nonzero(halo_tab[cols, r])[0]
        idx = np.concatenate([own, halo])
        lp = torch.from_numpy(np.ascontiguousarray(pos[idx])).to(dev)
        lq = torch.from_numpy(np.ascontiguousarray(q[idx])).to(dev)
        out = torch.empty(len(idx), dtype=torch.float64, device=dev)
        _native.call("se_realspace_domain_dev", pl.handle, _native.ptr(lp), _native.ptr(lq), len(idx), len(own),
                     part.ncols, part.col_lo[r], part.col_hi[r], _native.ptr(out), 1)
        o = out.cpu().numpy()
        np.add.at(phi, idx, o)
    ref = se.real_space_sum(se.ParticleSystem(pos, q, L), xi, rc, peri) + se.self_term(q, xi)
    err = se.relative_rms_error(phi, ref)
    print(f"D={D} world={world} ncols={part.ncols} reach={part.reach}: rel rms {err:.2e}")
    assert err < 1e-13


@pytest.mark.parametrize("D,kspace", [(3, "slab"), (3, "replicated"), (0, "slab"), (0, "replicated")])
def test_domain_pipeline_one_rank_matches_fused(D, kspace):
    pos, q, L = _system(D, N=40000)
    prm = se.SEParams(xi=6.0, rc=0.4, M=32, P=8, window="bm", shape=20.0, s0=4.0, R=3.5)
    peri = se.Periodicity(D)
    dev = torch.device("cuda", 0)
    pd = torch.from_numpy(pos).to(dev)
    qd = torch.from_numpy(q).to(dev)
    be = NativeBackend(L, prm, peri, dev)
    # a permuted input order: potentials come back in the caller's order
    perm = torch.randperm(len(q), generator=torch.Generator().manual_seed(3)).to(dev)
    phi = total_potential_domain(pd[perm].contiguous(), qd[perm].contiguous(), be, kspace=kspace)
    ref = sedev.total_potential(pd, qd, L, prm, peri)[perm]
    err = se.relative_rms_error(phi.cpu().numpy(), ref.cpu().numpy())
    print(f"D={D} {kspace}: one-rank domain pipeline vs fused: {err:.2e}")
    assert err < 1e-13


def test_domain_rejects_minimum_image_geometry():
    pos, q, L = _system(3, N=1000, L=1.0)
    prm = se.SEParams(xi=6.0, rc=0.45, M=16, P=4, window="bm", shape=10.0)
    with pytest.raises(ValueError):
        DomainPartition(L, prm, se.Periodicity(3), 2, len(q))


@pytest.mark.parametrize("D,world", [(2, 2), (2, 4), (1, 2), (1, 3), (1, 4)])
def test_row_distributed_aft_virtual_ranks(D, world):
    """The se_zslab_* stages of `world` virtual ranks in one process (the
    two all-to-alls done by indexing) reproduce the single-GPU AFT stage."""
    pos, q, L = _system(D, N=20000, L=3.0)
    prm = se.SEParams(xi=6.0, rc=0.4, M=24, P=8, window="bm", shape=20.0, s0=3.0, s=2.0, nI=3, R=3.0)
    peri = se.Periodicity(D)
    dev = torch.device("cuda", 0)
    be = NativeBackend(L, prm, peri, dev)
    pd = torch.from_numpy(pos).to(dev)
    qd = torch.from_numpy(q).to(dev)
    H = be.empty_grid()
    be.spread_all(pd, qd, H)
    ref = H.clone()
    be.kspace_apply(ref)
    geo = [be.zslab_geometry(world, r) for r in range(world)]
    X, Y, Zt = H.shape
    specs = []
    for r in range(world):
        z0, nz = geo[r]["nz0"], geo[r]["nz"]
        zs = H[:, :, z0:z0 + nz].contiguous()
        sp = torch.empty(geo[r]["rows_total"] * geo[r]["per_y"] * nz * 2, dtype=torch.float64, device=dev)
        be.zslab_forward(zs, world, r, sp)
        specs.append(sp)

    def chunk(s, r):  # rank r's rows inside rank s's spectrum
        w = geo[s]["per_y"] * geo[s]["nz"] * 2
        return slice(geo[r]["row0"] * w, (geo[r]["row0"] + geo[r]["nrows"]) * w)

    for r in range(world):
        recv = torch.cat([specs[s][chunk(s, r)] for s in range(world)])
        be.zslab_rows(recv, world, r)
        off = 0
        for s in range(world):
            n = chunk(s, r).stop - chunk(s, r).start
            specs[s][chunk(s, r)] = recv[off:off + n]
            off += n
    out = torch.empty_like(H)
    for r in range(world):
        z0, nz = geo[r]["nz0"], geo[r]["nz"]
        zs = torch.empty((X, Y, nz), dtype=torch.float64, device=dev)
        be.zslab_inverse(specs[r], world, r, zs)
        out[:, :, z0:z0 + nz] = zs
    torch.cuda.synchronize()
    err = float((out - ref).norm() / ref.norm())
    print(f"D={D} world={world}: row-distributed AFT vs single-GPU stage {err:.2e}")
    assert err < 1e-13


@pytest.mark.parametrize("D", [2, 1])
def test_domain_pipeline_one_rank_zslab(D):
    pos, q, L = _system(D, N=30000, L=3.0)
    prm = se.SEParams(xi=6.0, rc=0.4, M=24, P=8, window="bm", shape=20.0, s0=3.0, s=2.0, nI=3, R=3.0)
    peri = se.Periodicity(D)
    dev = torch.device("cuda", 0)
    pd = torch.from_numpy(pos).to(dev)
    qd = torch.from_numpy(q).to(dev)
    be = NativeBackend(L, prm, peri, dev)
    phi = total_potential_domain(pd, qd, be, kspace="zslab")
    ref = sedev.total_potential(pd, qd, L, prm, peri)
    err = se.relative_rms_error(phi.cpu().numpy(), ref.cpu().numpy())
    print(f"D={D} zslab: one-rank domain pipeline vs fused: {err:.2e}")
    assert err < 1e-13
