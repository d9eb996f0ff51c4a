"""World-size-2 gloo test of the sharded pipeline's orchestration
(paper_1712_04732_b200.distributed.total_potential_sharded) on CPU.

The collectives (sum-all-reduce of the partial grids and of phi) and the
ownership rule (contiguous ranges of a sorted order, shard_bounds) are the
product code; the per-shard compute is supplied by a backend built from the
CPU oracle, since the sm_100a kernels need a GPU.  The result must equal the
single-process oracle total potential.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleBackend:
    """Shard stages on the CPU oracle with the library's ownership rule:
    each rank owns a contiguous range of a spatially sorted order."""

    def __init__(self, orc, pos, q, L, D, prm):
        self.orc, self.L, self.D, self.prm = orc, L, D, prm
        self.g = orc.geometry(L, D, prm["M"], prm["P"], prm.get("s0", 1.0), prm.get("s", 1.0), prm.get("R", 0.0))
        # tile order for spreading / gathering, cell order for real space
        T = 8
        first = np.floor((pos + self.g["offsets"]) / self.g["h"] - 0.5 * prm["P"]).astype(int) + 1
        tiles = np.mod(first, prm["M"]) // T
        nt = prm["M"] // T + 1
        self.tile_order = np.argsort((tiles[:, 0] * nt + tiles[:, 1]) * nt + tiles[:, 2], kind="stable")
        n = max(1, int(2 * L // prm["rc"]))
        c = np.minimum((pos / (L / n)).astype(int), n - 1)
        self.cell_order = np.argsort((c[:, 0] * n + c[:, 1]) * n + c[:, 2], kind="stable")

    def _owned(self, order, rank, world):
        from paper_1712_04732_b200.distributed import shard_bounds
        lo, hi = shard_bounds(len(order), rank, world)
        return order[lo:hi]

    def empty_grid(self):
        return torch.empty(self.g["shape"], dtype=torch.float64)

    def empty_phi(self, N):
        return torch.empty(N, dtype=torch.float64)

    def spread_shard(self, pos, q, rank, world, grid):
        own = self._owned(self.tile_order, rank, world)
        H = self.orc.spread(pos.numpy()[own], q.numpy()[own], self.g, self.prm["window"], self.prm["shape"])
        grid.copy_(torch.from_numpy(H))

    def kspace_apply(self, grid):
        H = self.orc.kspace_d3(grid.numpy(), self.g, self.prm["xi"], self.prm["window"], self.prm["shape"])
        grid.copy_(torch.from_numpy(np.ascontiguousarray(H)))

    def realspace_shard(self, pos, q, rank, world, phi):
        own = self._owned(self.cell_order, rank, world)
        out = np.zeros(len(q))
        p, qq = pos.numpy(), q.numpy()
        out[own] = self.orc.realspace(p, qq, self.L, self.D, self.prm["xi"], self.prm["rc"], targets=own) \
            + self.orc.self_term(qq[own], self.prm["xi"])
        phi.copy_(torch.from_numpy(out))

    def gather_shard(self, grid, pos, rank, world, phi):
        own = self._owned(self.tile_order, rank, world)
        v = self.orc.gather(grid.numpy(), pos.numpy()[own], self.g, self.prm["window"], self.prm["shape"])
        phi[torch.from_numpy(own)] += torch.from_numpy(v)

    # slab-decomposed k-space stage (D = 3), numpy transforms with the
    # library's buffer layouts: send / recv (world, nx, nky, nkz, re|im)
    def slab_geometry(self, world):
        M = self.prm["M"]
        return M // world, M // world, M // 2 + 1

    def empty_spectrum(self, world):
        nx, nky, nkz = self.slab_geometry(world)
        return torch.empty((world, nx, nky, nkz, 2), dtype=torch.float64)

    @staticmethod
    def _put(t, c):
        t.copy_(torch.from_numpy(np.ascontiguousarray(np.stack([c.real, c.imag], -1))))

    @staticmethod
    def _get(t):
        a = t.numpy()
        return a[..., 0] + 1j * a[..., 1]

    def slab_forward(self, slab, world, send):
        nx, nky, nkz = self.slab_geometry(world)
        A = np.fft.rfft2(slab.numpy(), axes=(1, 2))  # (nx, M, nkz)
        self._put(send, A.reshape(nx, world, nky, nkz).transpose(1, 0, 2, 3))

    def slab_xpass(self, recv, rank, world):
        nx, nky, nkz = self.slab_geometry(world)
        M = self.prm["M"]
        g, xi = self.g, self.prm["xi"]
        k = self.orc.wavenumbers(M, g["h"])
        wh = self.orc.window_fourier_checked(self.prm["window"], self.prm["shape"], 0.5 * g["P"] * g["h"], k)
        ky, kz = slice(rank * nky, (rank + 1) * nky), slice(0, nkz)
        k2 = k[:, None, None] ** 2 + k[None, ky, None] ** 2 + k[None, None, kz] ** 2
        inv = np.where(k2 > 0, 1.0 / np.where(k2 > 0, k2, 1.0), 0.0)
        W = wh[:, None, None] * wh[None, ky, None] * wh[None, None, kz]
        mult = self.orc.FOUR_PI * self.orc._mollify(k2, xi) * inv / W ** 2
        C = self._get(recv).reshape(M, nky, nkz)
        G = np.fft.ifft(np.fft.fft(C, axis=0) * mult, axis=0)
        self._put(recv, G.reshape(world, nx, nky, nkz))

    def slab_inverse(self, back, world, slab):
        nx, nky, nkz = self.slab_geometry(world)
        M = self.prm["M"]
        B = self._get(back).transpose(1, 0, 2, 3).reshape(nx, M, nkz)
        slab.copy_(torch.from_numpy(np.fft.irfft2(B, s=(M, M), axes=(1, 2))))


def _inputs():
    rng = np.random.default_rng(5)
    N, L = 400, 1.0
    pos = rng.random((N, 3)) * L
    q = rng.uniform(-1, 1, N)
    q -= q.mean()
    prm = dict(xi=8.0, rc=0.4, M=24, P=8, window="bm", shape=20.0)
    return pos, q, L, prm


# uneven particle partition for the partitioned-input API
_SPLIT = 150


def _worker(rank, world, port, out_path, mode):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "oracle")]
    import se_oracle as orc
    from paper_1712_04732_b200.distributed import total_potential_partitioned, total_potential_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pos, q, L, prm = _inputs()
    be = OracleBackend(orc, pos, q, L, 3, prm)
    if mode == "partitioned":
        lo, hi = (0, _SPLIT) if rank == 0 else (_SPLIT, len(q))
        phi = total_potential_partitioned(torch.from_numpy(pos[lo:hi].copy()), torch.from_numpy(q[lo:hi].copy()),
                                          be, kspace="slab")
    else:
        phi = total_potential_sharded(torch.from_numpy(pos), torch.from_numpy(q), be, kspace=mode)
    np.save(f"{out_path}.{rank}.npy", phi.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["replicated", "slab", "partitioned"])
def test_sharded_orchestration_world2_gloo(tmp_path, mode):
    """replicated: grid all-reduce; slab: reduce-scatter into x-slabs, two
    all-to-all transposes, all-gather; partitioned: each rank passes its own
    (uneven) particle subset and gets its own potentials back."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "oracle"))
    import se_oracle as orc

    world = 2
    out = str(tmp_path / "phi")
    mp.spawn(_worker, args=(world, _free_port(), out, mode), nprocs=world, join=True)
    pos, q, L, prm = _inputs()
    ref = orc.total_potential(pos, q, L, 3, prm)
    for r in range(world):
        phi = np.load(f"{out}.{r}.npy")
        want = ref if mode != "partitioned" else (ref[:_SPLIT] if r == 0 else ref[_SPLIT:])
        assert orc.relative_rms(phi, want) < 1e-13


def test_slab_single_process_matches_replicated():
    """world = 1 (no process group): the slab path aliases its buffers."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "oracle")]
    import se_oracle as orc
    from paper_1712_04732_b200.distributed import total_potential_sharded

    pos, q, L, prm = _inputs()
    be = OracleBackend(orc, pos, q, L, 3, prm)
    a = total_potential_sharded(torch.from_numpy(pos), torch.from_numpy(q), be, kspace="slab")
    ref = orc.total_potential(pos, q, L, 3, prm)
    assert orc.relative_rms(a.numpy(), ref) < 1e-13
    with pytest.raises(ValueError):
        total_potential_sharded(torch.from_numpy(pos), torch.from_numpy(q), be, kspace="pencil")


def test_shard_bounds_cover_exactly():
    from paper_1712_04732_b200.distributed import shard_bounds
    for N in (0, 1, 7, 1000, 1_000_003):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(N, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == N
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def _worker_error(rank, world, port, out_path):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "oracle")]
    import se_oracle as orc
    from paper_1712_04732_b200.core import SingularConfigurationError
    from paper_1712_04732_b200.distributed import total_potential_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pos, q, L, prm = _inputs()

    class Failing(OracleBackend):
        # a deferred device error found by rank 0's shard only
        def finish(self):
            if rank == 0:
                raise SingularConfigurationError("coincident distinct particles")

    try:
        total_potential_sharded(torch.from_numpy(pos), torch.from_numpy(q), Failing(orc, pos, q, L, 3, prm))
        outcome = "returned"
    except SingularConfigurationError:
        outcome = "raised"
    # the ranks are still in step: one more collective completes
    t = torch.ones(1)
    dist.all_reduce(t)
    open(f"{out_path}.{rank}", "w").write(f"{outcome} {int(t.item())}")
    dist.destroy_process_group()


def test_deferred_error_raised_on_every_rank(tmp_path):
    world = 2
    out = str(tmp_path / "err")
    mp.spawn(_worker_error, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        assert open(f"{out}.{r}").read() == "raised 2"
