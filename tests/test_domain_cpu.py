"""Domain decomposition (paper_1712_04732_b200.distributed.total_potential_domain)
on CPU with the gloo backend, world sizes 1, 2 and 3, D = 3 (slab k-space
with the halo-restricted plane exchange, and replicated k-space) and D = 0.

The collectives -- particle migration to the x-slab owners, the +x halo,
the return of the halo particles' Newton sums, the touched-plane exchange
with the k-space slab owners and the return of every potential to the rank
that passed the particle -- are the product code.  The per-rank compute is
an oracle backend with the semantics of the C ABI's domain entry point: the
own particles' pair sums over own + halo sources (+ self term) and the halo
particles' partial sums over the own sources.  The result must equal the
single-process oracle total potential for every particle, whatever subset
each rank passes in.
"""

import os
import socket
import sys
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class DomainOracleBackend:
    """CPU stand-in for distributed.NativeBackend's domain methods."""

    def __init__(self, orc, L, D, prm):
        from paper_1712_04732_b200.core import Periodicity
        self.orc, self.L, self.D, self.prm = orc, L, D, prm
        self.g = orc.geometry(L, D, prm["M"], prm["P"], prm.get("s0", 1.0), prm.get("s", 1.0), prm.get("R", 0.0))
        self.peri = Periodicity(D)
        self.params = SimpleNamespace(**prm)
        if D == 0:
            self.table, kg = orc.d0_kernel_table(L, prm["M"], prm["P"], prm["s0"], prm["rc"])
            self.nconv = kg["nconv"]

    def domain_partition(self, world, n_total):
        from paper_1712_04732_b200.distributed import DomainPartition
        return DomainPartition(self.L, self.params, self.peri, world, n_total, self.g["shape"])

    def slab_kgeo(self):
        n = self.prm["M"] if self.D >= 1 else self.nconv
        return {"planes": self.g["shape"][0], "n": n, "P": self.prm["P"], "h": self.g["h"],
                "off": 0.0 if self.D >= 1 else 0.5 * self.prm["P"] * self.g["h"], "periodic": self.D >= 1}

    def empty_grid(self):
        return torch.empty(tuple(self.g["shape"]), dtype=torch.float64)

    def empty_phi(self, n):
        return torch.empty(n, dtype=torch.float64)

    def spread_all(self, pos, q, grid):
        if q.shape[0] == 0:
            grid.zero_()
            return
        grid.copy_(torch.from_numpy(self.orc.spread(pos.numpy(), q.numpy(), self.g, self.prm["window"],
                                                    self.prm["shape"])))

    def kspace_apply(self, grid):
        H = grid.numpy()
        if self.D == 3:
            Ht = self.orc.kspace_d3(H, self.g, self.prm["xi"], self.prm["window"], self.prm["shape"])
        elif self.D == 0:
            Ht = self.orc.kspace_d0_kernel(H, self.g, self.prm["xi"], self.prm["window"], self.prm["shape"],
                                           self.table, self.nconv)
        else:
            Ht = self.orc.kspace_mixed(H, self.g, self.prm["xi"], self.prm["window"], self.prm["shape"],
                                       self.prm["nI"])
        grid.copy_(torch.from_numpy(np.ascontiguousarray(Ht)))

    def gather_all(self, grid, pos, phi, accumulate=False):
        if pos.shape[0] == 0:
            return
        v = torch.from_numpy(self.orc.gather(grid.numpy(), pos.numpy(), self.g, self.prm["window"],
                                             self.prm["shape"]))
        if accumulate:
            phi += v
        else:
            phi.copy_(v)

    def realspace_domain(self, pos, q, n_own, part, rank, phi):
        """Pair-by-pair restatement of se_realspace_domain_dev: own-own pairs
        all, own-halo pairs only where the halo column lies 1..reach columns
        in +x of the target's column (the column kernel's half shell)."""
        from scipy.special import erfc

        p, qq = pos.numpy(), q.numpy()
        n = len(qq)
        xi, rc, L = self.prm["xi"], self.prm["rc"], self.L
        d = p[:, None, :] - p[None, :, :]
        for a in range(self.D):
            d[..., a] -= L * np.rint(d[..., a] / L)
        r = np.sqrt(np.sum(d * d, axis=2))
        np.fill_diagonal(r, np.inf)
        f = np.where(r < rc, erfc(xi * np.where(r < rc, r, 1.0)) / np.where(r < rc, r, 1.0), 0.0)
        col = part.columns(torch.from_numpy(p[:, 0])).numpy()
        ahead = col[None, :] - col[:, None]  # column of j minus column of i
        if part.periodic_x:
            ahead %= part.ncols
        own = np.arange(n) < n_own
        oo = own[:, None] & own[None, :]
        oh = own[:, None] & ~own[None, :] & (ahead >= 1) & (ahead <= part.reach)
        out = np.zeros(n)
        out[:n_own] = (np.where(oo | oh, f, 0.0) @ qq)[:n_own] + self.orc.self_term(qq[:n_own], xi)
        out[n_own:] = (np.where(oh, f, 0.0).T @ qq)[n_own:]
        phi.copy_(torch.from_numpy(out))

    # slab k-space stage (D = 3, and D = 0 on its zero-padded nconv^3 grid),
    # numpy transforms in the library's layouts
    def _n(self):
        return self.prm["M"] if self.D == 3 else self.nconv

    def slab_geometry(self, world):
        n = self._n()
        return n // world, n // world, n // 2 + 1

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
        n = self._n()
        A = np.fft.rfft2(slab.numpy(), s=(n, n), axes=(1, 2))  # zero-padded for D = 0
        self._put(send, A.reshape(nx, world, nky, nkz).transpose(1, 0, 2, 3))

    def slab_xpass(self, recv, rank, world):
        nx, nky, nkz = self.slab_geometry(world)
        n = self._n()
        g, xi = self.g, self.prm["xi"]
        orc = self.orc
        w = 0.5 * g["P"] * g["h"]
        ky = slice(rank * nky, (rank + 1) * nky)
        if self.D == 3:
            k = orc.wavenumbers(n, g["h"])
            wh = orc.window_fourier_checked(self.prm["window"], self.prm["shape"], w, k)
            k2 = k[:, None, None] ** 2 + k[None, ky, None] ** 2 + k[None, None, :nkz] ** 2
            inv = np.where(k2 > 0, 1.0 / np.where(k2 > 0, k2, 1.0), 0.0)
            W = wh[:, None, None] * wh[None, ky, None] * wh[None, None, :nkz]
            mult = orc.FOUR_PI * orc._mollify(k2, xi) * inv / W ** 2
        else:
            kf = orc.wavenumbers(n, g["h"])
            kh = 2.0 * np.pi * np.fft.rfftfreq(n, d=g["h"])
            af = orc._mollify(kf ** 2, xi) / orc.window_fourier_checked(self.prm["window"], self.prm["shape"], w,
                                                                         kf) ** 2
            ah = orc._mollify(kh ** 2, xi) / orc.window_fourier_checked(self.prm["window"], self.prm["shape"], w,
                                                                         kh) ** 2
            mult = (self.table[:, ky, :] * orc.FOUR_PI * af[:, None, None] * af[None, ky, None]
                    * ah[None, None, :])
        C = self._get(recv).reshape(n, nky, nkz)
        self._put(recv, np.fft.ifft(np.fft.fft(C, axis=0) * mult, axis=0).reshape(world, nx, nky, nkz))

    def slab_inverse(self, back, world, slab):
        nx, nky, nkz = self.slab_geometry(world)
        n = self._n()
        B = self._get(back).transpose(1, 0, 2, 3).reshape(nx, n, nkz)
        out = np.fft.irfft2(B, s=(n, n), axes=(1, 2))
        slab.copy_(torch.from_numpy(np.ascontiguousarray(out[:, :slab.shape[1], :slab.shape[2]])))


    # row-distributed adaptive FFT (D = 1, 2): numpy restatement of the
    # se_zslab_* stages in the library's layouts
    def zslab_geometry(self, world, rank):
        M, Mt = self.prm["M"], self.g["Mt"]
        half = M // 2 + 1
        nz0 = Mt * rank // world
        nz = Mt * (rank + 1) // world - nz0
        if self.D == 2:
            nrows = (M // world) * half
            return dict(nz0=nz0, nz=nz, row0=rank * nrows, nrows=nrows, rows_total=M * half, per_y=1)
        c = -(-half // world)
        row0 = min(rank * c, half)
        return dict(nz0=nz0, nz=nz, row0=row0, nrows=min(half, row0 + c) - row0, rows_total=half, per_y=Mt)

    def zslab_forward(self, zslab, world, rank, spec):
        z = zslab.numpy()
        A = np.fft.rfftn(z, axes=(0, 1)) if self.D == 2 else np.fft.rfft(z, axis=0)
        self._put(spec.view(-1, 2), A.reshape(-1))

    def zslab_inverse(self, spec, world, rank, zslab):
        M = self.prm["M"]
        me = self.zslab_geometry(world, rank)
        A = self._get(spec.view(-1, 2))
        if self.D == 2:
            out = np.fft.irfftn(A.reshape(M, M // 2 + 1, me["nz"]), s=(M, M), axes=(0, 1))
        else:
            out = np.fft.irfft(A.reshape(M // 2 + 1, self.g["Mt"], me["nz"]), n=M, axis=0)
        zslab.copy_(torch.from_numpy(np.ascontiguousarray(out)))

    def zslab_rows(self, recv, world, rank):
        orc, g, D = self.orc, self.g, self.D
        M, Mt, h = self.prm["M"], g["Mt"], g["h"]
        half = M // 2 + 1
        me = self.zslab_geometry(world, rank)
        geo = [self.zslab_geometry(world, s) for s in range(world)]
        nr, py = me["nrows"], me["per_y"]
        flat = self._get(recv.view(-1, 2))
        blocks, off = [], 0
        for s in range(world):
            n = nr * py * geo[s]["nz"]
            blocks.append(flat[off:off + n].reshape(nr, py, geo[s]["nz"]))
            off += n
        Hk = np.concatenate(blocks, axis=2)  # (rows, per_y, Mt)
        kind, shape, xi = self.prm["window"], self.prm["shape"], self.prm["xi"]
        w = 0.5 * g["P"] * h
        kp = orc.wavenumbers(M, h)
        wp = orc.window_fourier_checked(kind, shape, w, kp)
        m = np.where(np.arange(M) < M // 2, np.arange(M), np.arange(M) - M)
        nfree = 3 - D
        faxes = tuple(range(1, 1 + nfree))
        for i in range(nr):
            row = me["row0"] + i
            if D == 2:
                ix, iy = divmod(row, half)
                mu = max(abs(m[ix]), abs(m[iy]))
                kr2, wr = kp[ix] ** 2 + kp[iy] ** 2, wp[ix] * wp[iy]
            else:
                ix = row
                mu = abs(m[ix])
                kr2, wr = kp[ix] ** 2, wp[ix]
            data = Hk[i].reshape(Mt) if D == 2 else Hk[i]
            glen = g["g0"] if mu == 0 else (g["gs"] if mu <= self.prm["nI"] else Mt)
            B = orc._zero_pad_axes(data[None], glen, faxes)[0]
            B = np.fft.fftn(B)
            kf = orc.wavenumbers(glen, h)
            wf = orc.window_fourier_checked(kind, shape, w, kf)
            if nfree == 1:
                kap2, wfree = kf ** 2, wf
            else:
                kap2 = kf[:, None] ** 2 + kf[None, :] ** 2
                wfree = wf[:, None] * wf[None, :]
            if mu == 0:
                B *= (orc.FOUR_PI * orc._mollify(kap2, xi) * orc.greens_zero_block(D, g["R"], np.sqrt(kap2))
                      / ((wp[0] ** D) * wfree) ** 2)
            else:
                k2 = kr2 + kap2
                B *= orc.FOUR_PI * orc._mollify(k2, xi) / (k2 * (wr * wfree) ** 2)
            out = np.fft.ifftn(B)[(slice(0, Mt),) * nfree]
            Hk[i] = out.reshape(Hk[i].shape)
        off = 0
        res = np.empty_like(flat)
        for s in range(world):
            z0, nzs = geo[s]["nz0"], geo[s]["nz"]
            n = nr * py * nzs
            res[off:off + n] = Hk[:, :, z0:z0 + nzs].reshape(-1)
            off += n
        self._put(recv.view(-1, 2), res)


def _case(D):
    rng = np.random.default_rng(11 + D)
    N, L = 500, 1.0
    pos = rng.random((N, 3)) * L
    q = rng.uniform(-1, 1, N)
    q -= q.mean()
    prm = dict(xi=9.0, rc=0.3, M=24, P=8, window="bm", shape=20.0)
    if D == 0:
        prm.update(s0=4.0, R=1.2)
    if D in (1, 2):
        prm.update(s0=3.0, s=2.0, nI=3, R=2.0)
    return pos, q, L, prm


def _subset(rank, world, N, seed=3, empty_rank=None):
    """An arbitrary (unsorted, uneven) subset of the particles per rank
    (empty_rank: that rank passes no particle at all)."""
    owner = np.random.default_rng(seed).integers(0, world, N)
    owner[:world] = np.arange(world)
    if empty_rank is not None:
        owner[owner == empty_rank] = (empty_rank + 1) % world
    return np.nonzero(owner == rank)[0]


def _worker(rank, world, port, out_path, D, kspace, empty_rank=None):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    import se_oracle as orc
    from paper_1712_04732_b200.distributed import total_potential_domain

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pos, q, L, prm = _case(D)
    mine = _subset(rank, world, len(q), empty_rank=empty_rank)
    be = DomainOracleBackend(orc, L, D, prm)
    phi = total_potential_domain(torch.from_numpy(pos[mine].copy()), torch.from_numpy(q[mine].copy()), be,
                                 kspace=kspace)
    np.save(f"{out_path}.{rank}.npy", phi.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,D,kspace", [(2, 3, "slab"), (3, 3, "slab"), (2, 3, "replicated"),
                                            (2, 0, "replicated"), (2, 0, "slab"), (4, 0, "slab"),
                                            (2, 2, "zslab"), (3, 2, "zslab"), (2, 1, "zslab"), (3, 1, "zslab"),
                                            (2, 2, "replicated")])
def test_domain_decomposition_gloo(tmp_path, world, D, kspace):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import se_oracle as orc

    out = str(tmp_path / "phi")
    mp.spawn(_worker, args=(world, _free_port(), out, D, kspace), nprocs=world, join=True)
    pos, q, L, prm = _case(D)
    ref = orc.total_potential(pos, q, L, D, prm)
    for r in range(world):
        mine = _subset(r, world, len(q))
        phi = np.load(f"{out}.{r}.npy")
        assert phi.shape == (len(mine),)
        assert orc.relative_rms(phi, ref[mine]) < 1e-13, (r, orc.relative_rms(phi, ref[mine]))


def test_domain_rank_with_no_particles(tmp_path):
    """A rank that passes an empty set still owns a slab: it receives its
    particles by migration and returns nothing."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import se_oracle as orc

    out = str(tmp_path / "phi")
    mp.spawn(_worker, args=(3, _free_port(), out, 3, "slab", 1), nprocs=3, join=True)
    pos, q, L, prm = _case(3)
    ref = orc.total_potential(pos, q, L, 3, prm)
    for r in range(3):
        mine = _subset(r, 3, len(q), empty_rank=1)
        phi = np.load(f"{out}.{r}.npy")
        assert phi.shape == (len(mine),)
        if len(mine):
            assert orc.relative_rms(phi, ref[mine]) < 1e-13


def test_domain_single_process():
    """No process group: own = every particle, no halo, the slab stage with
    one slab."""
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    import se_oracle as orc
    from paper_1712_04732_b200.distributed import total_potential_domain

    pos, q, L, prm = _case(3)
    be = DomainOracleBackend(orc, L, 3, prm)
    phi = total_potential_domain(torch.from_numpy(pos), torch.from_numpy(q), be)
    assert orc.relative_rms(phi.numpy(), orc.total_potential(pos, q, L, 3, prm)) < 1e-13


def test_partition_geometry():
    """Every column has one owner; the halo of rank d is exactly the `reach`
    columns after its slab (wrapping for a periodic x, cut for a free x);
    the plane exchange pieces tile each rank's touched planes."""
    from paper_1712_04732_b200.core import Periodicity
    from paper_1712_04732_b200.distributed import DomainPartition

    prm = SimpleNamespace(rc=1.0, M=128, P=8)
    for D in (3, 0):
        for world in (1, 2, 3, 4, 8):
            part = DomainPartition(10.0, prm, Periodicity(D), world, 1_000_000)
            assert part.ncols == 30 and part.reach == 3
            assert sorted(set(part.owner_of_col)) == list(range(world))
            for d in range(world):
                halo = [c for c in range(part.ncols) if part.halo_to[c][d]]
                want = [(part.col_hi[d] + k) for k in range(part.reach)]
                want = [c % part.ncols for c in want] if D >= 1 else [c for c in want if c < part.ncols]
                want = [c for c in want if part.owner_of_col[c] != d]
                assert halo == sorted(want)
            M, P, h = 128, 8, 10.0 / 128
            kg = {"planes": M if D == 3 else M + P, "n": M if D == 3 else 240, "P": P, "h": h,
                  "off": 0.0 if D == 3 else 0.5 * P * h, "periodic": D == 3}
            if kg["n"] % world:
                continue  # the slab exchange needs the transform size divisible by the ranks
            for r in range(world):
                touched = sorted(p for lo, hi in part.touched_pieces(r, kg) for p in range(lo, hi))
                assert len(touched) == len(set(touched))
                got = sorted(p for d in range(world) for lo, hi in part.exchange_pieces(r, d, kg)
                             for p in range(lo, hi))
                assert got == touched
                # the planes every particle of the slab touches are inside
                x = np.linspace(part.col_lo[r] * part.edge, part.col_hi[r] * part.edge, 2001)[:-1]
                f = np.floor((x + kg["off"]) / h - 0.5 * P).astype(int) + 1
                need = {int(v) % M if D == 3 else int(v) for v in (f[:, None] + np.arange(P)).ravel()}
                assert need <= set(touched)
    with pytest.raises(ValueError):
        DomainPartition(1.0, SimpleNamespace(rc=0.6, M=16, P=4), Periodicity(3), 2, 100)
