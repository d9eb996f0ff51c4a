"""One process per GPU: the SE pipeline sharded over torch.distributed ranks.

Work is split by ownership of contiguous ranges of the particles' sorted
order -- cell order for the real-space sum, tile order for spreading and
gathering -- so each stage's share is spatially compact and no data-path
exchange is needed inside a stage.  The exchange steps are the ones the
method has:

  1. spread_shard on every rank -> partial grids, reduced over the ranks
     (NCCL over NVLink), overlapped with the real-space shard (which does
     not read the grid):
       kspace="replicated": SUM all-reduce -> the full grid on every rank,
         k-space stage on every rank (the 32^3-128^3 FFTs are latency
         bound; at these sizes replicating them is cheaper than slabs);
       kspace="slab" (D = 3): SUM reduce-scatter into x-slabs of M / world
         planes, 2-D FFTs of the slab, all-to-all transpose, x-FFT +
         multiplier + inverse x-FFT on this rank's ky-chunk, all-to-all
         back, inverse 2-D FFTs, all-gather of the filtered slabs;
  2. realspace_shard (+ self term) and gather_shard write the owned entries
     of phi (others zero); SUM all-reduce of phi (or, for partitioned
     inputs, a reduce-scatter back to each rank's own particles).

Inputs are either replicated (every rank passes all N particles:
total_potential_sharded) or partitioned (each rank passes its own
particles: total_potential_partitioned, which all-gathers them first and
returns each rank its own potentials).

The compute backend is injectable so that the orchestration (the part that
owns the collectives) is the same code on B200 ranks (`NativeBackend`, the
sm_100a kernels) and in the CPU gloo tests (a backend built from the oracle).
"""

from __future__ import annotations

import contextlib
import ctypes
import math

import torch
import torch.distributed as dist

from . import _native
from .core import Periodicity, SEParams, SingularConfigurationError


class NativeBackend:
    """Shard stages on the SE B200 library (device tensors).

    Two plans: `plan` runs the real-space shard on the caller's current
    stream, `plan_k` the k-space chain (spread, grid exchange, FFT stage,
    gather) on `kstream`, a higher-priority side stream -- the same overlap
    of the issue-bound real-space kernel with the shared-memory-bound
    k-space kernels as the single-GPU total_potential, with the grid
    collectives issued on the side stream's order."""

    def __init__(self, L: float, params: SEParams, periodicity: Periodicity, device: torch.device):
        self.L, self.params, self.peri, self.device = L, params, periodicity, device
        # dedicated plans (not the process-wide cache): their stream and
        # deferred-check settings are this backend's
        self.plan = _native.Plan(periodicity.D, L, params, device.index or 0)
        self.plan.set_stream(torch.cuda.current_stream(device).cuda_stream)
        self.kstream = torch.cuda.Stream(device=device, priority=-1)
        self.plan_k = _native.Plan(periodicity.D, L, params, device.index or 0)
        self.plan_k.set_stream(self.kstream.cuda_stream)
        self.plans = (self.plan, self.plan_k)
        # the orchestration enqueues both streams' work before any host sync
        # (errors and profiling events are collected by finish())
        for p in self.plans:
            _native.call("se_plan_set_deferred_checks", p.handle, 1)
        g = self.plan.grid()
        self.shape = tuple(g.shape)

    def _k(self, name, *args):
        """A k-space-chain call on plan_k: inside the orchestration the
        current stream is kstream already; a direct caller on another stream
        is fenced on both sides, so the call is ordered like a plain one."""
        cur = torch.cuda.current_stream(self.device)
        if cur == self.kstream:
            _native.call(name, self.plan_k.handle, *args)
            return
        self.kstream.wait_stream(cur)
        _native.call(name, self.plan_k.handle, *args)
        cur.wait_stream(self.kstream)

    def bind_stream(self):
        """Order the real-space plan on the caller's current stream (the
        orchestration's joins are against the stream current at call time)."""
        self.plan.set_stream(torch.cuda.current_stream(self.device).cuda_stream)

    def check_system(self, pos, q, neutrality=True):
        """Box [0, L) and neutrality checks (core.py:65-77, 180-191) on the
        device inputs, once per call (the shard entry points run deferred)."""
        _native.call("se_check_system_dev", self.plan.handle, _native.ptr(pos), _native.ptr(q), q.shape[0],
                     int(bool(neutrality)))

    def finish(self):
        """Synchronise both plans; raise a deferred device error."""
        for p in self.plans:
            _native.call("se_plan_finish", p.handle)

    def empty_grid(self):
        return torch.empty(self.shape, dtype=torch.float64, device=self.device)

    def empty_phi(self, N):
        return torch.empty(N, dtype=torch.float64, device=self.device)

    def spread_shard(self, pos, q, rank, world, grid):
        self._k("se_spread_shard_dev", _native.ptr(pos), _native.ptr(q), q.shape[0],
                     rank, world, _native.ptr(grid))

    def kspace_apply(self, grid):
        uk = 1 if self.peri.D == 0 else 0
        self._k("se_kspace_apply_dev", _native.ptr(grid), uk, None)

    def realspace_shard(self, pos, q, rank, world, phi):
        _native.call("se_realspace_shard_dev", self.plan.handle, _native.ptr(pos), _native.ptr(q), q.shape[0],
                     rank, world, _native.ptr(phi), 1)

    def gather_shard(self, grid, pos, rank, world, phi, accumulate=True):
        self._k("se_gather_shard_dev", _native.ptr(grid), _native.ptr(pos), pos.shape[0],
                     rank, world, _native.ptr(phi), int(bool(accumulate)))

    # domain decomposition (total_potential_domain)
    def domain_partition(self, world, n_total):
        key = (world, n_total)
        cache = self.__dict__.setdefault("_partitions", {})
        if key not in cache:
            cache[key] = DomainPartition(self.L, self.params, self.peri, world, n_total, self.shape)
        return cache[key]

    def slab_kgeo(self):
        """Plane geometry of the slab k-space stage (DomainPartition.touched_pieces)."""
        g = self.plan.grid()
        D = self.peri.D
        if D >= 1:
            n = int(g.M)
        else:
            nconv, g0, R = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_double()
            _native.call("se_plan_d0_geometry", self.plan_k.handle, ctypes.byref(nconv), ctypes.byref(g0),
                         ctypes.byref(R))
            n = int(nconv.value)
        return {"planes": int(g.shape[0]), "n": n, "P": int(g.P), "h": float(g.h),
                "off": 0.0 if D >= 1 else 0.5 * g.P * g.h, "periodic": D >= 1}

    def spread_all(self, pos, q, grid):
        self._k("se_spread_shard_dev", _native.ptr(pos), _native.ptr(q), q.shape[0], 0, 1, _native.ptr(grid))

    def gather_all(self, grid, pos, phi, accumulate=False):
        self._k("se_gather_shard_dev", _native.ptr(grid), _native.ptr(pos), pos.shape[0], 0, 1, _native.ptr(phi),
                int(bool(accumulate)))

    def realspace_domain(self, pos, q, n_own, part, rank, phi):
        _native.call("se_realspace_domain_dev", self.plan.handle, _native.ptr(pos), _native.ptr(q), q.shape[0],
                     int(n_own), part.ncols, part.col_lo[rank], part.col_hi[rank], _native.ptr(phi), 1)

    # row-distributed adaptive FFT (D = 1, 2)
    def zslab_geometry(self, world, rank):
        out = (ctypes.c_int64 * 6)()
        _native.call("se_zslab_geometry", self.plan_k.handle, world, rank, out)
        return dict(zip(("nz0", "nz", "row0", "nrows", "rows_total", "per_y"), (int(v) for v in out)))

    def zslab_forward(self, zslab, world, rank, spec):
        self._k("se_zslab_forward_dev", world, rank, _native.ptr(zslab), _native.ptr(spec))

    def zslab_rows(self, recv, world, rank):
        self._k("se_zslab_rows_dev", world, rank, _native.ptr(recv))

    def zslab_inverse(self, spec, world, rank, zslab):
        self._k("se_zslab_inverse_dev", world, rank, _native.ptr(spec), _native.ptr(zslab))

    # slab-decomposed k-space stage (D = 3)
    def slab_geometry(self, world):
        nx, nky, nkz = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _native.call("se_slab_geometry", self.plan_k.handle, world, ctypes.byref(nx), ctypes.byref(nky),
                     ctypes.byref(nkz))
        return nx.value, nky.value, nkz.value

    def empty_spectrum(self, world):
        nx, nky, nkz = self.slab_geometry(world)
        return torch.empty((world, nx, nky, nkz, 2), dtype=torch.float64, device=self.device)

    def slab_forward(self, slab, world, send):
        self._k("se_slab_forward_dev", world, _native.ptr(slab), _native.ptr(send))

    def slab_xpass(self, recv, rank, world):
        self._k("se_slab_xpass_dev", world, rank, _native.ptr(recv))

    def slab_inverse(self, back, world, slab):
        self._k("se_slab_inverse_dev", world, _native.ptr(back), _native.ptr(slab))


def total_potential_sharded(pos, q, backend, group=None, kspace: str = "replicated", reduce_phi: bool = True):
    """core.total_potential across the ranks of `group`; returns the full phi
    on every rank.  pos (N,3) / q (N,) are this rank's replicated inputs.
    kspace: "replicated" (all-reduce of the grid, k-space on every rank) or
    "slab" (D = 3: reduce-scatter into x-slabs, slab FFT with two all-to-all
    transposes, all-gather).  reduce_phi=False returns this rank's partial
    phi (owned entries only) for the caller to reduce."""
    if kspace not in ("replicated", "slab"):
        raise ValueError(f"kspace must be 'replicated' or 'slab', got {kspace!r}")
    init = dist.is_initialized()
    rank = dist.get_rank(group) if init else 0
    world = dist.get_world_size(group) if init else 1
    N = q.shape[0]
    multi = init and world > 1
    if hasattr(backend, "bind_stream"):
        backend.bind_stream()
    if hasattr(backend, "check_system"):
        _agreed(lambda: backend.check_system(pos, q), q, group, multi)
    # the k-space chain on the backend's side stream (if it has one),
    # concurrent with the real-space shard on the current stream; buffers
    # are allocated here, on the current stream, and the final join orders
    # every later use after the side stream's work
    ks = getattr(backend, "kstream", None)
    cur = torch.cuda.current_stream() if ks is not None else None
    side = torch.cuda.stream(ks) if ks is not None else contextlib.nullcontext()
    grid = backend.empty_grid()
    phi = backend.empty_phi(N)
    phik = backend.empty_phi(N) if ks is not None else None
    if kspace == "slab":
        nx, nky, nkz = backend.slab_geometry(world)
        flat = grid.reshape(-1)
        # one rank: the slab is the grid and the transposes are identities
        slab = flat.new_empty((nx,) + tuple(grid.shape[1:])) if multi else grid
        send = backend.empty_spectrum(world)
        recv = torch.empty_like(send) if multi else send
    if ks is not None:
        ks.wait_stream(cur)
    with side:
        backend.spread_shard(pos, q, rank, world, grid)
        if kspace == "replicated":
            work = dist.all_reduce(grid, op=dist.ReduceOp.SUM, group=group, async_op=True) if init else None
        else:
            work = dist.reduce_scatter_tensor(slab.reshape(-1), flat, op=dist.ReduceOp.SUM, group=group,
                                              async_op=True) if multi else None
    backend.realspace_shard(pos, q, rank, world, phi)
    with side:
        if work is not None:
            work.wait()
        if kspace == "replicated":
            backend.kspace_apply(grid)
        else:
            backend.slab_forward(slab, world, send)
            if multi:
                dist.all_to_all_single(recv.reshape(-1), send.reshape(-1), group=group)
            backend.slab_xpass(recv, rank, world)
            if multi:
                dist.all_to_all_single(send.reshape(-1), recv.reshape(-1), group=group)
            backend.slab_inverse(send, world, slab)
            if multi:
                dist.all_gather_into_tensor(flat, slab.reshape(-1), group=group)
        if ks is None:
            backend.gather_shard(grid, pos, rank, world, phi)
        else:
            # phi_F into its own buffer, concurrent with the real-space
            # shard; one add after the join
            backend.gather_shard(grid, pos, rank, world, phik, accumulate=False)
    if ks is not None:
        cur.wait_stream(ks)
        phi.add_(phik)
    if init and reduce_phi:
        dist.all_reduce(phi, op=dist.ReduceOp.SUM, group=group)
    _finish(backend, phi, group, init and world > 1)
    return phi


def _agreed(fn, like, group, multi):
    """Run fn() on every rank and agree on failure: a rank whose call raised
    re-raises its own exception, every other rank raises the same class
    (so no rank enters the next collective alone).  Any exception counts:
    a deferred CUDA / cuFFT error as much as SingularConfigurationError."""
    err = None
    try:
        fn()
    except Exception as e:  # noqa: BLE001 -- re-raised below on every rank
        err = e
    if multi:
        code = 0.0 if err is None else (2.0 if isinstance(err, SingularConfigurationError) else
                                        3.0 if isinstance(err, ValueError) else 1.0)
        flag = torch.tensor([code], dtype=torch.float64, device=like.device)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
        c = flag.item()
        if err is None and c > 0:
            err = {2.0: SingularConfigurationError("coincident distinct particles (detected on another rank)"),
                   3.0: ValueError("invalid input (detected on another rank)")}.get(
                       c, RuntimeError("device error on another rank"))
    if err is not None:
        raise err


def _finish(backend, like, group, multi):
    """Deferred device checks of this call, agreed over the ranks: a rank
    whose shard found coincident particles (realspace.py:118-122) raises
    SingularConfigurationError, and so does every other rank (instead of
    entering the next collective alone)."""
    _agreed(backend.finish if hasattr(backend, "finish") else (lambda: None), like, group, multi)


def total_potential_partitioned(pos_local, q_local, backend, group=None, kspace: str = "replicated"):
    """core.total_potential for particles partitioned over the ranks: rank r
    passes its own (n_r, 3) positions and (n_r,) charges and receives their
    potentials (n_r,).  The particle sets are all-gathered (32 B per
    particle), the sharded pipeline runs, and the potential sum is
    reduce-scattered back to the owners."""
    init = dist.is_initialized()
    world = dist.get_world_size(group) if init else 1
    rank = dist.get_rank(group) if init else 0
    if not init or world == 1:
        return total_potential_sharded(pos_local, q_local, backend, group, kspace)
    dev = pos_local.device
    n = torch.tensor([q_local.shape[0]], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    nmax = max(counts)
    rec = torch.zeros((nmax, 4), dtype=torch.float64, device=dev)
    rec[:counts[rank], :3] = pos_local
    rec[:counts[rank], 3] = q_local
    allrec = torch.empty((world * nmax, 4), dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(allrec, rec, group=group)
    keep = torch.cat([torch.arange(r * nmax, r * nmax + counts[r], device=dev) for r in range(world)])
    allrec = allrec[keep]
    pos = allrec[:, :3].contiguous()
    q = allrec[:, 3].contiguous()
    partial = total_potential_sharded(pos, q, backend, group, kspace, reduce_phi=False)
    # reduce-scatter of the partial sums back to the owners (blocks padded to nmax)
    pad = torch.zeros(world * nmax, dtype=torch.float64, device=dev)
    pad[keep] = partial
    mine = torch.empty(nmax, dtype=torch.float64, device=dev)
    dist.reduce_scatter_tensor(mine, pad, op=dist.ReduceOp.SUM, group=group)
    return mine[:counts[rank]].clone()


def shard_bounds(N: int, rank: int, world: int) -> tuple[int, int]:
    """Owned range [lo, hi) of a sorted order (same rule as the C ABI)."""
    return N * rank // world, N * (rank + 1) // world


# --------------------------------------------------------------------------
# Domain decomposition: particles partitioned over the ranks
# --------------------------------------------------------------------------

class DomainPartition:
    """x-slabs of whole real-space columns, the same on every rank.

    The real-space column grid is ncols x ncols columns of edge L / ncols >=
    rc / reach in (x, y) (the kernel's rule: reach 3, or 2 when columns would
    hold < 256 particles of the whole system); rank r owns the columns
    cx in [col_lo[r], col_hi[r]) and every particle in them -- for real
    space (targets), spreading and gathering alike.  Its real-space halo is
    the `reach` columns beyond col_hi (+x side, wrapping on a periodic x):
    the half shell of the column kernel points to +x, so each unordered pair
    is evaluated by exactly one rank and the halo particles' Newton partial
    sums travel back to their owners.

    The k-space grid's x-planes are owned in equal slabs of M / world planes
    (D = 3); a rank's particles touch the planes of their stencils, a ring
    interval of x-planes (touched_planes), which is all a rank sends to and
    receives from the slab owners.
    """

    def __init__(self, L, params, periodicity, world, n_total, grid_shape=None):
        L, rc = float(L), float(params.rc)
        D = periodicity.D
        if D >= 1 and rc > L / 2 + 1e-12:
            raise ValueError("domain decomposition covers the cell path (rc <= L/2); use total_potential_sharded")
        reach = 3
        while True:
            n = int(min(1024, max(1, math.floor(reach * L / rc))))
            if reach == 2 or n_total / (n * n) >= 256.0:
                break
            reach -= 1
        # the column kernel's reach for this grid (se_realspace.cu cell_bin)
        reach = max(1, int(math.ceil(rc * n / L - 1e-12)))
        if D >= 1 and n < 2 * reach + 1:
            raise ValueError(f"{n} columns per periodic axis are too few for a domain decomposition "
                             f"(need >= {2 * reach + 1}); use total_potential_sharded")
        if n < world:
            raise ValueError(f"{world} ranks for {n} real-space columns; use total_potential_sharded")
        self.L, self.D, self.rc, self.ncols, self.reach, self.world = L, D, rc, n, reach, world
        self.edge = L / n
        self.periodic_x = D >= 1
        self.col_lo = [n * r // world for r in range(world)]
        self.col_hi = [n * (r + 1) // world for r in range(world)]
        owner = []
        for r in range(world):
            owner += [r] * (self.col_hi[r] - self.col_lo[r])
        self.owner_of_col = owner
        # halo_to[c][d]: column c is in rank d's +x halo
        self.halo_to = [[self._in_halo(c, d) for d in range(world)] for c in range(n)]
        self.grid_shape = tuple(grid_shape) if grid_shape is not None else None
        self.params = params

    def _in_halo(self, c, d):
        if self.owner_of_col[c] == d:
            return False
        off = c - self.col_hi[d]
        if self.periodic_x:
            off %= self.ncols
        return 0 <= off < self.reach

    def device_tables(self, dev):
        """(owner rank per column, halo[column, rank]) on `dev`, built once."""
        tabs = self.__dict__.setdefault("_tables", {})
        if dev not in tabs:
            tabs[dev] = (torch.tensor(self.owner_of_col, dtype=torch.int64, device=dev),
                         torch.tensor(self.halo_to, dtype=torch.bool, device=dev))
        return tabs[dev]

    def columns(self, x):
        """Column index cx of each x (the kernel's floor(x / edge), clamped)."""
        return torch.clamp(torch.floor(x / self.edge), 0, self.ncols - 1).to(torch.int64)

    # k-space plane bookkeeping (slab mode) ---------------------------------
    # kg: {"planes": x-planes of the spread grid (M, or Mt for D = 0),
    #      "n": the slab transform size (M, or nconv), "P", "h",
    #      "off": the x offset of the stencil (0, or P h / 2 on a free x),
    #      "periodic": x periodic}
    def slab(self, r, kg):
        nx = kg["n"] // self.world
        return r * nx, (r + 1) * nx

    def touched_pieces(self, r, kg):
        """x-plane intervals the stencils of rank r's particles can touch:
        first index floor((x + off) / h - P / 2) + 1 over x in
        [col_lo edge, col_hi edge), P planes each, one plane of margin on
        both sides for the rounding of x / h; a ring interval mod M on a
        periodic x, clipped to [0, planes) on a free one."""
        if self.col_hi[r] <= self.col_lo[r]:
            return []
        P, h, planes, off = kg["P"], kg["h"], kg["planes"], kg["off"]
        xa, xb = self.col_lo[r] * self.edge + off, self.col_hi[r] * self.edge + off
        f_lo = math.floor(xa / h - 0.5 * P) + 1 - 1
        f_hi = math.floor(xb / h - 0.5 * P) + 1 + P
        if kg["periodic"]:
            count = min(planes, f_hi - f_lo + 1)
            start = f_lo % planes
            if start + count <= planes:
                return [(start, start + count)]
            return [(start, planes), (0, start + count - planes)]
        lo, hi = max(0, f_lo), min(planes, f_hi + 1)
        return [(lo, hi)] if lo < hi else []

    def exchange_pieces(self, src, dst, kg):
        """Plane intervals of rank src's touched planes inside rank dst's slab."""
        a, b = self.slab(dst, kg)
        out = []
        for lo, hi in self.touched_pieces(src, kg):
            lo2, hi2 = max(lo, a), min(hi, b)
            if lo2 < hi2:
                out.append((lo2, hi2))
        return out


def _all_to_allv(send, send_counts, group, multi, recv_counts=None):
    """all_to_all_single of the rows of `send` (grouped by destination, counts
    per rank); returns (recv, recv_counts).  recv_counts, when the caller
    knows them (the partition fixes every plane exchange; a return path
    mirrors its outbound exchange), skip the count exchange and its host
    synchronisation."""
    if not multi:
        return send, list(send_counts)
    if recv_counts is None:
        dev = send.device
        sc = torch.tensor(send_counts, dtype=torch.int64, device=dev)
        rc = torch.empty_like(sc)
        dist.all_to_all_single(rc, sc, group=group)
        recv_counts = [int(v) for v in rc.tolist()]
    recv = send.new_empty((sum(recv_counts),) + tuple(send.shape[1:]))
    dist.all_to_all_single(recv, send.contiguous(), output_split_sizes=recv_counts, input_split_sizes=list(send_counts),
                           group=group)
    return recv, recv_counts


def total_potential_domain(pos_local, q_local, backend, group=None, kspace: str = "auto"):
    """core.total_potential for particles PARTITIONED over the ranks, by
    domain decomposition: rank r passes its own (n_r, 3) positions and
    (n_r,) charges (any subset of the system) and receives their potentials.

      1. migrate: every particle to the rank owning its x-slab of columns
         (all-to-allv of (x, y, z, q) records);
      2. halo: the particles of the `reach` columns beyond each slab's +x end
         to that slab's rank (all-to-allv);
      3. real space on own + halo particles (se_realspace_domain_dev: targets
         are the own particles, the half shell points to +x) -- concurrently
         with the k-space chain on the backend's side stream;
      4. the halo particles' Newton partial sums back to their owners;
      5. spread of the own particles into a local grid; the touched x-planes
         to the k-space slab owners (all-to-allv, summed there) -- D = 3
         with M divisible by the rank count ("slab"): slab FFT with two
         all-to-all transposes and the filtered planes back to the ranks that
         touch them; otherwise ("replicated") a sum all-reduce of the grid and
         the k-space stage on every rank;
      6. gather of the own particles, phi = phi_R + phi_self + phi_F + halo
         sums, and each potential back to the rank that passed the particle
         (all-to-allv in the order of step 1)."""
    init = dist.is_initialized()
    world = dist.get_world_size(group) if init else 1
    rank = dist.get_rank(group) if init else 0
    multi = init and world > 1
    dev = pos_local.device
    n_in = int(q_local.shape[0])
    if hasattr(backend, "bind_stream"):
        backend.bind_stream()
    if hasattr(backend, "check_system"):
        _agreed(lambda: backend.check_system(pos_local, q_local, neutrality=False), q_local, group, multi)
    # the neutrality check of the whole system (core.py:180-191) on the
    # reduced charge sums, and the total particle count, in one all-reduce
    sums = torch.stack([q_local.sum(), q_local.abs().sum(),
                        torch.tensor(float(n_in), dtype=torch.float64, device=dev)])
    if multi:
        dist.all_reduce(sums, group=group)
    qsum, qabs, n_all = sums.tolist()
    ntot = torch.tensor([int(n_all)])
    if abs(qsum) > 1e-12 * max(qabs, 1.0):
        if backend.peri.D > 0:
            raise ValueError("periodic Ewald summation requires a charge-neutral system")
        import warnings
        warnings.warn("system is not charge neutral; free-space potentials are still defined but the Ewald "
                      "split assumes neutrality", stacklevel=2)
    part = backend.domain_partition(world, int(ntot.item()))
    cols_of, halo_tab = part.device_tables(dev)

    if multi:
        # 1. migrate to the owners
        rec = torch.cat([pos_local, q_local[:, None]], dim=1)
        dest = cols_of[part.columns(pos_local[:, 0])]
        order = torch.argsort(dest, stable=True)
        send_counts = torch.bincount(dest, minlength=world).tolist()
        own, own_counts = _all_to_allv(rec[order], send_counts, group, multi)
        n_own = int(own.shape[0])

        # 2. halo: each own particle to the ranks whose +x halo holds its column
        cx = part.columns(own[:, 0])
        # every (own particle, destination) halo pair, grouped by destination
        # (a stable sort of the row-major nonzero list): one host sync for the
        # pairs and one for the counts, whatever the rank count
        pairs = torch.nonzero(halo_tab[cx], as_tuple=False)  # (k, 2): particle, rank
        if pairs.shape[0]:
            pairs = pairs[torch.argsort(pairs[:, 1], stable=True)]
        hidx = pairs[:, 0]
        hcounts = torch.bincount(pairs[:, 1], minlength=world).tolist() if pairs.shape[0] else [0] * world
        halo, halo_counts = _all_to_allv(own[hidx], hcounts, group, multi)
        local = torch.cat([own, halo], dim=0)
        lpos = local[:, :3].contiguous()
        lq = local[:, 3].contiguous()
        opos = own[:, :3].contiguous()
        oq = own[:, 3].contiguous()
    else:
        # one rank: every particle is its own, no halo, no exchange
        n_own = n_in
        lpos = opos = pos_local.contiguous()
        lq = oq = q_local.contiguous()
        hidx = None

    # 3. + 5. the k-space chain on the side stream, real space on this one
    ks = getattr(backend, "kstream", None)
    cur = torch.cuda.current_stream() if ks is not None else None
    side = torch.cuda.stream(ks) if ks is not None else contextlib.nullcontext()
    phi_local = backend.empty_phi(lpos.shape[0])
    phik = backend.empty_phi(n_own)
    grid = backend.empty_grid()
    D = backend.peri.D
    kg = backend.slab_kgeo()
    slab_ok = D in (0, 3) and kg["n"] % world == 0
    zslab_ok = D in (1, 2) and (D == 1 or kg["planes"] % world == 0) and grid.shape[2] >= world
    if kspace == "auto":
        kspace = "slab" if slab_ok else ("zslab" if zslab_ok and multi else "replicated")
    if kspace not in ("slab", "zslab", "replicated"):
        raise ValueError(f"kspace must be 'auto', 'slab', 'zslab' or 'replicated', got {kspace!r}")
    if kspace == "slab" and not slab_ok:
        raise ValueError("the slab k-space stage needs D = 3 or 0 and its transform size (M, or nconv for D = 0) "
                         "divisible by the rank count")
    if kspace == "zslab" and not zslab_ok:
        raise ValueError("the row-distributed AFT needs D = 1 or 2 (D = 2: M divisible by the rank count) and at "
                         "least one free-axis plane per rank")
    if ks is not None:
        ks.wait_stream(cur)
    with side:
        backend.spread_all(opos, oq, grid)
        if kspace == "replicated":
            work = dist.all_reduce(grid, op=dist.ReduceOp.SUM, group=group, async_op=True) if multi else None
    backend.realspace_domain(lpos, lq, n_own, part, rank, phi_local)
    with side:
        if kspace == "replicated":
            if work is not None:
                work.wait()
            backend.kspace_apply(grid)
        elif kspace == "zslab":
            _zslab_kspace_domain(backend, part, kg, grid, rank, world, group, multi)
        else:
            _slab_kspace_domain(backend, part, kg, grid, rank, world, group, multi)
        backend.gather_all(grid, opos, phik, accumulate=False)
    if ks is not None:
        cur.wait_stream(ks)

    if not multi:
        phi_local += phik
        _finish(backend, phi_local, group, multi)
        return phi_local

    # 4. the halo sums back to the owners (the order of step 2)
    back, _ = _all_to_allv(phi_local[n_own:].contiguous(), halo_counts, group, multi, recv_counts=hcounts)
    phi_own = phi_local[:n_own] + phik
    if back.numel():
        phi_own.index_add_(0, hidx, back)
    _finish(backend, phi_own, group, multi)

    # 6. potentials back to the ranks that passed the particles
    ret, _ = _all_to_allv(phi_own, own_counts, group, multi, recv_counts=send_counts)
    out = torch.empty(n_in, dtype=torch.float64, device=dev)
    out[order] = ret
    return out


def _slab_kspace_domain(backend, part, kg, grid, rank, world, group, multi):
    """k-space stage over x-slabs (D = 3, or the D = 0 kernel path on its
    zero-padded nconv^3 grid) with a halo-restricted grid exchange: each
    rank's touched x-planes go to the slab owners and are summed there
    (instead of a reduce-scatter of the whole grid), the slab FFT runs with
    its two all-to-all transposes, and each rank receives back the filtered
    planes it touches (instead of an all-gather of the whole grid)."""
    planes = kg["planes"]
    plane = grid.shape[1] * grid.shape[2]
    flat = grid.reshape(planes, plane)
    a, b = part.slab(rank, kg)
    # forward: my touched planes, grouped by the slab owner
    send_parts, send_counts = [], []
    for d in range(world):
        pieces = part.exchange_pieces(rank, d, kg)
        send_parts += [flat[lo:hi] for lo, hi in pieces]
        send_counts.append(sum(hi - lo for lo, hi in pieces))
    send = torch.cat(send_parts) if send_parts else flat.new_zeros((0, plane))
    rcounts = [sum(hi - lo for lo, hi in part.exchange_pieces(s, rank, kg)) for s in range(world)]
    recv, _ = _all_to_allv(send, send_counts, group, multi, recv_counts=rcounts)
    slab = flat.new_zeros((b - a, plane))
    row = 0
    for s in range(world):
        for lo, hi in part.exchange_pieces(s, rank, kg):
            slab[lo - a:hi - a] += recv[row:row + hi - lo]
            row += hi - lo
    slab = slab.reshape((b - a,) + tuple(grid.shape[1:]))
    send_s = backend.empty_spectrum(world)
    recv_s = torch.empty_like(send_s) if multi else send_s
    backend.slab_forward(slab, world, send_s)
    if multi:
        dist.all_to_all_single(recv_s.reshape(-1), send_s.reshape(-1), group=group)
    backend.slab_xpass(recv_s, rank, world)
    if multi:
        dist.all_to_all_single(send_s.reshape(-1), recv_s.reshape(-1), group=group)
    backend.slab_inverse(send_s, world, slab)
    sflat = slab.reshape(b - a, plane)
    # backward: the filtered planes each rank touches, from my slab
    parts2, counts2 = [], []
    for d in range(world):
        pieces = part.exchange_pieces(d, rank, kg)
        parts2 += [sflat[lo - a:hi - a] for lo, hi in pieces]
        counts2.append(sum(hi - lo for lo, hi in pieces))
    send2 = torch.cat(parts2) if parts2 else flat.new_zeros((0, plane))
    rcounts2 = [sum(hi - lo for lo, hi in part.exchange_pieces(rank, s, kg)) for s in range(world)]
    recv2, _ = _all_to_allv(send2, counts2, group, multi, recv_counts=rcounts2)
    row = 0
    for s in range(world):
        for lo, hi in part.exchange_pieces(rank, s, kg):
            flat[lo:hi] = recv2[row:row + hi - lo]
            row += hi - lo


def _zslab_kspace_domain(backend, part, kg, grid, rank, world, group, multi):
    """D = 1, 2: the adaptive FFT distributed over rows of periodic modes
    ("all-to-all to (kx, ky)-row ownership ... kx-plane
    ownership").  Each rank's touched x-planes go, cut into z-chunks, to the
    chunk owners (summed there); each rank transforms its z-chunk over the
    periodic axes, an all-to-all gives every rank all z of its row chunk, the
    zero / I / J free-axis blocks run there, and the reverse all-to-all, the
    inverse periodic transform and the return of the touched planes (every z)
    give each rank the filtered grid it gathers from."""
    X, Y, Zt = grid.shape
    geo = [backend.zslab_geometry(world, r) for r in range(world)]
    me = geo[rank]
    mine = part.touched_pieces(rank, kg)
    parts, counts = [], []
    for d in range(world):
        z0, z1 = geo[d]["nz0"], geo[d]["nz0"] + geo[d]["nz"]
        blocks = [grid[lo:hi, :, z0:z1].reshape(-1) for lo, hi in mine]
        parts += blocks
        counts.append(sum(int(b.numel()) for b in blocks))
    send = torch.cat(parts) if parts else grid.new_zeros(0)
    nz = me["nz"]
    rcounts = [sum((hi - lo) * Y * nz for lo, hi in part.touched_pieces(s, kg)) for s in range(world)]
    recv, _ = _all_to_allv(send, counts, group, multi, recv_counts=rcounts)
    zslab = grid.new_zeros((X, Y, nz))
    off = 0
    for s in range(world):
        for lo, hi in part.touched_pieces(s, kg):
            n = (hi - lo) * Y * nz
            zslab[lo:hi] += recv[off:off + n].view(hi - lo, Y, nz)
            off += n
    per_y = me["per_y"]
    spec = grid.new_empty(me["rows_total"] * per_y * nz * 2)
    backend.zslab_forward(zslab, world, rank, spec)
    send_c = [geo[d]["nrows"] * per_y * nz * 2 for d in range(world)]
    recv_c = [me["nrows"] * per_y * geo[s]["nz"] * 2 for s in range(world)]
    if multi:
        rows = grid.new_empty(sum(recv_c))
        dist.all_to_all_single(rows, spec, output_split_sizes=recv_c, input_split_sizes=send_c, group=group)
    else:
        rows = spec
    backend.zslab_rows(rows, world, rank)
    if multi:
        dist.all_to_all_single(spec, rows, output_split_sizes=send_c, input_split_sizes=recv_c, group=group)
    backend.zslab_inverse(spec, world, rank, zslab)
    parts2, counts2 = [], []
    for s in range(world):
        blocks = [zslab[lo:hi].reshape(-1) for lo, hi in part.touched_pieces(s, kg)]
        parts2 += blocks
        counts2.append(sum(int(b.numel()) for b in blocks))
    send2 = torch.cat(parts2) if parts2 else grid.new_zeros(0)
    rcounts2 = [sum((hi - lo) * Y * geo[d]["nz"] for lo, hi in mine) for d in range(world)]
    recv2, _ = _all_to_allv(send2, counts2, group, multi, recv_counts=rcounts2)
    off = 0
    for d in range(world):
        z0, nzd = geo[d]["nz0"], geo[d]["nz"]
        for lo, hi in mine:
            n = (hi - lo) * Y * nzd
            grid[lo:hi, :, z0:z0 + nzd] = recv2[off:off + n].view(hi - lo, Y, nzd)
            off += n
