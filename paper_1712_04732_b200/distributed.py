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
