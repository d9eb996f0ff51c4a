"""One process per GPU: the SE pipeline sharded over torch.distributed ranks.

Every rank holds all N particles (inputs are replicated once per call).
Work is split by ownership of contiguous ranges of the particles' sorted
order -- cell order for the real-space sum, tile order for spreading and
gathering -- so each stage's share is spatially compact and no data-path
exchange is needed inside a stage.  The exchange steps are the ones the
method has:

  1. spread_shard on every rank -> partial grids; SUM all-reduce (NCCL over
     NVLink) -> the full grid H on every rank, overlapped with the
     real-space shard (which does not read the grid);
  2. k-space stage on every rank (the 32^3-128^3 FFTs are latency bound;
     replicating them is cheaper than a slab all-to-all at these sizes);
  3. realspace_shard (+ self term) and gather_shard write the owned entries
     of phi (others zero); SUM all-reduce of phi -> the full potential.

The compute backend is injectable so that the orchestration (the part that
owns the collectives) is the same code on B200 ranks (`NativeBackend`, the
sm_100a kernels) and in the CPU gloo tests (a backend built from the oracle).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import _native
from .core import Periodicity, SEParams


class NativeBackend:
    """Shard stages on the SE B200 library (device tensors, current stream)."""

    def __init__(self, L: float, params: SEParams, periodicity: Periodicity, device: torch.device):
        self.L, self.params, self.peri, self.device = L, params, periodicity, device
        self.plan = _native.plan_for(periodicity.D, L, params, device.index or 0)
        self.plan.set_stream(torch.cuda.current_stream(device).cuda_stream)
        g = self.plan.grid()
        self.shape = tuple(g.shape)

    def empty_grid(self):
        return torch.empty(self.shape, dtype=torch.float64, device=self.device)

    def empty_phi(self, N):
        return torch.empty(N, dtype=torch.float64, device=self.device)

    def spread_shard(self, pos, q, rank, world, grid):
        _native.call("se_spread_shard_dev", self.plan.handle, _native.ptr(pos), _native.ptr(q), q.shape[0],
                     rank, world, _native.ptr(grid))

    def kspace_apply(self, grid):
        uk = 1 if self.peri.D == 0 else 0
        _native.call("se_kspace_apply_dev", self.plan.handle, _native.ptr(grid), uk, None)

    def realspace_shard(self, pos, q, rank, world, phi):
        _native.call("se_realspace_shard_dev", self.plan.handle, _native.ptr(pos), _native.ptr(q), q.shape[0],
                     rank, world, _native.ptr(phi), 1)

    def gather_shard(self, grid, pos, rank, world, phi):
        _native.call("se_gather_shard_dev", self.plan.handle, _native.ptr(grid), _native.ptr(pos), pos.shape[0],
                     rank, world, _native.ptr(phi), 1)


def total_potential_sharded(pos, q, backend, group=None):
    """core.total_potential across the ranks of `group`; returns the full phi
    on every rank.  pos (N,3) / q (N,) are this rank's replicated inputs."""
    init = dist.is_initialized()
    rank = dist.get_rank(group) if init else 0
    world = dist.get_world_size(group) if init else 1
    N = q.shape[0]
    grid = backend.empty_grid()
    backend.spread_shard(pos, q, rank, world, grid)
    # the grid all-reduce (NCCL over NVLink) overlaps the real-space shard,
    # which does not read the grid
    work = dist.all_reduce(grid, op=dist.ReduceOp.SUM, group=group, async_op=True) if init else None
    phi = backend.empty_phi(N)
    backend.realspace_shard(pos, q, rank, world, phi)
    if work is not None:
        work.wait()
    backend.kspace_apply(grid)
    backend.gather_shard(grid, pos, rank, world, phi)
    if init:
        dist.all_reduce(phi, op=dist.ReduceOp.SUM, group=group)
    return phi


def shard_bounds(N: int, rank: int, world: int) -> tuple[int, int]:
    """Owned range [lo, hi) of a sorted order (same rule as the C ABI)."""
    return N * rank // world, N * (rank + 1) // world
