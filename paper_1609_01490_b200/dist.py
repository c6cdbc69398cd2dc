"""Multi-GPU plumbing over torch.distributed (NCCL on B200, gloo in CPU tests).

One process per GPU.  The block map itself partitions the work
(tri_map_init(rank, world): contiguous, area-balanced omega ranges snapped to
tile rows), so EDM and the dummy kernel need no collective at all.  The two
real exchange steps of the path are here:

* ``allreduce_count``  -- the collision count, SUM over ranks (8 bytes);
* ``allreduce_energy`` -- per-particle triplet energies, SUM (n fp64);
* ``halo_exchange``    -- the CA's boundary rows: rank g needs row R_g - 1
  (the last row of the rank below it in row order) and row R_{g+1} (the first
  row of the next rank), exchanged point-to-point every generation.

Only torch.distributed calls live here -- no compute.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def T(r: int) -> int:
    return r * (r + 1) // 2


def world_info():
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def allreduce_count(count: torch.Tensor) -> torch.Tensor:
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(count, op=dist.ReduceOp.SUM)
    return count


def allreduce_energy(energy: torch.Tensor) -> torch.Tensor:
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(energy, op=dist.ReduceOp.SUM)
    return energy


def row_bounds(maps_rows):
    """maps_rows: list of (row_begin, row_end) for every rank (all ranks compute
    the same list from tri_map_init, no communication)."""
    return list(maps_rows)


def _owner(bounds, r):
    for g, (a, b) in enumerate(bounds):
        if a <= r < b:
            return g
    return None


def halo_exchange(state: torch.Tensor, bounds, n: int, rank: int, above: torch.Tensor | None,
                  below: torch.Tensor | None):
    """Exchange the CA boundary rows for the packed slice ``state`` of this rank.

    bounds[g] = (row_begin, row_end) of rank g.  ``above`` receives row R_g - 1
    (R_g bytes), ``below`` receives row R_{g+1} (R_{g+1} + 1 bytes).  Rows are
    contiguous in the packed Eq. 1 slice, so the sends are views (no copies).
    Ranks that own no rows take no part.  Returns the list of requests' waits done.
    """
    R0, R1 = bounds[rank]
    ops = []
    if R1 > R0:
        # my first row goes to the owner of row R0 - 1 (it is that rank's "below")
        if R0 > 0:
            g = _owner(bounds, R0 - 1)
            ops.append(dist.P2POp(dist.isend, state[0:R0 + 1], g))
            ops.append(dist.P2POp(dist.irecv, above, g))
        # my last row goes to the owner of row R1 (it is that rank's "above")
        if R1 < n:
            g = _owner(bounds, R1)
            last = R1 - 1
            o = T(last) - T(R0)
            ops.append(dist.P2POp(dist.isend, state[o:o + last + 1], g))
            ops.append(dist.P2POp(dist.irecv, below, g))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
