"""Multi-GPU plumbing over torch.distributed (NCCL on B200, gloo in CPU tests).

One process per GPU.  The block map itself partitions the work
(tri_map_init(rank, world): contiguous, area-balanced omega ranges snapped to
tile rows), so EDM and the dummy kernel need no collective at all.  The real
exchange steps of the path are here:

* ``allreduce_count``  -- the collision count, SUM over ranks (8 bytes);
* ``allreduce_energy`` -- per-particle triplet energies, SUM (n fp64);
* ``halo_exchange``    -- the CA's boundary rows: the rank owning rows
  [R0, R1) needs row R0 - 1 (from the rank that owns it) and row R1, every
  generation, point to point.

Only torch.distributed calls live here -- no compute.  With the gloo backend
CUDA tensors are staged through host copies (gloo has no CUDA P2P).
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


def _gloo() -> bool:
    return dist.get_backend() == "gloo"


def allreduce_count(count: torch.Tensor) -> torch.Tensor:
    """SUM the u64 collision count (stored as int64) across ranks, in place."""
    if dist.is_initialized() and dist.get_world_size() > 1:
        if _gloo() and count.is_cuda:
            h = count.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM)
            count.copy_(h)
        else:
            dist.all_reduce(count, op=dist.ReduceOp.SUM)
    return count


def allreduce_energy(energy: torch.Tensor) -> torch.Tensor:
    """SUM the per-particle fp64 triplet energies across ranks, in place."""
    return allreduce_count(energy)


def owner(bounds, r):
    """Rank whose row range [a, b) contains row r (None if none)."""
    for g, (a, b) in enumerate(bounds):
        if a <= r < b:
            return g
    return None


def halo_bytes(bounds, n: int, rank: int, k: int = 1):
    """Sizes of the packed halo blocks a rank receives: rows [R0-k, R0) and [R1, R1+k)."""
    R0, R1 = bounds[rank]
    a = T(R0) - T(max(R0 - k, 0))
    b = T(min(R1 + k, n)) - T(R1)
    return a, b


def halo_exchange(state: torch.Tensor, bounds, n: int, rank: int, above: torch.Tensor | None,
                  below: torch.Tensor | None, k: int = 1):
    """Exchange the CA boundary rows of this rank's packed slice ``state``.

    bounds[g] = (row_begin, row_end) of rank g (every rank computes the same
    list from tri_map_init; no communication).  ``above`` receives the k packed
    rows [R0-k, R0), ``below`` the k rows [R1, R1+k) (k = 1: the single
    neighbour rows of tri_ca_step; k > 1: the deep halos of tri_ca_steps).
    Rows are contiguous in the packed Eq. 1 slice, so the sends are views.
    Ranks that own no rows take no part; a rank's k halo rows must all belong to
    one neighbour (every non-empty rank owns >= k rows).
    """
    R0, R1 = bounds[rank]
    if R1 <= R0:
        return
    sends, recvs = [], []
    if R0 > 0:                                   # my first k rows are the "below" halo of owner(R0-1)
        g = owner(bounds, R0 - 1)
        if owner(bounds, max(R0 - k, 0)) != g:
            raise ValueError("deep halo spans several ranks: every rank needs >= k rows")
        sends.append((state[0:T(min(R0 + k, R1)) - T(R0)], g))
        recvs.append((above, g))
    if R1 < n:                                   # my last k rows are the "above" halo of owner(R1)
        g = owner(bounds, R1)
        if owner(bounds, min(R1 + k, n) - 1) != g:
            raise ValueError("deep halo spans several ranks: every rank needs >= k rows")
        first = max(R1 - k, R0)
        sends.append((state[T(first) - T(R0):T(R1) - T(R0)], g))
        recvs.append((below, g))
    if not sends:
        return
    staged = _gloo() and state.is_cuda
    ops, host_recvs = [], []
    for t, g in sends:
        ops.append(dist.P2POp(dist.isend, t.cpu() if staged else t.contiguous(), g))
    for t, g in recvs:
        buf = torch.empty(t.shape, dtype=t.dtype) if staged else t
        host_recvs.append((buf, t))
        ops.append(dist.P2POp(dist.irecv, buf, g))
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    if staged:
        for buf, t in host_recvs:
            t.copy_(buf)
