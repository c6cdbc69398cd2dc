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


# ---------------------------------------------------------------------------
# Fused halo exchange (tri_ca_steps_p2p): the CA kernel itself stores its first /
# last k rows into the neighbours' halo buffers over NVLink (CUDA IPC mappings),
# so an epoch needs no send/recv -- only a stream-ordered 4-byte all-reduce that
# orders the peer stores before the neighbours' next launch.  Halo buffers are
# double-buffered by epoch parity: launch e reads its parity-e buffers and writes
# the neighbours' parity-(e+1) ones, which the neighbours last read in launch e-1
# (finished, by the all-reduce after it).

def peer_below_shift(bounds, rank: int, k: int) -> int:
    """T(R1 - k) - T(R0): where the sender's rows [R1 - k, R1) start in its slice."""
    R0, R1 = bounds[rank]
    return T(max(R1 - k, R0)) - T(R0)


class P2PHalo:
    """Double-buffered receive buffers of one rank plus the neighbours' buffers it
    stores into.  ``exchange=True`` swaps CUDA IPC handles over torch.distributed
    and maps the neighbours' buffers (one process per GPU); ``exchange=False``
    leaves the peers to ``link`` (ranks emulated in one process, in tests)."""

    def __init__(self, bounds, n: int, rank: int, k: int, device=None, exchange: bool = True):
        self.bounds, self.n, self.rank, self.k = bounds, n, rank, k
        R0, R1 = bounds[rank]
        self.R0, self.R1 = R0, R1
        self.na, self.nb = halo_bytes(bounds, n, rank, k)
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        # the above buffer's address must match the sender's store phase mod 16:
        # the sender writes its slice offset x at (its peer_below) + x, 16-byte aligned
        g_up = owner(bounds, R0 - 1) if R0 > 0 else None
        self.phase = (peer_below_shift(bounds, g_up, k) % 16) if g_up is not None else 0
        self._bufs = [torch.zeros(self.na + 32, dtype=torch.uint8, device=dev) for _ in range(2)]
        self._belows = [torch.zeros(max(self.nb, 1) + 16, dtype=torch.uint8, device=dev) for _ in range(2)]
        self.above = [b[self.phase:self.phase + max(self.na, 1)] for b in self._bufs]
        self.below = [b[:max(self.nb, 1)] for b in self._belows]
        self.peer_above = [None, None]     # addresses in the upper neighbour's below buffers
        self.peer_below = [None, None]     # base addresses for the lower neighbour's above buffers
        self._opened = []
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        if exchange:
            self._exchange()

    def handles(self):
        from . import tri
        return {"above": [tri.tri_ipc_handle(t) for t in self.above],
                "below": [tri.tri_ipc_handle(t) for t in self.below]}

    def link(self, up_below_addrs, down_above_addrs):
        """Peers given as addresses: the upper neighbour's below buffers and the lower
        neighbour's above buffers (per parity), or None at the domain edge."""
        shift = peer_below_shift(self.bounds, self.rank, self.k)
        for p in range(2):
            self.peer_above[p] = None if up_below_addrs is None else up_below_addrs[p]
            self.peer_below[p] = None if down_above_addrs is None else down_above_addrs[p] - shift

    def _exchange(self):
        """Collective and failure-safe: every rank takes part in both gathers and, if
        any rank failed to export or map a handle, every rank raises (none is left
        waiting in a collective)."""
        from . import tri
        world = dist.get_world_size()
        try:
            mine, err = self.handles(), None
        except Exception as ex:  # noqa: BLE001 -- reported to every rank below
            mine, err = None, repr(ex)
        allh = [None] * world
        dist.all_gather_object(allh, (mine, err))
        bad = [e for _, e in allh if e]
        if bad:
            raise RuntimeError(f"CUDA IPC handle export failed: {bad[0]}")
        allh = [h for h, _ in allh]
        up = owner(self.bounds, self.R0 - 1) if self.R0 > 0 and self.R1 > self.R0 else None
        down = owner(self.bounds, self.R1) if self.R1 < self.n and self.R1 > self.R0 else None

        def open_all(hs):
            out = []
            for h, off in hs:
                ptr, base = tri.tri_ipc_open(h, off)
                self._opened.append(base)
                out.append(ptr)
            return out
        try:
            self.link(open_all(allh[up]["below"]) if up is not None else None,
                      open_all(allh[down]["above"]) if down is not None else None)
            err = None
        except Exception as ex:  # noqa: BLE001
            err = repr(ex)
        errs = [None] * world
        dist.all_gather_object(errs, err)
        bad = [e for e in errs if e]
        if bad:
            self.close()
            raise RuntimeError(f"CUDA IPC mapping failed: {bad[0]}")

    def close(self):
        from . import tri
        for b in self._opened:
            tri.tri_ipc_close(b)
        self._opened = []

    def prime(self, state: torch.Tensor):
        """Parity-0 halos of the initial state (one ordinary exchange)."""
        halo_exchange(state, self.bounds, self.n, self.rank, self.above[0] if self.R0 > 0 else None,
                      self.below[0] if self.R1 < self.n else None, self.k)

    def args(self, epoch: int):
        """(halo_above, halo_below, peer_above, peer_below) for launch ``epoch``."""
        p, q = epoch % 2, (epoch + 1) % 2
        return (self.above[p] if self.R0 > 0 else None, self.below[p] if self.R1 < self.n else None,
                self.peer_above[q], self.peer_below[q])

    def epoch_barrier(self):
        """Order this launch's peer stores before the neighbours' next launch."""
        if not (dist.is_initialized() and dist.get_world_size() > 1):
            return
        if _gloo():
            torch.cuda.synchronize()
            dist.barrier()
        else:
            dist.all_reduce(self.flag)          # stream-ordered, 4 bytes
