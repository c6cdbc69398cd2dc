"""Multi-process tests of the distributed plumbing (-m "not gpu"): gloo backend,
world size 2 and 3, on CPU tensors.  The partition comes from the real C ABI
(tri_map_init is host code); the per-rank CA generation is the CPU oracle run on
the rows the rank owns plus its received halos, so the test checks that the
exchange delivers exactly the rows the kernel would read: the distributed run
must equal the single-process oracle bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def T(r):
    return r * (r + 1) // 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _ca_worker(rank, world, port, n, rho, steps, q, k=1):
    try:
        _init(rank, world, port)
        import oracle
        from paper_1609_01490_b200 import dist as tdist, inputs, tri
        maps = [tri.tri_map_init(n, rho, 1, g, world, 1) for g in range(world)]
        bounds = [(m.row_begin, m.row_end) for m in maps]
        m = maps[rank]
        full0 = inputs.ca_state(n, 42)
        state = torch.from_numpy(full0[m.out_offset:m.out_offset + m.out_cells].copy())
        R0, R1 = bounds[rank]
        na, nb = tdist.halo_bytes(bounds, n, rank, k)
        above = torch.zeros(max(na, 1), dtype=torch.uint8)
        below = torch.zeros(max(nb, 1), dtype=torch.uint8)
        for _ in range(steps):
            tdist.halo_exchange(state, bounds, n, rank, above if R0 > 0 else None, below if R1 < n else None, k)
            if R1 > R0:
                # the rank's rows plus its k-deep halos, everything else dead; k
                # generations of the oracle are exact on [R0, R1) (light cone)
                work = np.zeros(T(n), np.uint8)
                work[T(R0):T(R1)] = state.numpy()
                if R0 > 0:
                    work[T(max(R0 - k, 0)):T(R0)] = above.numpy()[:na]
                if R1 < n:
                    work[T(R1):T(min(R1 + k, n))] = below.numpy()[:nb]
                for _ in range(k - 1):
                    work = oracle.ca_step(n, work)
                state = torch.from_numpy(oracle.ca_step_rows(n, work, R0, R1).copy())
        parts = [None] * world
        dist.all_gather_object(parts, state.numpy().tobytes())
        cnt = torch.tensor([rank + 1], dtype=torch.int64)
        tdist.allreduce_count(cnt)
        e = torch.full((5,), float(rank), dtype=torch.float64)
        tdist.allreduce_energy(e)
        if rank == 0:
            q.put((b"".join(parts), int(cnt.item()), e.tolist()))
        dist.destroy_process_group()
    except Exception as ex:  # surface worker errors
        q.put(repr(ex))
        raise


@pytest.mark.parametrize("world,n,rho,k", [(2, 700, 128, 1), (3, 1000, 128, 1), (2, 300, 256, 1),
                                           (3, 900, 128, 3), (2, 600, 128, 8)])
def test_ca_halo_exchange_matches_oracle(orc, world, n, rho, k):
    from paper_1609_01490_b200 import inputs
    steps = 4 if k == 1 else 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ca_worker, args=(g, world, port, n, rho, steps, q, k)) for g in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    assert not isinstance(res, str), res
    data, cnt, e = res
    got = np.frombuffer(data, np.uint8)
    assert np.array_equal(got, orc.ca_run(n, inputs.ca_state(n, 42), steps * k))
    assert cnt == world * (world + 1) // 2
    assert e == [float(sum(range(world)))] * 5


# ---------------------------------------------------------------- allreduce paths
# Collision and triplet ranks own plain contiguous omega ranges (tri_map_init /
# tet_map_init with snap = 0) and sum their partials with all_reduce.  Each worker
# computes its partial over exactly its tiles (host lambda / tetrahedral map from the
# C ABI), so the reduced result equals the single-process oracle only if the
# partition covers every tile once and the collective sums correctly.
def _tile_worker(rank, world, port, kind, n, rho, q):
    try:
        _init(rank, world, port)
        from paper_1609_01490_b200 import dist as tdist, inputs, tri
        if kind == "collide":
            # 11-bit-quantised spheres: every fp32 op of the predicate is exact, so an
            # fp64 evaluation decides identically (the oracle pin in test_oracle_pins)
            s = inputs.spheres_quantized(n, 7, 11, 0.1).astype(np.float64)
            m = tri.tri_map_init(n, rho, 1, rank, world, 0)
            cnt = 0
            for w in range(m.omega_begin, m.omega_end):
                bi, bj = tri.tri_lambda(w)
                I = np.arange(bi * rho, min(n, bi * rho + rho))
                J = np.arange(bj * rho, min(n, bj * rho + rho))
                if len(I) == 0 or len(J) == 0:
                    continue
                d = s[I][:, None, :3] - s[J][None, :, :3]
                d2 = (d * d).sum(-1)
                rr = s[I][:, None, 3] + s[J][None, :, 3]
                cnt += int(((d2 < rr * rr) & (J[None, :] < I[:, None])).sum())
            c = torch.tensor([cnt], dtype=torch.int64)
            tdist.allreduce_count(c)
            res = int(c.item())
        else:
            p = inputs.points4(n, 42).astype(np.float64)
            m = tri.tet_map_init(n, rho, rank, world)
            e = np.zeros(n)
            for w in range(m.omega_begin, m.omega_end):
                ib, jb, kb = tri.tet_lambda(w)
                for pp in range(kb * rho, min(n, kb * rho + rho)):
                    for qq in range(ib * rho, min(n, ib * rho + rho)):
                        if qq >= pp:
                            continue
                        S = np.arange(jb * rho, min(n, jb * rho + rho))
                        S = S[S < qq]
                        if len(S) == 0:
                            continue
                        a = ((p[pp, :3] - p[qq, :3]) ** 2).sum()
                        b = ((p[qq, :3] - p[S, :3]) ** 2).sum(-1)
                        c2 = ((p[S, :3] - p[pp, :3]) ** 2).sum(-1)
                        abc = a * b * c2
                        P = (a + c2 - b) * (a + b - c2) * (b + c2 - a)
                        E = (1.0 + 3.0 * P / (8.0 * abc)) / abc ** 1.5
                        e[pp] += E.sum() / 3
                        e[qq] += E.sum() / 3
                        np.add.at(e, S, E / 3)
            et = torch.from_numpy(e)
            tdist.allreduce_energy(et)
            res = et.numpy().tolist()
        if rank == 0:
            q.put(res)
        dist.destroy_process_group()
    except Exception as ex:  # surface worker errors
        q.put(repr(ex))
        raise


def _run_tiles(kind, world, n, rho):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tile_worker, args=(g, world, port, kind, n, rho, q)) for g in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    assert not isinstance(res, str), res
    return res


@pytest.mark.parametrize("world,n,rho", [(2, 600, 16), (3, 517, 32)])
def test_collide_partition_allreduce_matches_oracle(orc, world, n, rho):
    from paper_1609_01490_b200 import inputs
    got = _run_tiles("collide", world, n, rho)
    want = orc.collide(inputs.spheres_quantized(n, 7, 11, 0.1))
    assert want > 100 and got == want


@pytest.mark.parametrize("world,n,rho", [(2, 48, 4), (3, 61, 8)])
def test_triplet_partition_allreduce_matches_oracle(orc, world, n, rho):
    from paper_1609_01490_b200 import inputs
    got = np.array(_run_tiles("triplet", world, n, rho))
    want = orc.triplet(inputs.points4(n, 42))
    assert np.allclose(got, want, rtol=1e-9, atol=1e-12 * np.abs(want).max())


# ---------------------------------------------------------------- fused P2P halo address arithmetic
@pytest.mark.parametrize("n,rho,world,k", [(2000, 128, 2, 4), (2000, 224, 3, 8), (5000, 128, 4, 16),
                                           (1500, 224, 2, 1), (32768, 224, 8, 8)])
def test_p2p_halo_addresses(n, rho, world, k):
    """Host-only: P2PHalo buffers built on the CPU for every rank and linked by address.
    Every cell a sender's kernel stores to a peer (include/tri.h: first k rows at
    peer_above + slice offset, last k rows at peer_below + slice offset) must land
    exactly where the receiver's next launch reads its halo (halo_above = rows
    [R0 - k, R0) from T(R0 - k), halo_below = rows [R1, R1 + k) from T(R1)), in the
    parity buffer that launch reads, and every peer pointer must be 16-byte aligned."""
    from paper_1609_01490_b200 import dist as tdist
    from paper_1609_01490_b200 import tri
    maps = [tri.tri_map_init(n, rho, 1, g, world, 1) for g in range(world)]
    bounds = [(m.row_begin, m.row_end) for m in maps]
    hs = [tdist.P2PHalo(bounds, n, g, k, device="cpu", exchange=False) for g in range(world)]
    for g, h in enumerate(hs):
        R0, R1 = bounds[g]
        up = tdist.owner(bounds, R0 - 1) if R0 > 0 else None
        down = tdist.owner(bounds, R1) if R1 < n else None
        h.link([t.data_ptr() for t in hs[up].below] if up is not None else None,
               [t.data_ptr() for t in hs[down].above] if down is not None else None)
    for e in range(3):
        for g, h in enumerate(hs):
            R0, R1 = bounds[g]
            _, _, pa, pb = h.args(e)                  # what launch e of rank g stores into
            for p in (pa, pb):
                assert p is None or p % 16 == 0
            if R0 > 0:                                # first k rows -> upper neighbour's below halo
                up = tdist.owner(bounds, R0 - 1)
                _, hb_next, _, _ = hs[up].args(e + 1)
                for r in range(R0, min(R0 + k, R1)):
                    for c in (0, r // 2, r):
                        assert pa + (T(r) + c - T(R0)) == hb_next.data_ptr() + (T(r) + c - T(R0))
                        assert 0 <= T(r) + c - T(R0) < hs[up].nb
            if R1 < n:                                # last k rows -> lower neighbour's above halo
                down = tdist.owner(bounds, R1)
                ha_next, _, _, _ = hs[down].args(e + 1)
                lo = max(R1 - k, 0)
                for r in range(max(R1 - k, R0), R1):
                    for c in (0, r // 2, r):
                        assert pb + (T(r) + c - T(R0)) == ha_next.data_ptr() + (T(r) + c - T(lo))
                        assert 0 <= T(r) + c - T(lo) < hs[down].na
