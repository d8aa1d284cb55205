"""Collectives and their accounting on CPU: the threaded in-process world and
a real 2-process gloo world (the same code path NCCL takes on the GPU box,
minus the device).  Mirrors the reference's t/test_comm.py checks: exact
off-rank counters, round trips, adjoint identities, mismatch detection."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2211_12709_b200 import (
    CollectiveMismatchError,
    CollectiveTimeoutError,
    Communicator,
    DenseTensor,
    DimLabel,
    Partition,
    run_ranks,
)
from paper_2211_12709_b200.comm import REPARTITION

CPU = torch.device("cpu")


def global_tensor(nx=8, ny=8, c=2):
    rng = np.random.default_rng(0)
    return rng.standard_normal((1, c, nx, ny))


def repartition_roundtrip(comm, g, nx, ny):
    src = Partition.block("x", nx, comm.world_size)
    dst = Partition.block("y", ny, comm.world_size)
    r = src.range_of(comm.rank)
    local = DenseTensor(("b", "c", "x", "y"), g[:, :, r.start:r.stop])
    moved = comm.repartition(local, src, dst, label="x->y")
    back = comm.repartition(moved, dst, src, label="y->x")
    return local, moved, back


@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_thread_repartition_counts_and_roundtrip(P):
    nx, ny = 8, 8
    g = global_tensor(nx, ny)

    def worker(comm):
        local, moved, back = repartition_roundtrip(comm, g, nx, ny)
        d = Partition.block("y", ny, P).range_of(comm.rank)
        assert np.array_equal(moved.numpy(), g[:, :, :, d.start:d.stop])
        assert np.array_equal(back.numpy(), local.numpy())
        return comm.stats.get(REPARTITION)

    stats = run_ranks(P, worker, device=CPU)
    # t/test_comm.py:122-140: 8x8 at P=4 moves 12 elements (per channel) per rank
    total = sum(s.elements for s in stats)
    xs = Partition.block("x", nx, P)
    ys = Partition.block("y", ny, P)
    expect = 2 * sum(xs.extent_of(r) * (ny - ys.extent_of(r)) for r in range(P)) * 2
    assert total == expect
    assert all(s.calls == 2 for s in stats)


def test_thread_repartition_is_adjoint():
    # <R x, y> = <x, R^T y> (t/test_comm.py)
    nx, ny, P = 9, 6, 3
    rng = np.random.default_rng(1)
    gx = rng.standard_normal((1, 2, nx, ny))
    gy = rng.standard_normal((1, 2, nx, ny))

    def worker(comm):
        src = Partition.block("x", nx, P)
        dst = Partition.block("y", ny, P)
        r, d = src.range_of(comm.rank), dst.range_of(comm.rank)
        lx = DenseTensor(("b", "c", "x", "y"), gx[:, :, r.start:r.stop])
        ly = DenseTensor(("b", "c", "x", "y"), gy[:, :, :, d.start:d.stop])
        rx = comm.repartition(lx, src, dst)
        rty = comm.repartition(ly, dst, src)
        a = float((rx.data * ly.data).sum())
        b = float((lx.data * rty.data).sum())
        return comm.allreduce_sum_scalar(a), comm.allreduce_sum_scalar(b)

    a, b = run_ranks(P, worker, device=CPU)[0]
    assert abs(a - b) < 1e-12 * abs(a)


def test_thread_broadcast_reduce_gather():
    P = 3

    def worker(comm):
        t = DenseTensor(("c", "co"), torch.full((2, 2), float(comm.rank + 1), dtype=torch.float64))
        b = comm.broadcast(t if comm.rank == 0 else None, root=0, label="b")
        s = comm.reduce_sum(t, root=0, label="s")
        part = Partition.block("x", 7, P)
        r = part.range_of(comm.rank)
        slab = DenseTensor(("x",), torch.arange(r.start, r.stop, dtype=torch.float64))
        gathered = comm.gather(slab, part)
        return b, s, gathered, comm.stats

    res = run_ranks(P, worker, device=CPU)
    for b, _, _, _ in res:
        assert torch.all(b.data == 1)
    assert torch.all(res[0][1].data == 6) and res[1][1] is None
    assert torch.equal(res[0][2].data, torch.arange(7, dtype=torch.float64))
    # broadcast accounting: root counts size * (P - 1) (reference comm.py:377-378)
    assert res[0][3].get("broadcast").elements == 4 * (P - 1)
    assert res[1][3].get("broadcast").elements == 0
    assert res[1][3].get("reduce_sum").elements == 4


def test_tag_mismatch_detected():
    def worker(comm):
        t = DenseTensor(("x",), torch.zeros(2))
        if comm.rank == 0:
            comm.broadcast(t, label="a")
        else:
            comm.reduce_sum(t, label="a")

    with pytest.raises(CollectiveMismatchError):
        run_ranks(2, worker, device=CPU)


def test_skipped_collective_times_out():
    def worker(comm):
        if comm.rank == 0:
            comm.allreduce_sum_scalar(1.0)

    with pytest.raises(CollectiveTimeoutError):
        run_ranks(2, worker, device=CPU, timeout=1.0)


# --------------------------------------------------------------------------
# real processes over gloo (world_size 2)
# --------------------------------------------------------------------------


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = Communicator.from_process_group()
        # (1) the hot-path exchange with uneven splits: XK -> KX for an
        # 5-plane x extent over 2 ranks (x blocks 3/2) and ry = 3 (ky 2/1)
        nx, ry, c, rzt = 5, 3, 2, 4
        xs = Partition.block("x", nx, world)
        ks = Partition.block("ky", ry, world)
        rng = np.random.default_rng(7)
        glob = rng.standard_normal((1, c, nx, ry, rzt)) + 1j * rng.standard_normal((1, c, nx, ry, rzt))
        xr, kr = xs.range_of(rank), ks.range_of(rank)
        mine = glob[:, :, xr.start:xr.stop]
        send = np.concatenate([mine[:, :, :, k.start:k.stop].reshape(-1) for k in ks.ranges])
        send_counts = [c * xs.extent_of(rank) * ks.extent_of(p) * rzt for p in range(world)]
        recv_counts = [c * xs.extent_of(p) * ks.extent_of(rank) * rzt for p in range(world)]
        recv = torch.empty(sum(recv_counts), dtype=torch.complex128)
        comm.exchange(torch.from_numpy(send), recv, send_counts, recv_counts, label="a2a")
        expect = np.concatenate([glob[:, :, x.start:x.stop, kr.start:kr.stop].reshape(-1) for x in xs.ranges])
        ok_a2a = np.array_equal(recv.numpy(), expect)
        # (2) generic repartition round trip
        g = global_tensor(6, 4)
        local, moved, back = repartition_roundtrip(comm, g, 6, 4)
        d = Partition.block("y", 4, world).range_of(rank)
        ok_rep = np.array_equal(moved.numpy(), g[:, :, :, d.start:d.stop]) and np.array_equal(back.numpy(),
                                                                                              local.numpy())
        # (3) broadcast with None on non-root, reduce, scalar allreduce
        t = DenseTensor(("c", "co"), torch.full((2, 3), float(rank + 1), dtype=torch.float32))
        b = comm.broadcast(t if rank == 0 else None, root=0, label="w")
        s = comm.reduce_sum(t, root=0, label="gw")
        tot = comm.allreduce_sum_scalar(float(rank + 1), label="loss")
        stats = {k: (v.calls, v.elements, v.bytes) for k, v in comm.stats.primitives.items()}
        q.put((rank, ok_a2a, ok_rep, bool(torch.all(b.data == 1)), None if s is None else float(s.data.sum()), tot,
               stats))
    finally:
        dist.destroy_process_group()


def test_gloo_two_process_world():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, ok_a2a, ok_rep, ok_b, s, tot, stats in results:
        assert ok_a2a and ok_rep and ok_b
        assert tot == 3.0
        # off-rank elements of the hot-path exchange: rank 0 sends 2*3*1*4, rank 1 sends 2*2*2*4
        rep = stats["repartition"]
        assert rep[0] == 3
    assert results[0][4] == 6 * 3.0
    assert results[1][4] is None
    # rank 0 off-rank elements: exchange c*x0*ky1*rzt = 2*3*1*4, then x->y and
    # y->x of the (1,2,6,4) tensor move 1*2*3*2 each
    assert results[0][6]["repartition"][1] == 24 + 12 + 12
