"""The multi-process path on one GPU: two processes (torch.distributed, gloo,
both on cuda:0) run the distributed forward + backward through
Communicator.from_process_group -- the code path one-process-per-GPU NCCL
runs take (process-group collectives, uneven all-to-all splits, rank-ordered
mixer-gradient reduction) -- and the gathered results are checked against
the numpy oracle.  The thread-rank tests (test_gpu_parity.py) cover P up to 8
with the same kernels; this covers the process boundary."""

import multiprocessing as mp
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GRID, MODES, C, BLOCKS = (9, 8, 8, 8), (4, 2, 3, 4), 3, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_2211_12709_b200 as P

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        comm = P.Communicator.from_process_group(device=dev)
        cfg = P.FnoConfig(*GRID, C, C, C, P.ModeSpec.of_xyzt(*MODES), BLOCKS, "gelu", "real32", world)
        params = P.init_params(cfg, 5, device=dev)
        lp = P.shard_params(params, cfg, rank)
        x = np.random.default_rng(11).standard_normal((1, C) + GRID).astype(np.float32)
        xl = P.slice_local(P.DenseTensor(P.DATA_LABELS, torch.from_numpy(x).to(dev)), cfg.x_partition(), rank)
        cache = P.ForwardCache()
        y = P.fno_forward(comm, xl, lp, cfg, cache)
        gx, grads = P.fno_backward(comm, y, lp, cfg, cache)
        q.put((rank, y.numpy(), gx.numpy(), grads.we.numpy(), grads.wd.numpy(),
               [g.numpy() for g in grads.blocks], comm.stats.get("repartition").elements))
    except Exception as e:  # pragma: no cover - reported by the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_processes_match_oracle():
    from oracle import fno_oracle as O

    import paper_2211_12709_b200 as P

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in procs), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert len(r) > 2, f"rank {r[0]} failed: {r[1]}"
    y = np.concatenate([r[1] for r in res], axis=2)
    gx = np.concatenate([r[2] for r in res], axis=2)
    # mixer grads are replicated and bit-identical across ranks (d/fno.py:501-508)
    assert np.array_equal(res[0][3], res[1][3]) and np.array_equal(res[0][4], res[1][4])
    cfg = P.FnoConfig(*GRID, C, C, C, P.ModeSpec.of_xyzt(*MODES), BLOCKS, "gelu", "real64", 1)
    params = P.init_params(cfg, 5, device="cpu")
    we, wd = params.we.numpy(), params.wd.numpy()
    blocks = [w.numpy() for w in params.blocks]
    x = np.random.default_rng(11).standard_normal((1, C) + GRID).astype(np.float32).astype(np.float64)
    # the fp32 run used fp32-rounded weights
    we32, wd32 = we.astype(np.float32).astype(np.float64), wd.astype(np.float32).astype(np.float64)
    bl32 = [b.astype(np.complex64).astype(np.complex128) for b in blocks]
    ry, cache = O.forward(x, we32, wd32, bl32, MODES, with_cache=True)
    rgx, rgwe, rgwd, rgws = O.backward(ry, we32, wd32, bl32, MODES, cache)
    assert O.rel_err(y, ry) < 1e-5
    assert O.rel_err(gx, rgx) < 1e-4
    assert O.rel_err(res[0][3], rgwe) < 1e-4 and O.rel_err(res[0][4], rgwd) < 1e-4
    ky = cfg.ky_partition()
    for i, gw in enumerate(rgws):
        shards = np.concatenate([res[r][5][i] for r in range(2)], axis=3)
        assert shards.shape == gw.shape
        assert O.rel_err(shards, gw) < 1e-4
    # exact off-rank element counts of the 2 * 2 * BLOCKS repartitions (d/fno.py:234-261)
    vol = P.predicted_block_volume(P.FnoConfig(*GRID, C, C, C, P.ModeSpec.of_xyzt(*MODES), BLOCKS, "gelu",
                                               "real32", 2))
    assert res[0][6] + res[1][6] == 2 * vol.per_forward_elements
    del ky
