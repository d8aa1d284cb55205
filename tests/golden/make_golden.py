"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference package read-only from /root/reference/pkg/src and
writes ``tests/golden/*.npz`` -- inputs, weights, forward outputs, gradients,
partition tables and communication counters of the reference's own drivers
(``fno_forward`` / ``fno_backward`` / ``serial_fno_forward`` over its
in-process transport).  The fixtures are committed; nothing at test time
reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from distfno.bench import DATA_LABELS, run_distributed  # noqa: E402
from distfno.comm import REPARTITION, run_ranks  # noqa: E402
from distfno.fno import (  # noqa: E402
    FnoConfig,
    ForwardCache,
    fno_backward,
    fno_forward,
    init_params,
    predicted_block_volume,
    shard_params,
    slice_local,
)
from distfno.oracle import serial_fno_forward  # noqa: E402
from distfno.partition import Partition, block_decompose, repartition_plan  # noqa: E402
from distfno.spectral import ModeSpec  # noqa: E402
from distfno.tensor import DenseTensor, DimLabel  # noqa: E402


def cfg_of(grid, modes, c, blocks, dtype, P, act="gelu", cin=None, cout=None):
    return FnoConfig(nx=grid[0], ny=grid[1], nz=grid[2], nt=grid[3], in_channels=cin or c,
                     out_channels=cout or c, hidden_channels=c, modes=ModeSpec.of_xyzt(*modes),
                     num_blocks=blocks, activation=act, dtype=dtype, num_ranks=P)


def rng_input(cfg, batch, seed):
    rng = np.random.default_rng(seed)
    data = rng.standard_normal((batch, cfg.in_channels) + cfg.grid)
    return DenseTensor(DATA_LABELS, data.astype(cfg.dtype.np_dtype))


def run_case(name, grid, modes, c, blocks, dtype, ranks, seed=11, batch=1, act="gelu", cin=None, cout=None):
    """Forward + backward (g = y, loss 0.5||y||^2 as d/bench.py:383) at every
    rank count; saves global x, weights, gathered y, gx, mixer grads and the
    gathered spectral-weight grads, plus per-rank repartition counters."""
    out = {}
    meta = {"grid": grid, "modes": modes, "channels": c, "blocks": blocks, "dtype": dtype, "ranks": ranks,
            "seed": seed, "batch": batch, "activation": act, "in_channels": cin or c, "out_channels": cout or c}
    base = cfg_of(grid, modes, c, blocks, dtype, 1, act, cin, cout)
    params = init_params(base, seed)
    x = rng_input(base, batch, seed + 1000)
    out["x"] = x.data
    out["we"] = params.we.data
    out["wd"] = params.wd.data
    for i, w in enumerate(params.blocks):
        out[f"w{i}"] = w.data
    out["y_serial"] = serial_fno_forward(x, params, base).data
    for P in ranks:
        cfg = cfg_of(grid, modes, c, blocks, dtype, P, act, cin, cout)
        xpart = cfg.x_partition()

        def worker(comm, cfg=cfg, xpart=xpart):
            lp = shard_params(params, cfg, comm.rank)
            local = slice_local(x, xpart, comm.rank)
            cache = ForwardCache()
            before = comm.stats.snapshot()
            y = fno_forward(comm, local, lp, cfg, cache=cache)
            fwd = comm.stats.minus(before)
            gx, grads = fno_backward(comm, DenseTensor(y.labels, y.data.copy()), lp, cfg, cache)
            both = comm.stats.minus(before)
            yg = comm.gather(y, xpart, label="g.y")
            gxg = comm.gather(gx, xpart, label="g.gx")
            counters = {k: [v.calls, v.elements, v.bytes] for k, v in fwd.primitives.items()}
            counters_all = {k: [v.calls, v.elements, v.bytes] for k, v in both.primitives.items()}
            return (yg, gxg, grads, counters, counters_all)

        res = run_ranks(P, worker)
        yg, gxg, grads, _, _ = res[0]
        out[f"y_p{P}"] = yg.data
        out[f"gx_p{P}"] = gxg.data
        out[f"gwe_p{P}"] = grads.we.data
        out[f"gwd_p{P}"] = grads.wd.data
        for i in range(blocks):
            out[f"gw{i}_p{P}"] = np.concatenate([r[2].blocks[i].data for r in res], axis=3)
        meta[f"counters_fwd_p{P}"] = [r[3] for r in res]
        meta[f"counters_fwdbwd_p{P}"] = [r[4] for r in res]
        vol = predicted_block_volume(cfg, batch)
        meta[f"predicted_p{P}"] = [vol.per_repartition_elements, vol.per_block_elements,
                                   vol.per_forward_elements, vol.naive_per_repartition_elements,
                                   vol.reduction_ratio, vol.bytes_per_element]
    np.savez_compressed(OUT / f"{name}.npz", **out)
    (OUT / f"{name}.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    print(name, {k: v.shape for k, v in out.items()})


def partitions():
    """block_decompose tables and repartition plans for extents <= 40,
    P <= 8 (bit-exact integer goldens; reference d/partition.py:47-66,
    :135-188)."""
    tables = {}
    for n in range(1, 41):
        for P in range(1, min(n, 8) + 1):
            tables[f"{n}/{P}"] = [[r.start, r.stop] for r in block_decompose(n, P)]
    plans = {}
    for (nx, ry, P) in [(8, 4, 2), (9, 4, 3), (16, 16, 8), (262, 16, 8), (10, 6, 4), (7, 7, 7)]:
        src = Partition.block(DimLabel.X, nx, P)
        dst = Partition.block(DimLabel.KY, ry, P)
        dims = [(DimLabel.B, 2), (DimLabel.C, 3), (DimLabel.X, nx), (DimLabel.KY, ry), (DimLabel.KZ, 4),
                (DimLabel.KT, 3)]
        for rank in range(P):
            plan = repartition_plan(src, dst, dims, rank)
            plans[f"{nx}/{ry}/{P}/{rank}"] = [
                [e.peer, [[r.start, r.stop] for r in e.send], [[r.start, r.stop] for r in e.recv]] for e in plan]
    (OUT / "partitions.json").write_text(json.dumps({"block_decompose": tables, "plans": plans}))


def init_digests():
    """sha256 of init_params arrays (reference d/fno.py:155-180)."""
    out = {}
    for (grid, modes, c, blocks, dtype, seed, cin, cout) in [
        ((8, 8, 8, 4), (2, 2, 2, 2), 2, 2, "real64", 11, None, None),
        ((16, 16, 16, 8), (4, 4, 4, 3), 2, 4, "real32", 5, None, None),
        ((9, 12, 8, 4), (2, 3, 2, 2), 3, 1, "real64", 0, 1, 2),
        ((32, 32, 32, 16), (8, 8, 8, 8), 20, 1, "real32", 42, None, None),
    ]:
        cfg = cfg_of(grid, modes, c, blocks, dtype, 1, cin=cin, cout=cout)
        p = init_params(cfg, seed)
        key = json.dumps([grid, modes, c, blocks, dtype, seed, cin, cout])
        out[key] = {k: hashlib.sha256(np.ascontiguousarray(v.data).tobytes()).hexdigest()
                    for k, v in p.named().items()}
    (OUT / "init_digests.json").write_text(json.dumps(out, indent=1))


def comm_volume_case():
    """The reference's measured == predicted case (t/test_fno.py:246-255)."""
    opts = {"grid": [9, 8, 6, 4], "modes": [2, 2, 2, 2], "channels": 2, "blocks": 2, "dtype": "real64",
            "seed": 0, "batch": 2, "activation": "gelu", "workers": 3}
    res = run_distributed("commvolume", opts, 3, "inproc")
    (OUT / "commvolume_9864_p3.json").write_text(json.dumps(res, indent=1, sort_keys=True))


def training_case():
    """The reference's Adam (d/training.py:52-74) on fixed real32 / complex64
    inputs over 3 steps, and its train_step (d/training.py:96-133) for 3
    steps at P = 1 and P = 2 on a small real32 config with a smooth target."""
    from distfno.training import AdamState, adam_update, train_step

    rng = np.random.default_rng(99)
    out = {}
    for name, dt in (("r32", np.float32), ("c64", np.complex64)):
        shape = (5, 7, 3)
        p0 = rng.standard_normal(shape)
        if dt == np.complex64:
            p0 = p0 + 1j * rng.standard_normal(shape)
        p0 = p0.astype(dt)
        out[f"adam_{name}_p0"] = p0
        st = AdamState()
        lab = ("c", "co", "kx") if dt == np.complex64 else ("c", "co", "x")
        p = DenseTensor(lab, p0)
        for k in range(3):
            g0 = rng.standard_normal(shape) * 10.0 ** (-k)
            if dt == np.complex64:
                g0 = g0 + 1j * rng.standard_normal(shape)
            g0 = g0.astype(dt)
            out[f"adam_{name}_g{k}"] = g0
            st.step += 1
            p = adam_update(st, "w", p, DenseTensor(lab, g0), 1e-3)
            out[f"adam_{name}_p{k + 1}"] = p.data.copy()
    meta = {"lr": 1e-3}
    grid, modes, c, blocks = (8, 8, 8, 4), (2, 2, 2, 2), 2, 2
    base = cfg_of(grid, modes, c, blocks, "real32", 1)
    params = init_params(base, 3)
    x = rng_input(base, 1, 44)
    xx = np.linspace(0.0, 1.0, grid[0])[None, None, :, None, None, None]
    y = (np.sin(2 * np.pi * xx) * np.ones((1, c) + grid)).astype(np.float32)
    out["train_x"], out["train_y"] = x.data, y
    for P in (1, 2):
        cfg = cfg_of(grid, modes, c, blocks, "real32", P)
        xpart = cfg.x_partition()

        def worker(comm, cfg=cfg, xpart=xpart):
            lp = shard_params(params, cfg, comm.rank)
            xl = slice_local(x, xpart, comm.rank)
            yl = slice_local(DenseTensor(DATA_LABELS, y), xpart, comm.rank)
            st = AdamState()
            losses = []
            for _ in range(3):
                lp, loss = train_step(comm, xl, yl, lp, st, 1e-3, cfg)
                losses.append(loss)
            return losses, lp

        res = run_ranks(P, worker)
        meta[f"train_losses_p{P}"] = res[0][0]
        out[f"train_we_p{P}"] = res[0][1].we.data
        out[f"train_wd_p{P}"] = res[0][1].wd.data
        for i in range(blocks):
            out[f"train_w{i}_p{P}"] = np.concatenate([r[1].blocks[i].data for r in res], axis=3)
    np.savez_compressed(OUT / "training_r32.npz", **out)
    (OUT / "training_r32.json").write_text(json.dumps(meta, indent=1))
    print("training", list(out))


TRAIN_OPTS = {"grid": [8, 8, 8, 4], "modes": [2, 2, 2, 2], "channels": 3, "in_channels": 1, "out_channels": 1,
              "blocks": 2, "dtype": "real32", "seed": 13, "train_samples": 6, "test_samples": 3, "batch": 2,
              "lr": 3e-2, "epochs": 4}


def train_case():
    """The reference's synthetic dataset (d/bench.py:403-430) and a short
    drive_train run (d/bench.py:433-508) at P = 1 and P = 2."""
    from distfno.bench import make_dataset

    cfg = cfg_of((8, 8, 8, 4), (2, 2, 2, 2), 3, 2, "real32", 1, cin=1, cout=2)
    x, y = make_dataset(cfg, 3, 77)
    out = {"ds_x": x, "ds_y": y}
    meta = {"dataset": {"grid": [8, 8, 8, 4], "modes": [2, 2, 2, 2], "channels": 3, "in_channels": 1,
                        "out_channels": 2, "blocks": 2, "dtype": "real32", "workers": 1, "samples": 3, "seed": 77},
            "opts": TRAIN_OPTS}
    for P in (1, 2):
        res = run_distributed("train", dict(TRAIN_OPTS, workers=P), P, "inproc")
        meta[f"train_p{P}"] = res
    np.savez_compressed(OUT / "train_ref.npz", **out)
    (OUT / "train_ref.json").write_text(json.dumps(meta, indent=1))
    print("train", meta["train_p1"]["metrics"][-1], meta["train_p2"]["metrics"][-1])


def dtns_case():
    """The reference's DTNS bytes (d/tensor.py:258-320) for four dtypes and
    a reference checkpoint directory (d/training.py:176-208)."""
    import shutil

    from distfno.tensor import tensor_to_bytes
    from distfno.training import save_checkpoint

    rng = np.random.default_rng(21)
    out = {}
    cases = {
        "r32": (("b", "c", "x", "y", "z", "t"), rng.standard_normal((1, 2, 3, 2, 2, 3)).astype(np.float32)),
        "r64": (("c", "co"), rng.standard_normal((3, 4))),
        "c64": (("c", "co", "kx", "ky"), (rng.standard_normal((2, 2, 3, 2)) + 1j * rng.standard_normal(
            (2, 2, 3, 2))).astype(np.complex64)),
        "c128": (("kz", "kt"), rng.standard_normal((2, 5)) + 1j * rng.standard_normal((2, 5))),
    }
    for k, (labels, data) in cases.items():
        out[f"{k}_data"] = data
        out[f"{k}_bytes"] = np.frombuffer(tensor_to_bytes(DenseTensor(labels, data)), dtype=np.uint8)
    np.savez_compressed(OUT / "dtns_ref.npz", **out)
    cfg = cfg_of((8, 8, 8, 4), (2, 2, 2, 2), 2, 2, "real32", 2, cin=1, cout=3)
    d = OUT / "ckpt_ref"
    shutil.rmtree(d, ignore_errors=True)
    save_checkpoint(str(d), init_params(cfg, 5), cfg, 5)
    print("dtns", sorted(out), sorted(p.name for p in d.iterdir()))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "dtns":
        dtns_case()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "train":
        train_case()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "training":
        training_case()
        sys.exit(0)
    training_case()
    train_case()
    dtns_case()
    partitions()
    init_digests()
    comm_volume_case()
    # t/test_fno.py:177-187 parity config (real64) at P = 1, 2, 4
    run_case("g8_c2_l2_f64", (8, 8, 8, 4), (2, 2, 2, 2), 2, 2, "real64", [1, 2, 4], seed=11)
    # acceptance criterion 1 config (t/test_acceptance.py:24-27): 16^3 x 8, modes (4,4,4,3), 4 blocks
    run_case("acc16_c2_l4_f64", (16, 16, 16, 8), (4, 4, 4, 3), 2, 4, "real64", [1, 8], seed=7)
    run_case("acc16_c2_l4_f32", (16, 16, 16, 8), (4, 4, 4, 3), 2, 4, "real32", [1, 8], seed=7)
    # uneven partitions, batch 2, in != hidden != out channels, relu
    run_case("uneven_9864_p3", (9, 8, 6, 4), (2, 2, 2, 2), 3, 2, "real64", [1, 3], seed=3, batch=2, act="relu",
             cin=2, cout=4)
    # odd extents (x not divisible, t odd) and full retention along t (2m >= N)
    run_case("odd_11x10x6x5_f64", (11, 10, 6, 5), (3, 2, 2, 3), 4, 2, "real64", [1, 2], seed=5, act="identity")
