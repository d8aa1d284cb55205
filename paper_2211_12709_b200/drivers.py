"""Verification drivers over the device path.

Rank-generic drivers with the reference's names, options and result
dictionaries (d/bench.py:60-356), running on the libdfno kernels and the
process-group / thread communicators, so the reference's ``parity``,
``adjoint`` and ``commvolume`` checks (SPEC criteria 1, 2, 4) and its
finite-difference gradient check (criterion 3) run unchanged on B200:

  drive_parity_forward  distributed forward vs the undistributed (P = 1)
                        forward of the same weights and input -- the
                        decomposition-invariance half of the reference's
                        oracle check; the numpy oracle itself is test
                        infrastructure (tests/, oracle/) and is not imported
  drive_adjoint         <L x, y> = <x, L^T y> for broadcast / reduce-sum and
                        for a repartition / its reverse (d/bench.py:131-184)
  drive_gradient        central finite differences vs the adjoint backward
                        along random parameter directions (d/bench.py:229-280)
  drive_comm_volume     measured repartition traffic == predicted_block_volume
                        (d/bench.py:314-356), integer-exact
  make_dataset          the synthetic spectral-propagator problem
                        (d/bench.py:403-430): same PCG64 draws, transforms
                        and mixing in float64 on the device
  drive_train           a full training run on it (d/bench.py:433-508):
                        train_step epochs, globally reduced test MSE / MAE /
                        R^2 per epoch, optional checkpoint
"""

from __future__ import annotations

import hashlib
from typing import Optional

import numpy as np
import torch

from .comm import REPARTITION, Communicator, run_ranks
from .fno import (
    ActivationKind,
    FnoConfig,
    FnoParams,
    ForwardCache,
    fno_backward,
    fno_block_forward,
    fno_forward,
    init_params,
    predicted_block_volume,
    shard_params,
    slice_local,
    _W_LABELS,
)
from .errors import ExtensionMissingError
from .partition import Partition
from .spectral import ModeSpec, retained_indices
from .training import AdamState, global_output_count, train_step
from .tensor import DATA_LABELS, DenseTensor, DimLabel, DType


def config_from_opts(opts: dict) -> FnoConfig:
    """Reference d/bench.py:60-73."""
    grid, modes = opts["grid"], opts["modes"]
    return FnoConfig(nx=grid[0], ny=grid[1], nz=grid[2], nt=grid[3],
                     in_channels=opts.get("in_channels", opts["channels"]),
                     out_channels=opts.get("out_channels", opts["channels"]), hidden_channels=opts["channels"],
                     modes=ModeSpec.of_xyzt(*modes), num_blocks=opts.get("blocks", 4),
                     activation=ActivationKind(opts.get("activation", "gelu")),
                     dtype=DType(opts.get("dtype", "real64")), num_ranks=opts["workers"])


def _device(comm: Communicator) -> torch.device:
    return comm.device if comm.device.type == "cuda" else torch.device("cuda", torch.cuda.current_device())


def _rng_input(config: FnoConfig, batch: int, seed: int, device) -> DenseTensor:
    """Reference d/bench.py:76-80 (same PCG64 stream), placed on ``device``."""
    rng = np.random.default_rng(seed)
    data = rng.standard_normal((batch, config.in_channels) + config.grid).astype(config.dtype.np_dtype)
    return DenseTensor(DATA_LABELS, torch.from_numpy(data).to(device))


def _rel_err(a: torch.Tensor, b: torch.Tensor) -> float:
    """Reference d/bench.py:83-85."""
    scale = max(float(a.abs().max()), float(b.abs().max()), 1e-300)
    return float((a - b).abs().max()) / scale


def _complex_dot(comm: Communicator, a: torch.Tensor, b: torch.Tensor, label: str) -> complex:
    local = complex(torch.vdot(a.reshape(-1).to(torch.complex128), b.reshape(-1).to(torch.complex128)))
    return complex(comm.allreduce_sum_scalar(local.real, label=f"{label}.re"),
                   comm.allreduce_sum_scalar(local.imag, label=f"{label}.im"))


def _digest(t: torch.Tensor) -> str:
    return hashlib.sha256(t.detach().cpu().contiguous().numpy().tobytes()).hexdigest()


def drive_parity_forward(comm: Communicator, opts: dict, serial_forward=None) -> Optional[dict]:
    """Distributed forward vs a serial forward on identical inputs and weights
    (reference d/bench.py:100-124).  ``serial_forward(x_global, params,
    serial_config) -> tensor`` is the reference's ``serial_fno_forward``
    slot: the tests pass the all-at-once float64 oracle
    (oracle/fno_oracle.py); without one the undistributed (P = 1) device
    forward is the comparison."""
    config = config_from_opts(opts)
    batch, seed = opts.get("batch", 1), opts["seed"]
    dev = _device(comm)
    params = init_params(config, seed, device=dev)
    x_global = _rng_input(config, batch, seed + 1000, dev)
    local = slice_local(x_global, config.x_partition(), comm.rank)
    before = comm.stats.snapshot()
    y_local = fno_forward(comm, local, shard_params(params, config, comm.rank), config)
    delta = comm.stats.minus(before)
    elems = comm.allreduce_sum_scalar(float(delta.get(REPARTITION).elements), label="parity.elems")
    gathered = comm.gather(y_local, config.x_partition(), root=0, label="parity.gather")
    if comm.rank != 0:
        return None
    serial_cfg = config_from_opts(dict(opts, workers=1))
    if serial_forward is not None:
        ref = serial_forward(x_global, params, serial_cfg)
        ref = ref.data if isinstance(ref, DenseTensor) else ref
    else:
        ref = run_ranks(1, lambda c: fno_forward(c, x_global, params, serial_cfg), device=dev)[0].data
    return {"max_rel_err": _rel_err(gathered.data, torch.as_tensor(ref, device=gathered.data.device)),
            "repart_calls_per_rank": delta.get(REPARTITION).calls,
            "repart_elements_total": int(elems), "output_digest": _digest(gathered.data)}


def drive_adjoint(comm: Communicator, opts: dict) -> Optional[dict]:
    """Dot tests of the communicating primitives (reference d/bench.py:131-184)."""
    pairs, seed, world = opts.get("pairs", 20), opts["seed"], comm.world_size
    shape = tuple(opts.get("shape", (3, 4, 5)))
    labels = (DimLabel.B, DimLabel.C, DimLabel.Z)
    dev = _device(comm)

    def cplx(rng, shp):
        return torch.from_numpy(rng.standard_normal(shp) + 1j * rng.standard_normal(shp)).to(dev)

    max_b = 0.0
    for trial in range(pairs):
        x = DenseTensor(labels, cplx(np.random.default_rng(seed + trial), shape))
        y_local = DenseTensor(labels, cplx(np.random.default_rng(seed + 7000 + trial * world + comm.rank), shape))
        bx = comm.broadcast(x if comm.rank == 0 else None, root=0, label="adj.b")
        lhs = _complex_dot(comm, bx.data, y_local.data, "adj.lhs")
        red = comm.reduce_sum(y_local, root=0, label="adj.r")
        if comm.rank == 0:
            rhs = complex(torch.vdot(x.data.reshape(-1), red.data.reshape(-1).to(x.data.device)))
            max_b = max(max_b, abs(lhs - rhs) / max(abs(lhs), abs(rhs), 1e-300))
    max_r = 0.0
    nx, ny = opts.get("repart_extents", (8, 6))
    src, dst = Partition.block(DimLabel.X, nx, world), Partition.block(DimLabel.Y, ny, world)
    for trial in range(pairs):
        rng = np.random.default_rng(seed + 3000 + trial * (comm.rank + 1))
        xl = DenseTensor((DimLabel.X, DimLabel.Y), cplx(rng, (src.extent_of(comm.rank), ny)))
        yl = DenseTensor((DimLabel.X, DimLabel.Y), cplx(rng, (nx, dst.extent_of(comm.rank))))
        lhs = _complex_dot(comm, comm.repartition(xl, src, dst, label="adj.fwd").data, yl.data, "adj.rl")
        rhs = _complex_dot(comm, xl.data, comm.repartition(yl, dst, src, label="adj.rev").data, "adj.rr")
        max_r = max(max_r, abs(lhs - rhs) / max(abs(lhs), abs(rhs), 1e-300))
    if comm.rank != 0:
        return None
    return {"broadcast_reduce_max_err": max_b, "repartition_max_err": max_r}


def _loss_half_norm(comm, config, params_local, x_local) -> float:
    y = fno_forward(comm, x_local, params_local, config)
    return comm.allreduce_sum_scalar(0.5 * float((y.data.double() ** 2).sum()), label="fd.loss")


def _perturb(params: FnoParams, direction: FnoParams, h: float) -> FnoParams:
    def add(a, d):
        return DenseTensor(a.labels, a.data + h * d.data.to(a.data.device))

    return FnoParams(add(params.we, direction.we), add(params.wd, direction.wd),
                     tuple(add(w, d) for w, d in zip(params.blocks, direction.blocks)), sharded=params.sharded)


def _random_direction(config: FnoConfig, seed: int, device) -> FnoParams:
    """Reference d/bench.py:201-226 (same stream)."""
    rng = np.random.default_rng(seed)
    real, cplx = config.dtype.np_dtype, config.complex_dtype.np_dtype
    we = rng.standard_normal((config.in_channels, config.hidden_channels)).astype(real)
    wd = rng.standard_normal((config.hidden_channels, config.out_channels)).astype(real)
    shape = config.spectral_weight_shape()
    labels = (DimLabel.C, DimLabel.CO, DimLabel.KX, DimLabel.KY, DimLabel.KZ, DimLabel.KT)
    blocks = tuple(DenseTensor(labels, torch.from_numpy(
        (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(cplx)).to(device))
        for _ in range(config.num_blocks))
    return FnoParams(DenseTensor((DimLabel.C, DimLabel.CO), torch.from_numpy(we).to(device)),
                     DenseTensor((DimLabel.C, DimLabel.CO), torch.from_numpy(wd).to(device)), blocks, sharded=False)


def drive_gradient(comm: Communicator, opts: dict) -> Optional[dict]:
    """Central finite differences of 0.5||y||^2 vs <grad, d> (reference
    d/bench.py:229-280)."""
    config = config_from_opts(opts)
    batch, seed = opts.get("batch", 1), opts["seed"]
    directions, h = opts.get("directions", 20), opts.get("step", 1e-6)
    dev = _device(comm)
    params = init_params(config, seed, device=dev)
    x_local = slice_local(_rng_input(config, batch, seed + 1000, dev), config.x_partition(), comm.rank)
    local_params = shard_params(params, config, comm.rank)
    cache = ForwardCache()
    y = fno_forward(comm, x_local, local_params, config, cache=cache)
    _, grads = fno_backward(comm, DenseTensor(y.labels, y.data.clone()), local_params, config, cache)
    errors = []
    for trial in range(directions):
        direction = _random_direction(config, seed + 5000 + trial, dev)
        dir_local = shard_params(direction, config, comm.rank)
        inner = sum(float(torch.vdot(g.data.reshape(-1), d.data.reshape(-1)).real)
                    for g, d in zip(grads.blocks, dir_local.blocks))
        if comm.rank == 0:
            inner += float((grads.we.data * direction.we.data).sum()) + float((grads.wd.data * direction.wd.data).sum())
        analytic = comm.allreduce_sum_scalar(inner, label="fd.inner")
        plus = _loss_half_norm(comm, config, shard_params(_perturb(params, direction, +h), config, comm.rank), x_local)
        minus = _loss_half_norm(comm, config, shard_params(_perturb(params, direction, -h), config, comm.rank),
                                x_local)
        numeric = (plus - minus) / (2.0 * h)
        errors.append(abs(numeric - analytic) / max(abs(numeric), abs(analytic), 1e-300))
    if comm.rank != 0:
        return None
    return {"max_rel_err": max(errors), "errors": errors,
            "ky_extent": len(config.ky_partition().range_of(comm.rank))}


def drive_comm_volume(comm: Communicator, opts: dict) -> Optional[dict]:
    """Measured repartition traffic vs the exact prediction (reference
    d/bench.py:314-356)."""
    config = config_from_opts(opts)
    batch, seed = opts.get("batch", 1), opts["seed"]
    dev = _device(comm)
    local_params = shard_params(init_params(config, seed, device=dev), config, comm.rank)
    rng = np.random.default_rng(seed + comm.rank)
    shape = (batch, config.hidden_channels, config.x_partition().extent_of(comm.rank), config.ny, config.nz,
             config.nt)
    hidden = DenseTensor(DATA_LABELS, torch.from_numpy(rng.standard_normal(shape).astype(config.dtype.np_dtype)).to(dev))
    before = comm.stats.snapshot()
    fno_block_forward(comm, hidden, local_params.blocks[0], config, label="vol")
    bd = comm.stats.minus(before).get(REPARTITION)
    block_total = comm.allreduce_sum_scalar(float(bd.elements), label="vol.b")
    block_bytes = comm.allreduce_sum_scalar(float(bd.bytes), label="vol.bb")
    x_local = slice_local(_rng_input(config, batch, seed + 1, dev), config.x_partition(), comm.rank)
    before = comm.stats.snapshot()
    fno_forward(comm, x_local, local_params, config)
    fd = comm.stats.minus(before).get(REPARTITION)
    fwd_total = comm.allreduce_sum_scalar(float(fd.elements), label="vol.f")
    if comm.rank != 0:
        return None
    p = predicted_block_volume(config, batch)
    return {"block_repart_calls_per_rank": bd.calls, "block_elements_total": int(block_total),
            "block_bytes_total": int(block_bytes), "forward_repart_calls_per_rank": fd.calls,
            "forward_elements_total": int(fwd_total), "predicted_per_repartition": p.per_repartition_elements,
            "predicted_per_block": p.per_block_elements, "predicted_per_forward": p.per_forward_elements,
            "predicted_naive": p.naive_per_repartition_elements, "reduction_ratio": p.reduction_ratio,
            "bytes_per_element": p.bytes_per_element}


def make_dataset(config: FnoConfig, samples: int, seed: int, device=None) -> tuple:
    """(inputs, targets) of the synthetic problem (reference d/bench.py:403-430):
    white-noise inputs pushed through a fixed random truncated-spectral
    propagator.  The random draws are the reference's (numpy PCG64, same order
    and shapes).  The propagator is itself one spectral block without
    activation -- truncated x/y/z/t DFT, per-mode channel mixing, zero padding,
    inverse DFT, real part -- so it runs on libdfno's block kernels
    (``fno_block_forward``): with c = max(c_in, c_out) channels (zero-padded
    inputs, the propagator embedded in a c x c weight W[i, o] = P[o, i]) and in
    float64 like the reference, then cast once to the config's real dtype.
    Both tensors are returned on ``device`` (a CUDA device: there is no host
    path), shaped (samples, c, Nx, Ny, Nz, Nt)."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise ExtensionMissingError("make_dataset runs its transforms on libdfno's CUDA kernels (no host path)")
    rng = np.random.default_rng(seed)
    keep = [retained_indices(n, m) for n, m in zip(config.grid, config.mode_counts)]
    r_shape = tuple(len(k) for k in keep)
    cin, cout = config.in_channels, config.out_channels
    scale = 1.0 / np.sqrt(2.0 * cin)
    prop = scale * (rng.standard_normal((cout, cin) + r_shape) + 1j * rng.standard_normal((cout, cin) + r_shape))
    inputs = torch.from_numpy(rng.standard_normal((samples, cin) + config.grid)).to(dev)
    c = max(cin, cout)
    block = FnoConfig(*config.grid, c, c, c, config.modes, 1, ActivationKind.IDENTITY, DType.REAL64, 1)
    x = torch.zeros((samples, c) + config.grid, dtype=torch.float64, device=dev)
    x[:, :cin] = inputs
    w = torch.zeros((c, c) + r_shape, dtype=torch.complex128, device=dev)
    w[:cin, :cout] = torch.from_numpy(np.ascontiguousarray(prop.transpose((1, 0) + tuple(range(2, 6))))).to(dev)

    def body(comm):
        return fno_block_forward(comm, DenseTensor(DATA_LABELS, x), DenseTensor(_W_LABELS, w), block,
                                 label="dataset").data

    targets = run_ranks(1, body, device=dev)[0][:, :cout]
    real = torch.float32 if config.dtype == DType.REAL32 else torch.float64
    return inputs.to(real).contiguous(), targets.to(real).contiguous()


def drive_train(comm: Communicator, opts: dict) -> Optional[dict]:
    """Training run on the synthetic problem (reference d/bench.py:433-508).
    Every rank regenerates the dataset from the seed and keeps its x slab on
    the device; the per-epoch rows are globally reduced, so they do not
    depend on the rank count."""
    config = config_from_opts(opts)
    seed = opts["seed"]
    n_train, n_test = opts.get("train_samples", 200), opts.get("test_samples", 50)
    batch, lr, epochs = opts.get("batch", 10), opts.get("lr", 2e-3), opts.get("epochs", 50)
    stop_r2 = opts.get("early_stop_r2")
    dev = _device(comm)
    inputs, targets = make_dataset(config, n_train + n_test, seed + 9000, device=dev)
    my_x = config.x_partition().range_of(comm.rank).as_slice()
    inputs, targets = inputs[:, :, my_x].contiguous(), targets[:, :, my_x].contiguous()

    def local_pair(lo: int, hi: int) -> tuple:
        return DenseTensor(DATA_LABELS, inputs[lo:hi]), DenseTensor(DATA_LABELS, targets[lo:hi])

    params = shard_params(init_params(config, seed, device=dev), config, comm.rank)
    state = AdamState()
    test_t = targets[n_train:].double()
    test_count = global_output_count(config, n_test)
    test_mean = comm.allreduce_sum_scalar(float(test_t.sum()), label="tr.mean") / test_count
    sst_local = float(((test_t - test_mean) ** 2).sum())

    def evaluate() -> tuple:
        sse = sae = 0.0
        for lo in range(n_train, n_train + n_test, batch):
            x_local, t_local = local_pair(lo, min(lo + batch, n_train + n_test))
            resid = (fno_forward(comm, x_local, params, config).data - t_local.data).double()
            sse += float((resid * resid).sum())
            sae += float(resid.abs().sum())
        sse = comm.allreduce_sum_scalar(sse, label="ev.sse")
        sae = comm.allreduce_sum_scalar(sae, label="ev.sae")
        sst = comm.allreduce_sum_scalar(sst_local, label="ev.sst")
        return sse / test_count, sae / test_count, 1.0 - sse / sst

    mse0, mae0, r20 = evaluate()
    metrics = [{"epoch": 0, "train_mse_median": None, "test_mse": mse0, "test_mae": mae0, "test_r2": r20}]
    for epoch in range(1, epochs + 1):
        losses = []
        for lo in range(0, n_train, batch):
            x_local, t_local = local_pair(lo, min(lo + batch, n_train))
            params, loss = train_step(comm, x_local, t_local, params, state, lr, config)
            losses.append(loss)
        mse, mae, r2 = evaluate()
        metrics.append({"epoch": epoch, "train_mse_median": float(np.median(losses)), "test_mse": mse,
                        "test_mae": mae, "test_r2": r2})
        if stop_r2 is not None and r2 > stop_r2:
            break
    if opts.get("checkpoint"):
        from .dtns import gather_params, save_checkpoint

        full = gather_params(comm, params, config)
        if comm.rank == 0:
            save_checkpoint(opts["checkpoint"], full, config, seed)
    if comm.rank != 0:
        return None
    return {"metrics": metrics, "epochs_run": metrics[-1]["epoch"]}


__all__ = ["config_from_opts", "drive_parity_forward", "drive_adjoint", "drive_gradient", "drive_comm_volume",
           "make_dataset", "drive_train"]
