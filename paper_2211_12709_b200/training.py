"""Distributed training step and Adam on B200 (the first "next" row of the
hot path).

Mirrors the reference's ``distfno.training`` (d/training.py:34-133): the
loss is the mean squared error over every output element globally, identical
on all ranks; the replicated encoder/decoder weights are updated from the
reduced gradient with identical arithmetic on every rank and asserted
bit-identical each step; the spectral weights update their ky shard locally.

Device work is three libdfno kernels per step besides the forward /
backward: the fused residual + loss + output-gradient pass (dfno_mse_grad),
and Adam on each parameter's real view (dfno_adam_out, written to a new array) with the reference's fp32
operation order.  Only the scalar loss crosses to the host.
"""

from __future__ import annotations

import ctypes
import math
import threading
from dataclasses import dataclass, field

import torch

from . import _lib
from .comm import Communicator
from .errors import DTypeMismatchError, NonFiniteLossError, ReplicationError, ShapeMismatchError
from .fno import FnoConfig, FnoParams, ForwardCache, fno_backward, fno_forward
from .tensor import DenseTensor, bit_equal


@dataclass
class AdamState:
    """First / second moments per parameter on the real view of complex
    weights (reference d/training.py:34-44); tensors live on the device."""

    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    step: int = 0
    m: dict = field(default_factory=dict)
    v: dict = field(default_factory=dict)


def _real_view(t: torch.Tensor) -> torch.Tensor:
    t = t.reshape(-1)
    return torch.view_as_real(t).reshape(-1) if t.is_complex() else t


def _geom_for(dtype: torch.dtype) -> _lib.Geom:
    real = {torch.float32: _lib.F32, torch.complex64: _lib.F32, torch.float64: _lib.F64,
            torch.complex128: _lib.F64}.get(dtype)
    if real is None:
        raise DTypeMismatchError(f"unsupported parameter dtype {dtype}")
    return _lib.make_geom(batch=1, c_in=1, c=1, c_out=1, grid=(1, 1, 1, 1), modes=(1, 1, 1, 1), retained=(1, 1, 1, 1),
                          nranks=1, rank=0, dtype=real, act=_lib.ACT_IDENTITY, x_starts=(0, 1), ky_starts=(0, 1))


def adam_update(state: AdamState, key: str, param: DenseTensor, grad: DenseTensor, lr: float) -> DenseTensor:
    """One Adam step for one parameter; returns the updated tensor
    (reference d/training.py:52-74).  ``state.step`` must already be advanced
    by the caller (once per training step)."""
    if not _lib.available():
        raise _lib.ExtensionMissingError("libdfno.so and a CUDA device are required (no CPU fallback)")
    lib = _lib.load()
    p_in = param.data.to("cuda").contiguous()
    p = torch.empty_like(p_in)  # the new parameter (the old one stays valid, as the reference's arrays do)
    gd = grad.data.to(p.device).contiguous()
    if gd.dtype != p.dtype or gd.shape != p.shape:
        raise ShapeMismatchError(f"{key}: gradient {tuple(gd.shape)} {gd.dtype} vs parameter {tuple(p.shape)} {p.dtype}")
    pin_v, pv, gv = _real_view(p_in), _real_view(p), _real_view(gd)
    if key not in state.m:
        state.m[key] = torch.zeros_like(pv)
        state.v[key] = torch.zeros_like(pv)
    g = _geom_for(p.dtype)
    _lib.check(lib.dfno_adam_out(ctypes.byref(g), pv.numel(), _lib.ptr(pin_v), _lib.ptr(pv), _lib.ptr(gv),
                                 _lib.ptr(state.m[key]), _lib.ptr(state.v[key]), float(lr), float(state.beta1),
                                 float(state.beta2), float(state.eps), int(state.step), _lib.stream_handle()),
               "dfno_adam_out")
    return DenseTensor(param.labels, p)


def _assert_replicated(comm: Communicator, t: DenseTensor, name: str) -> None:
    """Rank 0's copy broadcast and compared bitwise (d/training.py:77-82)."""
    reference = comm.broadcast(t if comm.rank == 0 else None, root=0, label=f"repl.{name}")
    if not bit_equal(reference, t):
        raise ReplicationError(f"replicated weight {name!r} diverged on rank {comm.rank}")


def global_output_count(config: FnoConfig, batch_size: int) -> int:
    """Elements of the global output (d/training.py:85-93)."""
    return batch_size * config.out_channels * config.nx * config.ny * config.nz * config.nt


class _LossBuffers(threading.local):
    # per thread: ranks of a ThreadWorld run concurrently in one process
    def __init__(self):
        self.key = None

    def get(self, n: int, like: torch.Tensor):
        key = (n, like.dtype, str(like.device))
        if self.key != key:
            k = ctypes.c_int()
            _lib.check(_lib.load().dfno_mse_partials(n, ctypes.byref(k)), "dfno_mse_partials")
            self.partials = torch.empty(k.value, dtype=torch.float64, device=like.device)
            self.sse = torch.empty(1, dtype=torch.float64, device=like.device)
            self.grad = torch.empty_like(like)
            self.key = key
        return self.partials, self.sse, self.grad


_LOSS = _LossBuffers()


def mse_and_grad(pred: torch.Tensor, target: torch.Tensor, grad_scale: float):
    """Local sum of squared residuals (device double) and grad_scale * resid,
    one fused pass (d/training.py:114-125)."""
    if pred.shape != target.shape or pred.dtype != target.dtype:
        raise ShapeMismatchError(f"prediction {tuple(pred.shape)} vs target {tuple(target.shape)}")
    lib = _lib.load()
    n = pred.numel()
    partials, sse, grad = _LOSS.get(n, pred)
    g = _geom_for(pred.dtype)
    _lib.check(lib.dfno_mse_grad(ctypes.byref(g), n, _lib.ptr(pred), _lib.ptr(target), float(grad_scale),
                                 _lib.ptr(grad), _lib.ptr(partials), _lib.ptr(sse), _lib.stream_handle()),
               "dfno_mse_grad")
    return sse, grad


def train_step(comm: Communicator, x_local: DenseTensor, y_local: DenseTensor, params: FnoParams,
               state: AdamState, lr: float, config: FnoConfig) -> tuple:
    """Forward, global MSE, backward, Adam update (reference
    d/training.py:96-133).  Returns the updated parameters and the
    rank-identical loss; raises NonFiniteLossError before touching any
    parameter."""
    batch = x_local.shape[0]
    n_total = global_output_count(config, batch)
    cache = ForwardCache()
    pred = fno_forward(comm, x_local, params, config, cache=cache)
    target = y_local.data.to(pred.data.device).contiguous()
    sse, grad = mse_and_grad(pred.data, target, 2.0 / n_total)
    total_sse = comm.allreduce_sum_scalar(float(sse.item()), label="loss")
    loss = total_sse / n_total
    if not math.isfinite(loss):
        raise NonFiniteLossError(f"loss is {loss!r}; aborting the step")
    _, grads = fno_backward(comm, DenseTensor(pred.labels, grad), params, config, cache)
    state.step += 1
    we = adam_update(state, "we", params.we, grads.we, lr)
    wd = adam_update(state, "wd", params.wd, grads.wd, lr)
    blocks = tuple(adam_update(state, f"block{i}", params.blocks[i], grads.blocks[i], lr)
                   for i in range(len(params.blocks)))
    new_params = FnoParams(we, wd, blocks, sharded=params.sharded)
    _assert_replicated(comm, new_params.we, "we")
    _assert_replicated(comm, new_params.wd, "wd")
    return new_params, loss


__all__ = ["AdamState", "adam_update", "global_output_count", "mse_and_grad", "train_step"]
