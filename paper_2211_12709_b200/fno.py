"""Domain-decomposed 4-D Fourier neural operator on B200.

Drop-in for the reference's model layer
(/root/reference/pkg/src/distfno/fno.py): same configuration, parameter,
cache and gradient types, same functions and call signatures
(``fno_forward(comm, x_local, params, config, cache)`` etc.), same
partitioning (x slabs for physical space, ky pencils for the x transform and
the spectral weights) and the same two repartitions per block direction.

What changes is underneath.  Every numpy stage is one sm_100a kernel of
libdfno.so (include/dfno.h), launched on the current CUDA stream:

  encoder / decoder            dfno_mix_fwd / dfno_mix_bwd     (fno.py:286-306, :484-499)
  fft(y,z,t) + truncate        dfno_dft_yzt_fwd -> peer-major XK buffer     (:328-329)
  repartition x -> ky          Communicator.exchange (NCCL all-to-all)      (:330)
  fft(x), truncate, W, pad,    dfno_xspec_fwd (fused)                      (:331-336)
  ifft(x)
  repartition ky -> x          Communicator.exchange                        (:337)
  pad + ifft(y,z,t) + .real    dfno_dft_yzt_inv                             (:338-343)

Activations are never stored: each block keeps only its pre-activation and
the next consumer applies the activation on load (forward) or multiplies by
its derivative on load (backward).  ``ForwardCache.acts`` is therefore
computed on access.
"""

from __future__ import annotations

import ctypes
import enum
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib
from .comm import Communicator
from .errors import DimensionMismatchError, DTypeMismatchError, InfeasiblePartitionError, ShapeMismatchError
from .partition import Partition
from .spectral import ModeSpec, retained_extent
from .tensor import DATA_LABELS, DenseTensor, DimLabel, DType

_INV_SQRT2 = 1.0 / math.sqrt(2.0)
_INV_SQRT2PI = 1.0 / math.sqrt(2.0 * math.pi)


class ActivationKind(str, enum.Enum):
    """Point-wise nonlinearity (reference fno.py:36-55)."""

    RELU = "relu"
    GELU = "gelu"
    IDENTITY = "identity"

    @property
    def code(self) -> int:
        return {ActivationKind.RELU: _lib.ACT_RELU, ActivationKind.GELU: _lib.ACT_GELU,
                ActivationKind.IDENTITY: _lib.ACT_IDENTITY}[self]

    def apply(self, h: torch.Tensor) -> torch.Tensor:
        h = torch.as_tensor(h)
        if self is ActivationKind.RELU:
            return torch.clamp_min(h, 0)
        if self is ActivationKind.GELU:
            return 0.5 * h * (1.0 + torch.erf(h * _INV_SQRT2))
        return h.clone()

    def derivative(self, h: torch.Tensor) -> torch.Tensor:
        h = torch.as_tensor(h)
        if self is ActivationKind.RELU:
            return (h > 0).to(h.dtype)
        if self is ActivationKind.GELU:
            return 0.5 * (1.0 + torch.erf(h * _INV_SQRT2)) + h * _INV_SQRT2PI * torch.exp(-0.5 * h * h)
        return torch.ones_like(h)


@dataclass(frozen=True)
class FnoConfig:
    """Grid, widths, modes, depth, activation, dtype and rank count
    (reference fno.py:62-132; same defaults and feasibility rules)."""

    nx: int
    ny: int
    nz: int
    nt: int
    in_channels: int
    out_channels: int
    hidden_channels: int
    modes: ModeSpec
    num_blocks: int = 4
    activation: ActivationKind = ActivationKind.GELU
    dtype: DType = DType.REAL64
    num_ranks: int = 1

    def __post_init__(self):
        object.__setattr__(self, "activation", ActivationKind(self.activation))
        object.__setattr__(self, "dtype", DType(self.dtype))
        if self.dtype not in (DType.REAL32, DType.REAL64):
            raise DimensionMismatchError("model I/O dtype must be real32 or real64")
        if self.num_blocks < 1:
            raise DimensionMismatchError("need at least one block")
        for name in ("nx", "ny", "nz", "nt", "in_channels", "out_channels", "hidden_channels", "num_ranks"):
            if getattr(self, name) < 1:
                raise DimensionMismatchError(f"{name} must be positive")
        if self.num_ranks > self.nx:
            raise InfeasiblePartitionError(f"{self.num_ranks} ranks cannot partition x of extent {self.nx}")
        if self.num_ranks > self.retained_y:
            raise InfeasiblePartitionError(
                f"{self.num_ranks} ranks cannot partition the retained ky extent {self.retained_y} "
                f"(ny={self.ny}, my={self.modes.count(DimLabel.KY)})"
            )

    @property
    def grid(self) -> tuple:
        return (self.nx, self.ny, self.nz, self.nt)

    @property
    def mode_counts(self) -> tuple:
        return tuple(self.modes.count(k) for k in (DimLabel.KX, DimLabel.KY, DimLabel.KZ, DimLabel.KT))

    @property
    def retained_x(self) -> int:
        return retained_extent(self.nx, self.modes.count(DimLabel.KX))

    @property
    def retained_y(self) -> int:
        return retained_extent(self.ny, self.modes.count(DimLabel.KY))

    @property
    def retained_z(self) -> int:
        return retained_extent(self.nz, self.modes.count(DimLabel.KZ))

    @property
    def retained_t(self) -> int:
        return retained_extent(self.nt, self.modes.count(DimLabel.KT))

    @property
    def retained(self) -> tuple:
        return (self.retained_x, self.retained_y, self.retained_z, self.retained_t)

    @property
    def complex_dtype(self) -> DType:
        return DType.COMPLEX64 if self.dtype == DType.REAL32 else DType.COMPLEX128

    def x_partition(self) -> Partition:
        return Partition.block(DimLabel.X, self.nx, self.num_ranks)

    def ky_partition(self) -> Partition:
        return Partition.block(DimLabel.KY, self.retained_y, self.num_ranks)

    def spectral_weight_shape(self) -> tuple:
        c = self.hidden_channels
        return (c, c, self.retained_x, self.retained_y, self.retained_z, self.retained_t)


_W_LABELS = (DimLabel.C, DimLabel.CO, DimLabel.KX, DimLabel.KY, DimLabel.KZ, DimLabel.KT)
_S_LABELS = (DimLabel.B, DimLabel.C, DimLabel.KX, DimLabel.KY, DimLabel.KZ, DimLabel.KT)


@dataclass(frozen=True)
class FnoParams:
    """Encoder/decoder mixers and per-block spectral weights, global or one
    rank's ky shard (reference fno.py:135-152)."""

    we: DenseTensor
    wd: DenseTensor
    blocks: tuple
    sharded: bool = False

    def named(self) -> dict:
        out = {"we": self.we, "wd": self.wd}
        for i, w in enumerate(self.blocks):
            out[f"block{i}"] = w
        return out

    def to(self, device) -> "FnoParams":
        return FnoParams(self.we.to(device), self.wd.to(device), tuple(w.to(device) for w in self.blocks),
                         self.sharded)


def _default_device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")


def init_params(config: FnoConfig, seed: int, device=None) -> FnoParams:
    """Global parameters, identical for every rank count (reference
    fno.py:155-180): Glorot-uniform mixers, spectral weights with real and
    imaginary parts uniform on [0, 1) scaled by 1/c^2.  The numpy PCG64 stream
    is consumed in the reference's order (we, wd, then re/im per block) and in
    float64 before the cast, so the values are bit-identical to the
    reference's; they are then placed on ``device`` (default: current GPU)."""
    rng = np.random.default_rng(seed)
    c = config.hidden_channels
    real = config.dtype.np_dtype
    cplx = config.complex_dtype.np_dtype
    dev = torch.device(device) if device is not None else _default_device()

    def glorot(fan_in: int, fan_out: int) -> np.ndarray:
        limit = math.sqrt(6.0 / (fan_in + fan_out))
        return rng.uniform(-limit, limit, size=(fan_in, fan_out)).astype(real)

    we = DenseTensor((DimLabel.C, DimLabel.CO), torch.from_numpy(glorot(config.in_channels, c)).to(dev))
    wd = DenseTensor((DimLabel.C, DimLabel.CO), torch.from_numpy(glorot(c, config.out_channels)).to(dev))
    shape = config.spectral_weight_shape()
    scale = 1.0 / (c * c)
    blocks = []
    for _ in range(config.num_blocks):
        re = rng.random(size=shape)
        im = rng.random(size=shape)
        w = (scale * (re + 1j * im)).astype(cplx)
        del re, im
        blocks.append(DenseTensor(_W_LABELS, torch.from_numpy(w).to(dev)))
    return FnoParams(we, wd, tuple(blocks), sharded=False)


def shard_params(params: FnoParams, config: FnoConfig, rank: int) -> FnoParams:
    """This rank's view: spectral weights cut to its ky block
    (reference fno.py:183-194)."""
    if params.sharded:
        raise DimensionMismatchError("parameters are already sharded")
    rng = config.ky_partition().range_of(rank)
    blocks = []
    for w in params.blocks:
        axis = w.axis(DimLabel.KY)
        blocks.append(DenseTensor(w.labels, w.data.narrow(axis, rng.start, len(rng)).contiguous()))
    return FnoParams(params.we, params.wd, tuple(blocks), sharded=True)


def slice_local(x_global: DenseTensor, part: Partition, rank: int) -> DenseTensor:
    """This rank's slab of a global tensor (reference fno.py:512-517)."""
    axis = x_global.axis(part.dim)
    rng = part.range_of(rank)
    return DenseTensor(x_global.labels, x_global.data.narrow(axis, rng.start, len(rng)).contiguous())


# ---------------------------------------------------------------------------
# communication volume (reference fno.py:202-261)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class CommVolume:
    per_repartition_elements: int
    per_block_elements: int
    per_forward_elements: int
    naive_per_repartition_elements: int
    reduction_ratio: float
    bytes_per_element: int

    @property
    def per_repartition_bytes(self) -> int:
        return self.per_repartition_elements * self.bytes_per_element

    @property
    def per_block_bytes(self) -> int:
        return self.per_block_elements * self.bytes_per_element

    @property
    def per_forward_bytes(self) -> int:
        return self.per_forward_elements * self.bytes_per_element


def _off_rank_elements(src: Partition, dst: Partition, per_pair: int) -> int:
    return per_pair * sum(src.extent_of(r) * (dst.global_extent - dst.extent_of(r)) for r in range(src.num_ranks))


def predicted_block_volume(config: FnoConfig, batch_size: int = 1) -> CommVolume:
    """Exact off-rank elements per repartition (summed over ranks), the
    untruncated baseline and the truncation ratio (reference fno.py:234-261)."""
    c = config.hidden_channels
    per_pair = batch_size * c * config.retained_z * config.retained_t
    truncated = _off_rank_elements(config.x_partition(), config.ky_partition(), per_pair)
    naive = _off_rank_elements(config.x_partition(), Partition.block(DimLabel.Y, config.ny, config.num_ranks),
                               batch_size * c * config.nz * config.nt)
    ratio = (config.ny * config.nz * config.nt) / (config.retained_y * config.retained_z * config.retained_t)
    return CommVolume(truncated, 2 * truncated, 2 * config.num_blocks * truncated, naive, ratio,
                      config.complex_dtype.itemsize)


# ---------------------------------------------------------------------------
# caches and gradients
# ---------------------------------------------------------------------------


@dataclass
class BlockCache:
    spec_in: Optional[DenseTensor]          # input of the spectral multiply (ky shard)
    pre_activation: Optional[DenseTensor]   # block output before the outer activation


@dataclass
class ForwardCache:
    """What the backward pass needs (reference fno.py:269-283).  Only
    pre-activations are stored; ``acts`` is derived on access."""

    x_in: Optional[DenseTensor] = None
    enc_w: Optional[DenseTensor] = None
    enc_pre: Optional[DenseTensor] = None
    blocks: list = field(default_factory=list)
    dec_w: Optional[DenseTensor] = None
    dec_pre: Optional[DenseTensor] = None
    activation: ActivationKind = ActivationKind.GELU

    @property
    def acts(self) -> list:
        pres = [self.enc_pre] + [b.pre_activation for b in self.blocks]
        return [DenseTensor(p.labels, self.activation.apply(p.data)) for p in pres if p is not None]


@dataclass(frozen=True)
class FnoGrads:
    """we/wd replicated (reduce-summed, re-broadcast); blocks = this rank's
    ky shard (reference fno.py:388-402)."""

    we: DenseTensor
    wd: DenseTensor
    blocks: tuple

    def named(self) -> dict:
        out = {"we": self.we, "wd": self.wd}
        for i, w in enumerate(self.blocks):
            out[f"block{i}"] = w
        return out


# ---------------------------------------------------------------------------
# execution plan: geometry, split sizes and scratch exchange buffers
# ---------------------------------------------------------------------------


# Channel groups of the pipelined repartitions.  Process-group worlds (NCCL
# between GPUs) overlap each group's all-to-all with the next group's DFT;
# thread worlds share one GPU, where the exchange is a device copy competing
# for the same HBM and the split only costs wave quantisation, so they run
# unsplit unless PIPELINE_GROUPS_THREADED asks for it (the tests do).
PIPELINE_GROUPS = 2
PIPELINE_GROUPS_THREADED = 1


@dataclass
class _Group:
    c0: int
    c1: int
    geom: object
    gp: object
    xk_counts: list
    kx_counts: list
    a: torch.Tensor  # XK send (forward) / XK receive (return)
    b: torch.Tensor  # KX receive
    c: torch.Tensor  # KX send
    spec_off: int    # first element of the group's channels in a (b = 1) spectrum


class _Plan:
    def __init__(self, config: FnoConfig, rank: int, world: int, batch: int, device: torch.device,
                 threaded: bool = False):
        if world != config.num_ranks:
            raise ShapeMismatchError(f"config.num_ranks={config.num_ranks} but the communicator has {world} ranks")
        self.config = config
        self.rank = rank
        self.world = world
        self.batch = batch
        self.device = device
        xp, kp = config.x_partition(), config.ky_partition()
        self.xpart, self.kypart = xp, kp
        self.xl = xp.extent_of(rank)
        self.kyl = kp.extent_of(rank)
        self.lib = _lib.load()
        dt = _lib.F32 if config.dtype == DType.REAL32 else _lib.F64
        self.geom = _lib.make_geom(
            batch=batch, c_in=config.in_channels, c=config.hidden_channels, c_out=config.out_channels,
            grid=config.grid, modes=config.mode_counts, retained=config.retained, nranks=world, rank=rank,
            dtype=dt, act=config.activation.code, x_starts=xp.starts(), ky_starts=kp.starts(),
        )
        _lib.check(self.lib.dfno_geom_validate(ctypes.byref(self.geom)), "geometry")
        self.gp = ctypes.byref(self.geom)
        self.npts = self.xl * config.ny * config.nz * config.nt
        self.n_yzt = config.ny * config.nz * config.nt
        c, rz, rt = config.hidden_channels, config.retained_z, config.retained_t
        rx = config.retained_x
        self.real = config.dtype.torch_dtype
        self.cplx = config.complex_dtype.torch_dtype
        self.xk_elems = batch * c * self.xl * config.retained_y * rz * rt
        self.kx_elems = batch * c * config.nx * self.kyl * rz * rt
        self.spec_shape = (batch, c, rx, self.kyl, rz, rt)
        self.w_shape = (c, c, rx, self.kyl, rz, rt)
        # x -> ky: send chunk p = [b][c][xl][ky_p][rz][rt], recv chunk p = [b][c][x_p][kyl][rz][rt]
        self.xk_counts = [batch * c * self.xl * kp.extent_of(p) * rz * rt for p in range(world)]
        self.kx_counts = [batch * c * xp.extent_of(p) * self.kyl * rz * rt for p in range(world)]
        # scratch (reused across calls; consumed before the next call on the same stream)
        n = max(self.xk_elems, self.kx_elems)
        self.buf_a = torch.empty(self.xk_elems, dtype=self.cplx, device=device)   # XK send / XK recv
        self.buf_b = torch.empty(self.kx_elems, dtype=self.cplx, device=device)   # KX recv
        self.buf_c = torch.empty(self.kx_elems, dtype=self.cplx, device=device)   # KX send
        del n
        ws = ctypes.c_int64()
        _lib.check(self.lib.dfno_xspec_workspace(self.gp, ctypes.byref(ws)), "xspec workspace")
        self.xspec_work = torch.empty(max(1, ws.value), dtype=torch.uint8, device=device)
        self.partials = {}
        self.groups = self._channel_groups(xp, kp, rz, rt, PIPELINE_GROUPS_THREADED if threaded else PIPELINE_GROUPS)
        self.comm_stream = torch.cuda.Stream(device=device) if self.groups else None

    def _channel_groups(self, xp, kp, rz, rt, ngroups: int) -> list:
        """Channel groups of the pipelined exchanges (world > 1, b = 1, fp32):
        each group has its own geometry (c = group size) and its own
        peer-major XK / KX regions carved from the plan's buffers, so group
        k's all-to-all runs on the comm stream while group k + 1's DFT runs on
        the compute stream."""
        cfg, c = self.config, self.config.hidden_channels
        ng = min(ngroups, c)
        if self.world == 1 or self.batch != 1 or cfg.dtype != DType.REAL32 or ng < 2:
            return []
        bounds = [c * k // ng for k in range(ng + 1)]
        groups, xo, ko = [], 0, 0
        for k in range(ng):
            c0, c1 = bounds[k], bounds[k + 1]
            n = c1 - c0
            geom = _lib.make_geom(
                batch=1, c_in=n, c=n, c_out=n, grid=cfg.grid, modes=cfg.mode_counts, retained=cfg.retained,
                nranks=self.world, rank=self.rank, dtype=_lib.F32, act=cfg.activation.code,
                x_starts=xp.starts(), ky_starts=kp.starts())
            _lib.check(self.lib.dfno_geom_validate(ctypes.byref(geom)), "group geometry")
            xk = n * self.xl * cfg.retained_y * rz * rt
            kx = n * cfg.nx * self.kyl * rz * rt
            groups.append(_Group(
                c0=c0, c1=c1, geom=geom, gp=ctypes.byref(geom),
                xk_counts=[n * self.xl * kp.extent_of(p) * rz * rt for p in range(self.world)],
                kx_counts=[n * xp.extent_of(p) * self.kyl * rz * rt for p in range(self.world)],
                a=self.buf_a[xo:xo + xk], b=self.buf_b[ko:ko + kx], c=self.buf_c[ko:ko + kx],
                spec_off=c0 * cfg.retained_x * self.kyl * rz * rt))
            xo, ko = xo + xk, ko + kx
        return groups

    # -- shapes ----------------------------------------------------------
    def act_shape(self, ch: int) -> tuple:
        cfg = self.config
        return (self.batch, ch, self.xl, cfg.ny, cfg.nz, cfg.nt)

    def empty_act(self, ch: int) -> torch.Tensor:
        return torch.empty(self.act_shape(ch), dtype=self.real, device=self.device)

    def partial_buf(self, cin: int, cout: int):
        key = (cin, cout)
        if key not in self.partials:
            n = ctypes.c_int64()
            k = ctypes.c_int()
            _lib.check(self.lib.dfno_mix_bwd_partials(self.gp, self.npts, cin, cout, ctypes.byref(n), ctypes.byref(k)),
                       "mix_bwd_partials")
            self.partials[key] = (torch.empty(n.value, dtype=self.real, device=self.device), k.value)
        return self.partials[key]

    # -- kernels -----------------------------------------------------------
    def mix_fwd(self, cin, cout, src, src_act, w, pre, post, tag="mix_fwd"):
        _launch(tag, lambda: _lib.check(self.lib.dfno_mix_fwd(
            self.gp, self.npts, cin, cout, _lib.ptr(src), int(src_act), _lib.ptr(w), _lib.ptr(pre), _lib.ptr(post),
            _lib.stream_handle()), "dfno_mix_fwd"))

    def mix_bwd(self, cin, cout, gout, pre, src, src_act, w, gin, tag="mix_bwd", fuse_src_dact=False):
        """Mixer backward; with ``fuse_src_dact`` (src_act must be true) the
        library is first asked for gin * act'(src) in the same pass (status
        DFNO_ERR_UNSUPPORTED outside the tcgen05 envelope).  Returns (gw, fused)."""
        buf, nparts = self.partial_buf(cin, cout)
        fused = [False]

        def run():
            args = (self.gp, self.npts, cin, cout, _lib.ptr(gout), _lib.ptr(pre), _lib.ptr(src))
            tail = (_lib.ptr(w), _lib.ptr(gin), _lib.ptr(buf), _lib.stream_handle())
            if fuse_src_dact:
                rc = self.lib.dfno_mix_bwd(*args, 2, *tail)
                if rc == _DFNO_ERR_UNSUPPORTED:
                    rc = self.lib.dfno_mix_bwd(*args, 1, *tail)
                else:
                    fused[0] = rc == 0
            else:
                rc = self.lib.dfno_mix_bwd(*args, int(src_act), *tail)
            _lib.check(rc, "dfno_mix_bwd")

        _launch(f"mix_bwd.{tag}", run)
        gw = torch.empty((cin, cout), dtype=self.real, device=self.device)
        _launch(f"reduce.{tag}", lambda: _lib.check(self.lib.dfno_reduce_partials(
            self.gp, nparts, cin * cout, _lib.ptr(buf), _lib.ptr(gw), _lib.stream_handle()), "dfno_reduce_partials"))
        return (gw, fused[0]) if fuse_src_dact else gw

    def yzt_fwd(self, src, pre, mode, scale, out, tag="yzt_fwd", gp=None):
        _launch(tag, lambda: _lib.check(self.lib.dfno_dft_yzt_fwd(
            gp or self.gp, _lib.ptr(src), _lib.ptr(pre), mode, float(scale), _lib.ptr(out), _lib.stream_handle()),
            "dfno_dft_yzt_fwd"))

    def yzt_inv(self, xk_in, scale, out, tag="yzt_inv", gp=None):
        _launch(tag, lambda: _lib.check(self.lib.dfno_dft_yzt_inv(
            gp or self.gp, _lib.ptr(xk_in), float(scale), _lib.ptr(out), _lib.stream_handle()), "dfno_dft_yzt_inv"))

    # x-spectral stage by parts (pipelined blocks)
    def xdft(self, gp, kx_in, scale, X, tag):
        _launch(tag, lambda: _lib.check(self.lib.dfno_xdft(
            gp, _lib.ptr(kx_in), float(scale), _lib.ptr(X), _lib.stream_handle()), "dfno_xdft"))

    def xidft(self, gp, Y, scale, kx_out, tag):
        _launch(tag, lambda: _lib.check(self.lib.dfno_xidft(
            gp, _lib.ptr(Y), float(scale), _lib.ptr(kx_out), _lib.stream_handle()), "dfno_xidft"))

    def xmix_fwd(self, X, w, Y):
        _launch("xmix_fwd", lambda: _lib.check(self.lib.dfno_xmix_fwd(
            self.gp, _lib.ptr(X), _lib.ptr(w), _lib.ptr(Y), _lib.stream_handle()), "dfno_xmix_fwd"))

    def xmix_bwd(self, spec, D, w, gw, dX):
        _launch("xmix_bwd", lambda: _lib.check(self.lib.dfno_xmix_bwd(
            self.gp, _lib.ptr(spec), _lib.ptr(D), _lib.ptr(w), _lib.ptr(gw), _lib.ptr(dX), _lib.stream_handle()),
            "dfno_xmix_bwd"))

    def spectra(self) -> tuple:
        """The two spectrum-sized halves of the x-spectral workspace (complex)."""
        n = self.batch * self.config.hidden_channels * self.config.retained_x * self.kyl * \
            self.config.retained_z * self.config.retained_t
        flat = self.xspec_work.view(self.cplx)
        return flat[:n].view(self.spec_shape), flat[n:2 * n].view(self.spec_shape)

    def exchange_groups(self, comm: Communicator, send_of, recv_of, fwd: bool, label: str, after_each=None):
        """Chunked repartition: for each channel group, after ``after_each(k)``
        has enqueued its producer on the compute stream, the group's
        all-to-all runs on the comm stream; returns one event per group that
        the consumer of that group waits on.  Accounted as one repartition."""
        S, C = torch.cuda.current_stream(), self.comm_stream
        events, off_rank = [], 0
        for k, grp in enumerate(self.groups):
            if after_each is not None:
                after_each(k, grp)
            ready = torch.cuda.Event()
            ready.record(S)
            C.wait_event(ready)
            with torch.cuda.stream(C):
                sc, rc = (grp.xk_counts, grp.kx_counts) if fwd else (grp.kx_counts, grp.xk_counts)
                off_rank += comm.exchange(send_of(grp), recv_of(grp), sc, rc, f"{label}.g{k}", record=False)
                done = torch.cuda.Event()
                done.record(C)
            events.append(done)
        comm.record_repartition(off_rank, self.buf_a.element_size())
        return events

    def xspec_fwd(self, kx_in, w, spec, kx_out):
        _launch("xspec_fwd", lambda: _lib.check(self.lib.dfno_xspec_fwd_ws(
            self.gp, _lib.ptr(kx_in), _lib.ptr(w), _lib.ptr(spec), _lib.ptr(kx_out), _lib.ptr(self.xspec_work),
            _lib.stream_handle()), "dfno_xspec_fwd_ws"))

    def xspec_bwd(self, kx_in, spec, w, gw, kx_out):
        _launch("xspec_bwd", lambda: _lib.check(self.lib.dfno_xspec_bwd_ws(
            self.gp, _lib.ptr(kx_in), _lib.ptr(spec), _lib.ptr(w), _lib.ptr(gw), _lib.ptr(kx_out),
            _lib.ptr(self.xspec_work), _lib.stream_handle()), "dfno_xspec_bwd_ws"))

    # -- exchanges (reference fno.py:330, :337, :449, :458) ---------------
    def x_to_ky(self, comm: Communicator, label: str) -> torch.Tensor:
        if self.world == 1:
            comm.exchange(self.buf_a, self.buf_a, self.xk_counts, self.kx_counts, label)
            return self.buf_a
        comm.exchange(self.buf_a, self.buf_b, self.xk_counts, self.kx_counts, label)
        return self.buf_b

    def ky_to_x(self, comm: Communicator, kx_out: torch.Tensor, label: str) -> torch.Tensor:
        if self.world == 1:
            comm.exchange(kx_out, kx_out, self.kx_counts, self.xk_counts, label)
            return kx_out
        comm.exchange(kx_out, self.buf_a, self.kx_counts, self.xk_counts, label)
        return self.buf_a


_TIMER = None


def set_kernel_timer(timer) -> None:
    """Install ``timer(name, launch_fn)`` around every libdfno launch (used by
    bench.py to time kernels with CUDA events); None removes it."""
    global _TIMER
    _TIMER = timer


_DFNO_ERR_UNSUPPORTED = -7  # include/dfno.h


def _launch(name: str, fn) -> None:
    if _TIMER is None:
        fn()
    else:
        _TIMER(name, fn)


def _plan(config: FnoConfig, comm: Communicator, batch: int) -> _Plan:
    """The rank's plan (geometry, exchange buffers, xspec workspace), cached on
    the Communicator itself so its device buffers are released together with
    the rank's communicator (no process-wide cache that outlives rank threads)."""
    if not _lib.available():
        raise _lib.ExtensionMissingError("libdfno.so and a CUDA device are required (no CPU fallback)")
    check_envelope(config)
    device = comm.device if comm.device.type == "cuda" else _default_device()
    key = (config, batch, str(device), PIPELINE_GROUPS, PIPELINE_GROUPS_THREADED)
    plans = comm.__dict__.setdefault("_dfno_plans", {})
    plan = plans.get(key)
    if plan is None:
        plan = _Plan(config, comm.rank, comm.world_size, batch, device, threaded=comm.threaded)
        plans[key] = plan
    return plan


def clear_plans(comm: Optional[Communicator] = None) -> None:
    """Drop the cached plans (and their scratch buffers) of ``comm``; plans
    also go away with their communicator."""
    if comm is not None:
        comm.__dict__.pop("_dfno_plans", None)


MAX_CHANNELS_F64 = 32  # the fused fp64 x-spectral kernel keeps a channel row per thread


def check_envelope(config: FnoConfig) -> None:
    """Reject, before any kernel runs, configurations outside the kernels'
    envelope (the reference itself accepts any width): fp32 takes any channel
    width (wider mixers run in 32-channel blocks); the real64 path is limited to
    MAX_CHANNELS_F64 channels."""
    if config.dtype != DType.REAL64:
        return
    widths = {"in_channels": config.in_channels, "hidden_channels": config.hidden_channels,
              "out_channels": config.out_channels}
    wide = {k: v for k, v in widths.items() if v > MAX_CHANNELS_F64}
    if wide:
        raise DimensionMismatchError(
            f"channel widths {wide} exceed the real64 kernels' limit of {MAX_CHANNELS_F64} channels "
            f"(real32 takes any width)")


def _on_device(t: DenseTensor, plan: _Plan, dtype: torch.dtype, what: str) -> torch.Tensor:
    data = t.data
    if data.dtype != dtype:
        raise DTypeMismatchError(f"{what}: dtype {data.dtype} but the model computes in {dtype}")
    if data.device != plan.device:
        data = data.to(plan.device, non_blocking=True)
    return data.contiguous()


def _check_act_input(x: DenseTensor, plan: _Plan, ch: int, what: str) -> None:
    want = plan.act_shape(ch)
    if tuple(x.shape) != want:
        if len(x.shape) == 6 and x.shape[1] != ch:
            raise DimensionMismatchError(f"{what}: channel extent {x.shape[1]} does not match {ch}")
        raise ShapeMismatchError(f"{what}: local slab shape {tuple(x.shape)}, expected {want}")


def _check_weight(w: DenseTensor, plan: _Plan, what: str) -> torch.Tensor:
    if tuple(w.shape) != plan.w_shape:
        raise DimensionMismatchError(f"{what}: weight shard shape {tuple(w.shape)}, expected {plan.w_shape}")
    return _on_device(w, plan, plan.cplx, what)


def _wrap(data: torch.Tensor) -> DenseTensor:
    return DenseTensor(DATA_LABELS, data)


# ---------------------------------------------------------------------------
# forward (reference fno.py:286-380)
# ---------------------------------------------------------------------------


def _mix_forward(comm, plan: _Plan, src: torch.Tensor, src_act: bool, w: DenseTensor, cin: int, cout: int,
                 label: str, want_post: bool):
    w_used = comm.broadcast(w, root=0, label=label)
    wt = _on_device(w_used, plan, plan.real, f"{label} weight")
    if tuple(wt.shape) != (cin, cout):
        raise DimensionMismatchError(f"{label} weight shape {tuple(wt.shape)}, expected {(cin, cout)}")
    pre = plan.empty_act(cout)
    post = plan.empty_act(cout) if want_post else None
    plan.mix_fwd(cin, cout, src, src_act, wt, pre, post, tag="mix_fwd.enc" if label == "encoder" else "mix_fwd.dec")
    return pre, post, w_used


def encoder_forward(comm: Communicator, x_local: DenseTensor, we: DenseTensor,
                    activation: ActivationKind = ActivationKind.GELU) -> DenseTensor:
    """Broadcast the encoder weights and mix channels rank-locally
    (reference fno.py:292-298)."""
    return _mixer_api(comm, x_local, we, activation, "encoder")


def decoder_forward(comm: Communicator, x_local: DenseTensor, wd: DenseTensor,
                    activation: ActivationKind = ActivationKind.GELU) -> DenseTensor:
    """Reference fno.py:301-306."""
    return _mixer_api(comm, x_local, wd, activation, "decoder")


def _mixer_api(comm, x_local, w, activation, label):
    activation = ActivationKind(activation)
    dtype = DType.REAL32 if x_local.dtype == DType.REAL32 else DType.REAL64
    if w.dtype != x_local.dtype:
        raise DTypeMismatchError(f"mixed precision is disallowed: {x_local.dtype.value} vs {w.dtype.value}")
    b, cin = x_local.shape[0], x_local.shape[1]
    cout = w.shape[1]
    if w.shape[0] != cin:
        raise DimensionMismatchError(f"channel extent {cin} does not match weight rows {w.shape[0]}")
    npts = int(np.prod(x_local.shape[2:]))
    lib = _lib.load()
    if not _lib.available():
        raise _lib.ExtensionMissingError("libdfno.so and a CUDA device are required (no CPU fallback)")
    dev = comm.device if comm.device.type == "cuda" else _default_device()
    w_used = comm.broadcast(w, root=0, label=label)
    x = x_local.data.to(dev).contiguous()
    wt = w_used.data.to(dev).contiguous()
    g = _lib.make_geom(batch=b, c_in=cin, c=max(cin, cout), c_out=cout, grid=(1, 1, 1, 1), modes=(1, 1, 1, 1),
                       retained=(1, 1, 1, 1), nranks=1, rank=0,
                       dtype=_lib.F32 if dtype == DType.REAL32 else _lib.F64, act=activation.code,
                       x_starts=(0, 1), ky_starts=(0, 1))
    pre = torch.empty((b, cout) + tuple(x_local.shape[2:]), dtype=x.dtype, device=dev)
    post = torch.empty_like(pre)
    _lib.check(lib.dfno_mix_fwd(ctypes.byref(g), npts, cin, cout, _lib.ptr(x), 0, _lib.ptr(wt), _lib.ptr(pre),
                                _lib.ptr(post), _lib.stream_handle()), "dfno_mix_fwd")
    return DenseTensor(x_local.labels, post)


def _block_forward_pipelined(comm, plan: _Plan, src: torch.Tensor, mode: int, w: torch.Tensor, label: str,
                             want_spec: bool):
    """_block_forward with the two repartitions chunked by channel group:

        compute stream   yzt(g0) yzt(g1)           xdft(g0) xdft(g1) xmix xidft(g0) xidft(g1)            yzt^-1(g0) yzt^-1(g1)
        comm stream              a2a(g0)  a2a(g1)                                   a2a'(g0)  a2a'(g1)

    group k's all-to-all overlaps group k+1's DFT on either side of the
    x-spectral stage (the contraction itself needs every channel)."""
    S = torch.cuda.current_stream()
    X0, Y = plan.spectra()
    spec = torch.empty(plan.spec_shape, dtype=plan.cplx, device=plan.device) if want_spec else X0
    x_of = lambda t, grp: t.view(-1)[grp.spec_off:]  # noqa: E731 - b = 1: channel slice of a spectrum
    ev = plan.exchange_groups(
        comm, lambda grp: grp.a, lambda grp: grp.b, True, f"{label}.fwd.x->ky",
        after_each=lambda k, grp: plan.yzt_fwd(src[:, grp.c0:grp.c1], None, mode, 1.0, grp.a, tag="yzt_fwd.fwd",
                                               gp=grp.gp))
    for grp, e in zip(plan.groups, ev):
        S.wait_event(e)
        plan.xdft(grp.gp, grp.b, 1.0, x_of(spec, grp), "xdft.fwd")  # fft_x unnormalised (d/spectral.py:36)
    plan.xmix_fwd(spec, w, Y)
    ev = plan.exchange_groups(
        comm, lambda grp: grp.c, lambda grp: grp.a, False, f"{label}.fwd.ky->x",
        after_each=lambda k, grp: plan.xidft(grp.gp, x_of(Y, grp), 1.0 / plan.config.nx, grp.c, "xidft.fwd"))
    pre = plan.empty_act(plan.config.hidden_channels)
    for grp, e in zip(plan.groups, ev):
        S.wait_event(e)
        plan.yzt_inv(grp.a, 1.0 / plan.n_yzt, pre[:, grp.c0:grp.c1], tag="yzt_inv.fwd", gp=grp.gp)
    return pre, (spec if want_spec else None)


def _block_forward(comm, plan: _Plan, src: torch.Tensor, mode: int, w: torch.Tensor, label: str,
                   want_spec: bool):
    """fft_yzt -> truncate -> R(x->ky) -> fft_x -> truncate -> W -> pad ->
    ifft_x -> R(ky->x) -> pad -> ifft_yzt -> real  (reference fno.py:309-347)."""
    if plan.groups:
        return _block_forward_pipelined(comm, plan, src, mode, w, label, want_spec)
    plan.yzt_fwd(src, None, mode, 1.0, plan.buf_a, tag="yzt_fwd.fwd")
    kx_in = plan.x_to_ky(comm, f"{label}.fwd.x->ky")
    spec = torch.empty(plan.spec_shape, dtype=plan.cplx, device=plan.device) if want_spec else None
    plan.xspec_fwd(kx_in, w, spec, plan.buf_c)
    xk_in = plan.ky_to_x(comm, plan.buf_c, f"{label}.fwd.ky->x")
    pre = plan.empty_act(plan.config.hidden_channels)
    plan.yzt_inv(xk_in, 1.0 / plan.n_yzt, pre, tag="yzt_inv.fwd")
    return pre, spec


def fno_block_forward(comm: Communicator, x_local: DenseTensor, w_shard: DenseTensor, config: FnoConfig,
                      label: str = "block", cache: Optional[BlockCache] = None) -> DenseTensor:
    """One distributed spectral block without the outer activation
    (reference fno.py:309-347).  ``x_local`` is the block input (already
    activated), exactly as in the reference."""
    plan = _plan(config, comm, x_local.shape[0])
    _check_act_input(x_local, plan, config.hidden_channels, "block input")
    x = _on_device(x_local, plan, plan.real, "block input")
    w = _check_weight(w_shard, plan, "spectral weight")
    pre, spec = _block_forward(comm, plan, x, _lib.SRC_RAW, w, label, cache is not None)
    out = _wrap(pre)
    if cache is not None:
        cache.spec_in = DenseTensor(_S_LABELS, spec)
        cache.pre_activation = out
    return out


def fno_forward(comm: Communicator, x_local: DenseTensor, params: FnoParams, config: FnoConfig,
                cache: Optional[ForwardCache] = None) -> DenseTensor:
    """Full distributed forward on this rank's x slab (reference fno.py:350-380):
    y = act(dec(act(block_L(... act(block_1(act(enc(x))))))))."""
    if not params.sharded and config.num_ranks > 1:
        raise DimensionMismatchError("fno_forward needs this rank's sharded parameters (shard_params)")
    plan = _plan(config, comm, x_local.shape[0])
    _check_act_input(x_local, plan, config.in_channels, "input")
    x = _on_device(x_local, plan, plan.real, "input")
    c = config.hidden_channels
    want = cache is not None
    enc_pre, _, enc_w = _mix_forward(comm, plan, x, False, params.we, config.in_channels, c, "encoder", False)
    if want:
        cache.x_in = _wrap(x)
        cache.enc_w = enc_w
        cache.enc_pre = _wrap(enc_pre)
        cache.blocks = []
        cache.activation = config.activation
    src = enc_pre
    for i, w_shard in enumerate(params.blocks):
        w = _check_weight(w_shard, plan, f"block{i} weight")
        pre, spec = _block_forward(comm, plan, src, _lib.SRC_ACT, w, f"block{i}", want)
        if want:
            cache.blocks.append(BlockCache(DenseTensor(_S_LABELS, spec), _wrap(pre)))
        src = pre
    dec_pre, y, dec_w = _mix_forward(comm, plan, src, True, params.wd, c, config.out_channels, "decoder", True)
    if want:
        cache.dec_pre = _wrap(dec_pre)
        cache.dec_w = dec_w
    return _wrap(y)


# ---------------------------------------------------------------------------
# backward (reference fno.py:405-509)
# ---------------------------------------------------------------------------


def _block_backward(comm, plan: _Plan, g: torch.Tensor, pre: Optional[torch.Tensor], mode: int, w: torch.Tensor,
                    spec: torch.Tensor, label: str):
    """Adjoint chain (reference fno.py:445-464): fft_yzt/N_yzt -> truncate ->
    R(x->ky) -> fft_x/Nx -> truncate -> gW, dX -> pad -> ifft_x*Nx -> R(ky->x)
    -> pad -> ifft_yzt*N_yzt -> real."""
    tag = "yzt_fwd.bwd" if mode == _lib.SRC_GRAD else "yzt_fwd.bwd_raw"
    if plan.groups:  # chunked exchanges, as _block_forward_pipelined
        S = torch.cuda.current_stream()
        D, dX = plan.spectra()
        x_of = lambda t, grp: t.view(-1)[grp.spec_off:]  # noqa: E731
        ev = plan.exchange_groups(
            comm, lambda grp: grp.a, lambda grp: grp.b, True, f"{label}.bwd.x->ky",
            after_each=lambda k, grp: plan.yzt_fwd(
                g[:, grp.c0:grp.c1], None if pre is None else pre[:, grp.c0:grp.c1], mode, 1.0 / plan.n_yzt, grp.a,
                tag=tag, gp=grp.gp))
        for grp, e in zip(plan.groups, ev):
            S.wait_event(e)
            plan.xdft(grp.gp, grp.b, 1.0 / plan.config.nx, x_of(D, grp), "xdft.bwd")  # fft_x / Nx (d/fno.py:450-452)
        gw = torch.empty(plan.w_shape, dtype=plan.cplx, device=plan.device)
        plan.xmix_bwd(spec, D, w, gw, dX)
        ev = plan.exchange_groups(
            comm, lambda grp: grp.c, lambda grp: grp.a, False, f"{label}.bwd.ky->x",
            after_each=lambda k, grp: plan.xidft(grp.gp, x_of(dX, grp), 1.0, grp.c, "xidft.bwd"))
        gin = plan.empty_act(plan.config.hidden_channels)
        for grp, e in zip(plan.groups, ev):
            S.wait_event(e)
            plan.yzt_inv(grp.a, 1.0, gin[:, grp.c0:grp.c1], tag="yzt_inv.bwd", gp=grp.gp)
        return gin, gw
    plan.yzt_fwd(g, pre, mode, 1.0 / plan.n_yzt, plan.buf_a, tag=tag)
    kx_in = plan.x_to_ky(comm, f"{label}.bwd.x->ky")
    gw = torch.empty(plan.w_shape, dtype=plan.cplx, device=plan.device)
    plan.xspec_bwd(kx_in, spec, w, gw, plan.buf_c)
    xk_in = plan.ky_to_x(comm, plan.buf_c, f"{label}.bwd.ky->x")
    gin = plan.empty_act(plan.config.hidden_channels)
    plan.yzt_inv(xk_in, 1.0, gin, tag="yzt_inv.bwd")
    return gin, gw


def fno_block_backward(comm: Communicator, g: DenseTensor, w_shard: DenseTensor, spec_in: DenseTensor,
                       config: FnoConfig, label: str = "block") -> tuple:
    """Gradient w.r.t. the block input and this rank's weight shard, given the
    gradient w.r.t. the block output (reference fno.py:426-465)."""
    plan = _plan(config, comm, g.shape[0])
    _check_act_input(g, plan, config.hidden_channels, "block gradient")
    gd = _on_device(g, plan, plan.real, "block gradient")
    w = _check_weight(w_shard, plan, "spectral weight")
    s = _on_device(spec_in, plan, plan.cplx, "spec_in")
    gin, gw = _block_backward(comm, plan, gd, None, _lib.SRC_RAW, w, s, label)
    return _wrap(gin), DenseTensor(w_shard.labels, gw)


def fno_backward(comm: Communicator, g_local: DenseTensor, params: FnoParams, config: FnoConfig,
                 cache: ForwardCache) -> tuple:
    """Reverse-mode gradients from the upstream output gradient
    (reference fno.py:468-509).  Spectral-weight gradients stay rank-local;
    mixer gradients are reduce-summed to rank 0 in rank order and
    re-broadcast, so replicas are bit-identical."""
    plan = _plan(config, comm, g_local.shape[0])
    _check_act_input(g_local, plan, config.out_channels, "output gradient")
    g = _on_device(g_local, plan, plan.real, "output gradient")
    c, L = config.hidden_channels, len(params.blocks)
    if len(cache.blocks) != L:
        raise ShapeMismatchError("forward cache does not match the parameter set")
    dec_w = _on_device(cache.dec_w, plan, plan.real, "decoder weight")
    last_pre = cache.blocks[-1].pre_activation.data
    g_a = plan.empty_act(c)
    # the decoder's input is act(last block output): when the library fuses
    # act'(last_pre) into the decoder's input gradient, the last block's
    # backward DFT reads one stream (RAW) instead of g and pre (GRAD)
    gwd_local, fused = plan.mix_bwd(c, config.out_channels, g, cache.dec_pre.data, last_pre, True, dec_w, g_a,
                                    tag="dec", fuse_src_dact=True)

    block_grads = [None] * L
    for i in reversed(range(L)):
        bc = cache.blocks[i]
        w = _check_weight(params.blocks[i], plan, f"block{i} weight")
        raw = fused and i == L - 1
        g_a, gw = _block_backward(comm, plan, g_a, None if raw else bc.pre_activation.data,
                                  _lib.SRC_RAW if raw else _lib.SRC_GRAD, w, bc.spec_in.data, f"block{i}")
        block_grads[i] = DenseTensor(params.blocks[i].labels, gw)

    enc_w = _on_device(cache.enc_w, plan, plan.real, "encoder weight")
    gx = plan.empty_act(config.in_channels)
    gwe_local = plan.mix_bwd(config.in_channels, c, g_a, cache.enc_pre.data, cache.x_in.data, False, enc_w, gx,
                             tag="enc")

    labels = (DimLabel.C, DimLabel.CO)
    # reduce_sum + broadcast of both mixer gradients (d/fno.py:501-508) as one
    # all-gather with a rank-ordered device sum: no host synchronisation
    gwe_t, gwd_t = comm.allreduce_sum_many([gwe_local, gwd_local], ["bwd.we", "bwd.wd"])
    return _wrap(gx), FnoGrads(DenseTensor(labels, gwe_t), DenseTensor(labels, gwd_t), tuple(block_grads))
