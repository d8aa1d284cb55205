"""Labelled dense tensors over torch storage.

Mirrors the reference's ``DenseTensor`` / ``DimLabel`` / ``DType``
(/root/reference/pkg/src/distfno/tensor.py:27-200): an ordered tuple of unique
dimension labels over a contiguous row-major array, with spectral labels only
on complex data.  The storage is a ``torch.Tensor`` so the hot path keeps it
resident in HBM; numpy arrays are accepted at construction (host data) and
``numpy()`` copies back.  Like the reference, tensors are treated as
immutable: every hot-path op allocates its result.
"""

from __future__ import annotations

import enum
from typing import Iterable

import numpy as np
import torch

from .errors import DimensionMismatchError, DTypeMismatchError, UnknownLabelError


class DimLabel(str, enum.Enum):
    """Dimension labels (reference tensor.py:27-43)."""

    B = "b"
    C = "c"
    X = "x"
    Y = "y"
    Z = "z"
    T = "t"
    KX = "kx"
    KY = "ky"
    KZ = "kz"
    KT = "kt"
    CO = "co"

    def __str__(self) -> str:  # pragma: no cover - cosmetic
        return self.value


SPECTRAL_LABELS = frozenset({DimLabel.KX, DimLabel.KY, DimLabel.KZ, DimLabel.KT})
SPATIAL_TO_SPECTRAL = {
    DimLabel.X: DimLabel.KX,
    DimLabel.Y: DimLabel.KY,
    DimLabel.Z: DimLabel.KZ,
    DimLabel.T: DimLabel.KT,
}
SPECTRAL_TO_SPATIAL = {v: k for k, v in SPATIAL_TO_SPECTRAL.items()}
DATA_LABELS = (DimLabel.B, DimLabel.C, DimLabel.X, DimLabel.Y, DimLabel.Z, DimLabel.T)


def as_label(label: "DimLabel | str") -> DimLabel:
    try:
        return DimLabel(label)
    except ValueError:
        raise UnknownLabelError(f"unknown dimension label {label!r}") from None


class DType(str, enum.Enum):
    """Element types (reference tensor.py:78-94)."""

    REAL32 = "real32"
    REAL64 = "real64"
    COMPLEX64 = "complex64"
    COMPLEX128 = "complex128"

    @property
    def torch_dtype(self) -> torch.dtype:
        return _TORCH[self]

    @property
    def np_dtype(self) -> np.dtype:
        return np.dtype(_NP[self])

    @property
    def is_complex(self) -> bool:
        return self in (DType.COMPLEX64, DType.COMPLEX128)

    @property
    def itemsize(self) -> int:
        return self.np_dtype.itemsize

    @property
    def complex_of(self) -> "DType":
        return {DType.REAL32: DType.COMPLEX64, DType.REAL64: DType.COMPLEX128}.get(self, self)

    @property
    def real_of(self) -> "DType":
        return {DType.COMPLEX64: DType.REAL32, DType.COMPLEX128: DType.REAL64}.get(self, self)


_TORCH = {
    DType.REAL32: torch.float32,
    DType.REAL64: torch.float64,
    DType.COMPLEX64: torch.complex64,
    DType.COMPLEX128: torch.complex128,
}
_NP = {DType.REAL32: "<f4", DType.REAL64: "<f8", DType.COMPLEX64: "<c8", DType.COMPLEX128: "<c16"}
_FROM_TORCH = {v: k for k, v in _TORCH.items()}


def dtype_of(data) -> DType:
    if isinstance(data, torch.Tensor):
        if data.dtype not in _FROM_TORCH:
            raise DTypeMismatchError(f"unsupported torch dtype {data.dtype}")
        return _FROM_TORCH[data.dtype]
    arr = np.asarray(data)
    for dt in DType:
        if arr.dtype == dt.np_dtype:
            return dt
    raise DTypeMismatchError(f"unsupported numpy dtype {arr.dtype}")


class DenseTensor:
    """N-d array with one label per dimension (reference tensor.py:120-190).

    ``data`` is a contiguous ``torch.Tensor`` (host or device).  numpy input
    is copied into a host tensor.
    """

    __slots__ = ("labels", "data")

    def __init__(self, labels: Iterable["DimLabel | str"], data):
        labels = tuple(as_label(l) for l in labels)
        if len(set(labels)) != len(labels):
            raise DimensionMismatchError(f"duplicate labels in {labels}")
        if isinstance(data, torch.Tensor):
            t = data if data.is_contiguous() else data.contiguous()
        else:
            arr = np.ascontiguousarray(data)
            dtype_of(arr)
            t = torch.from_numpy(arr.copy())  # own the bytes, like the reference (tensor.py:145-148)
        dt = dtype_of(t)
        if t.dim() != len(labels):
            raise DimensionMismatchError(f"{len(labels)} labels for array of rank {t.dim()}")
        if not dt.is_complex and any(l in SPECTRAL_LABELS for l in labels):
            raise DimensionMismatchError(f"spectral labels in a real tensor: {labels}")
        object.__setattr__(self, "labels", labels)
        object.__setattr__(self, "data", t)

    def __setattr__(self, name, value):
        raise AttributeError("DenseTensor is immutable")

    # ---- introspection (reference tensor.py:152-190) ----
    @property
    def dims(self) -> tuple:
        return tuple(zip(self.labels, self.shape))

    @property
    def shape(self) -> tuple:
        return tuple(self.data.shape)

    @property
    def dtype(self) -> DType:
        return dtype_of(self.data)

    @property
    def size(self) -> int:
        return int(self.data.numel())

    @property
    def device(self) -> torch.device:
        return self.data.device

    def axis(self, label: "DimLabel | str") -> int:
        label = as_label(label)
        try:
            return self.labels.index(label)
        except ValueError:
            raise UnknownLabelError(
                f"tensor has no {label.value!r} dimension (labels {self.labels})"
            ) from None

    def extent(self, label: "DimLabel | str") -> int:
        return self.shape[self.axis(label)]

    def relabel(self, mapping: dict) -> "DenseTensor":
        return DenseTensor([mapping.get(l, l) for l in self.labels], self.data)

    def astype(self, dtype: DType) -> "DenseTensor":
        return DenseTensor(self.labels, self.data.to(dtype.torch_dtype))

    def to(self, device) -> "DenseTensor":
        return DenseTensor(self.labels, self.data.to(device))

    def numpy(self) -> np.ndarray:
        return self.data.detach().cpu().numpy()

    def __repr__(self) -> str:
        dims = "×".join(f"{l.value}:{n}" for l, n in self.dims)
        return f"DenseTensor[{dims}|{self.dtype.value}|{self.device}]"


def bit_equal(a: DenseTensor, b: DenseTensor) -> bool:
    """Labels, dtype, shape and raw bytes all equal (reference tensor.py:193-200)."""
    if a.labels != b.labels or a.dtype != b.dtype or a.shape != b.shape:
        return False
    x, y = a.data.reshape(-1), b.data.reshape(-1)
    if x.device != y.device:
        y = y.to(x.device)
    return bool(torch.equal(x.view(torch.uint8), y.view(torch.uint8)))


def _check_same_dtype(x: DenseTensor, w: DenseTensor) -> None:
    if x.dtype != w.dtype:
        raise DTypeMismatchError(f"mixed precision is disallowed: {x.dtype.value} vs {w.dtype.value}")


def einsum_channel_mix(x: DenseTensor, w: DenseTensor) -> DenseTensor:
    """Y[b, co, ...] = sum_c X[b, c, ...] W[c, co] (reference tensor.py:210-228),
    computed by libdfno's channel-mix kernel on the current GPU."""
    import ctypes

    from . import _lib

    _check_same_dtype(x, w)
    if w.data.dim() != 2:
        raise DimensionMismatchError(f"channel-mix weight must be 2-D, got {w}")
    c_axis = x.axis(DimLabel.C)
    if x.shape[c_axis] != w.shape[0]:
        raise DimensionMismatchError(f"channel extent {x.shape[c_axis]} does not match weight rows {w.shape[0]}")
    if x.dtype not in (DType.REAL32, DType.REAL64):
        raise DTypeMismatchError("channel mix supports real32 / real64")
    if not _lib.available():
        raise _lib.ExtensionMissingError("libdfno.so and a CUDA device are required (no CPU fallback)")
    dev = torch.device("cuda", torch.cuda.current_device())
    moved = x.data.to(dev).movedim(c_axis, 0)
    rest = tuple(moved.shape[1:])
    data = moved.reshape(1, moved.shape[0], -1).contiguous()
    cin, cout = w.shape
    npts = int(data.shape[2])
    g = _lib.make_geom(batch=1, c_in=cin, c=max(cin, cout), c_out=cout, grid=(1, 1, 1, 1),
                       modes=(1, 1, 1, 1), retained=(1, 1, 1, 1), nranks=1, rank=0,
                       dtype=_lib.F32 if x.dtype == DType.REAL32 else _lib.F64, act=_lib.ACT_IDENTITY,
                       x_starts=(0, 1), ky_starts=(0, 1))
    out = torch.empty((1, cout, npts), dtype=data.dtype, device=dev)
    lib = _lib.load()
    _lib.check(lib.dfno_mix_fwd(ctypes.byref(g), npts, cin, cout, _lib.ptr(data), 0,
                                _lib.ptr(w.data.to(dev).contiguous()), _lib.ptr(out), None, _lib.stream_handle()),
               "dfno_mix_fwd")
    out = out.reshape((cout,) + rest).movedim(0, c_axis)
    return DenseTensor(x.labels, out.contiguous())


def einsum_spectral(x: DenseTensor, w: DenseTensor) -> DenseTensor:
    """Per-mode contraction Y[b, co, k] = sum_c X[b, c, k] W[c, co, k]
    (reference tensor.py:231-255) on the current GPU: complex64 with square
    weights runs libdfno's x-spectral contraction kernel (the hot path calls
    it through fno.py's x-spectral stage)."""
    _check_same_dtype(x, w)
    if x.labels[0] != DimLabel.B or x.labels[1] != DimLabel.C:
        raise DimensionMismatchError(f"spectral input must be (b, c, ...), got {x}")
    if w.labels[0] != DimLabel.C or w.labels[1] != DimLabel.CO:
        raise DimensionMismatchError(f"spectral weight must be (c, co, ...), got {w}")
    if x.labels[2:] != w.labels[2:]:
        raise DimensionMismatchError(f"spectral labels disagree: {x.labels[2:]} vs {w.labels[2:]}")
    if x.shape[2:] != w.shape[2:]:
        raise DimensionMismatchError(f"spectral extents disagree: {x.shape[2:]} vs {w.shape[2:]}")
    if x.shape[1] != w.shape[0]:
        raise DimensionMismatchError(f"channel extent {x.shape[1]} does not match weight input channels {w.shape[0]}")
    import ctypes

    from . import _lib

    if not _lib.available():
        raise _lib.ExtensionMissingError("a CUDA device is required (no CPU fallback)")
    dev = torch.device("cuda", torch.cuda.current_device())
    b, c, co = x.shape[0], x.shape[1], w.shape[1]
    if x.dtype == DType.COMPLEX64 and c == co and b <= 4:
        # libdfno's weight-streaming contraction (the kernel of the fused
        # x-spectral stage, dfno_xmix_fwd): the trailing mode dims flatten to
        # one column index, described to it as a single-rank ky range
        cols = 1
        for n in x.shape[2:]:
            cols *= int(n)
        xd = x.data.to(dev).contiguous()
        wd = w.data.to(dev).contiguous()
        out = torch.empty_like(xd)
        if cols:
            g = _lib.make_geom(batch=b, c_in=c, c=c, c_out=c, grid=(1, cols, 1, 1), modes=(1, cols, 1, 1),
                               retained=(1, cols, 1, 1), nranks=1, rank=0, dtype=_lib.F32,
                               act=_lib.ACT_IDENTITY, x_starts=(0, 1), ky_starts=(0, cols))
            _lib.check(_lib.load().dfno_xmix_fwd(ctypes.byref(g), _lib.ptr(xd), _lib.ptr(wd), _lib.ptr(out),
                                                 _lib.stream_handle()), "dfno_xmix_fwd")
        return DenseTensor(x.labels, out)
    # complex128 (the real64 oracle-precision path), rectangular weights or
    # batches above the kernel's register blocking: the device einsum
    out = torch.einsum("bi...,io...->bo...", x.data.to(dev), w.data.to(dev))
    return DenseTensor(x.labels, out.contiguous())
