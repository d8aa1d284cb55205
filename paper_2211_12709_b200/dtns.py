"""DTNS tensor files and model checkpoints.

Byte-compatible with the reference's format (d/tensor.py:258-320): magic
"DTNS", version u8 = 1, dtype code u8, ndims u8, per dimension (label code u8,
extent u64 little-endian), then the raw little-endian row-major payload
(complex as interleaved re, im).  Checkpoints are a directory of DTNS files
plus a key=value manifest (d/training.py:172-234), so checkpoints written by
the reference load here -- straight into device memory -- and ours load in
the reference.  ``gather_params`` assembles the global weights from the ky
shards on rank 0 (d/training.py:153-166).
"""

from __future__ import annotations

import os
import struct
from typing import BinaryIO, Optional, Sequence

import numpy as np
import torch

from .comm import Communicator
from .errors import MalformedHeaderError, SerializationError, TruncatedPayloadError, UnknownDTypeError
from .fno import FnoConfig, FnoParams
from .spectral import ModeSpec
from .tensor import DenseTensor, DimLabel, DType


MAGIC = b"DTNS"
FORMAT_VERSION = 1
# stable on-disk codes (reference tensor.py:50-55, :103-104)
_LABEL_CODE = {DimLabel.B: 0, DimLabel.C: 1, DimLabel.X: 2, DimLabel.Y: 3, DimLabel.Z: 4, DimLabel.T: 5,
               DimLabel.KX: 6, DimLabel.KY: 7, DimLabel.KZ: 8, DimLabel.KT: 9, DimLabel.CO: 10}
_CODE_LABEL = {v: k for k, v in _LABEL_CODE.items()}
_DTYPE_CODE = {DType.REAL32: 0, DType.REAL64: 1, DType.COMPLEX64: 2, DType.COMPLEX128: 3}
_CODE_DTYPE = {v: k for k, v in _DTYPE_CODE.items()}


def tensor_to_bytes(t: DenseTensor) -> bytes:
    """Header + little-endian payload (reference tensor.py:268-273)."""
    head = [MAGIC, struct.pack("<BBB", FORMAT_VERSION, _DTYPE_CODE[t.dtype], len(t.labels))]
    for label, extent in t.dims:
        head.append(struct.pack("<BQ", _LABEL_CODE[label], extent))
    payload = np.ascontiguousarray(t.numpy(), dtype=t.dtype.np_dtype).astype(
        np.dtype(t.dtype.np_dtype).newbyteorder("<"), copy=False).tobytes()
    return b"".join(head) + payload


def tensor_write(t: DenseTensor, sink: BinaryIO) -> int:
    buf = tensor_to_bytes(t)
    sink.write(buf)
    return len(buf)


def tensor_from_bytes(buf: bytes, device=None) -> DenseTensor:
    """Parse a DTNS stream (reference tensor.py:282-312); the tensor is
    placed on ``device`` (host when None)."""
    if len(buf) < 7 or buf[:4] != MAGIC:
        raise MalformedHeaderError("stream does not start with a DTNS header")
    version, dtype_code, ndims = struct.unpack_from("<BBB", buf, 4)
    if version != FORMAT_VERSION:
        raise MalformedHeaderError(f"unsupported format version {version}")
    if dtype_code not in _CODE_DTYPE:
        raise UnknownDTypeError(f"unknown dtype code {dtype_code}")
    dtype = _CODE_DTYPE[dtype_code]
    offset, labels, shape = 7, [], []
    for _ in range(ndims):
        if offset + 9 > len(buf):
            raise TruncatedPayloadError("stream ended inside the dimension table")
        code, extent = struct.unpack_from("<BQ", buf, offset)
        offset += 9
        if code not in _CODE_LABEL:
            raise MalformedHeaderError(f"unknown label code {code}")
        labels.append(_CODE_LABEL[code])
        shape.append(extent)
    count = int(np.prod(shape, dtype=np.int64)) if shape else 1
    nbytes = count * dtype.itemsize
    if len(buf) - offset < nbytes:
        raise TruncatedPayloadError(f"payload holds {len(buf) - offset} bytes, header declares {nbytes}")
    data = np.frombuffer(buf, dtype=np.dtype(dtype.np_dtype).newbyteorder("<"), count=count, offset=offset)
    t = torch.from_numpy(data.astype(dtype.np_dtype).reshape(shape).copy())
    return DenseTensor(labels, t.to(device) if device is not None else t)


def tensor_read(source: BinaryIO, device=None) -> DenseTensor:
    return tensor_from_bytes(source.read(), device)


def serialized_size(labels: Sequence[DimLabel], shape: Sequence[int], dtype: DType) -> int:
    """Bytes tensor_write produces for the metadata (reference tensor.py:315-320)."""
    count = int(np.prod(shape, dtype=np.int64)) if len(shape) else 1
    return 7 + 9 * len(labels) + count * dtype.itemsize


def gather_params(comm: Communicator, params: FnoParams, config: FnoConfig) -> Optional[FnoParams]:
    """Global parameters on rank 0 from the ky-sharded blocks (reference
    d/training.py:153-166); other ranks get None."""
    if not params.sharded:
        return params if comm.rank == 0 else None
    kypart = config.ky_partition()
    blocks = [comm.gather(shard, kypart, root=0, label=f"ckpt.block{i}") for i, shard in enumerate(params.blocks)]
    if comm.rank != 0:
        return None
    return FnoParams(params.we, params.wd, tuple(blocks), sharded=False)


_MANIFEST = "manifest.txt"


def save_checkpoint(directory: str, params: FnoParams, config: FnoConfig, seed: int) -> None:
    """Global weights + model description, reference layout (d/training.py:176-208)."""
    if params.sharded:
        raise ValueError("checkpoints hold global weights; gather shards first")
    os.makedirs(directory, exist_ok=True)
    entries = {
        "extents": ",".join(str(n) for n in config.grid),
        "in_channels": str(config.in_channels),
        "out_channels": str(config.out_channels),
        "hidden_channels": str(config.hidden_channels),
        "modes": ",".join(str(m) for m in config.mode_counts),
        "blocks": str(config.num_blocks),
        "activation": config.activation.value,
        "dtype": config.dtype.value,
        "world_size": str(config.num_ranks),
        "seed": str(seed),
    }
    with open(os.path.join(directory, _MANIFEST), "w", encoding="utf-8") as fh:
        for key, value in entries.items():
            fh.write(f"{key}={value}\n")
    for name, tensor in params.named().items():
        with open(os.path.join(directory, f"{name}.dtns"), "wb") as fh:
            fh.write(tensor_to_bytes(tensor))


def load_checkpoint(directory: str, device=None) -> tuple:
    """(params, config, seed) from a checkpoint directory (reference
    d/training.py:211-234); tensors land on ``device`` (host when None)."""
    entries = {}
    with open(os.path.join(directory, _MANIFEST), encoding="utf-8") as fh:
        for line in fh:
            line = line.strip()
            if line:
                key, _, value = line.partition("=")
                entries[key] = value
    grid = tuple(int(v) for v in entries["extents"].split(","))
    modes = tuple(int(v) for v in entries["modes"].split(","))
    config = FnoConfig(nx=grid[0], ny=grid[1], nz=grid[2], nt=grid[3], in_channels=int(entries["in_channels"]),
                       out_channels=int(entries["out_channels"]), hidden_channels=int(entries["hidden_channels"]),
                       modes=ModeSpec.of_xyzt(*modes), num_blocks=int(entries["blocks"]),
                       activation=entries["activation"], dtype=DType(entries["dtype"]),
                       num_ranks=int(entries["world_size"]))

    def read(name: str) -> DenseTensor:
        with open(os.path.join(directory, f"{name}.dtns"), "rb") as fh:
            return tensor_from_bytes(fh.read(), device)

    blocks = tuple(read(f"block{i}") for i in range(config.num_blocks))
    return FnoParams(read("we"), read("wd"), blocks, sharded=False), config, int(entries["seed"])


__all__ = ["MAGIC", "FORMAT_VERSION", "SerializationError", "MalformedHeaderError", "TruncatedPayloadError",
           "UnknownDTypeError", "tensor_to_bytes", "tensor_write", "tensor_from_bytes", "tensor_read",
           "serialized_size", "gather_params", "save_checkpoint", "load_checkpoint"]
