"""Collectives of the FNO path with the reference's exact accounting.

``Communicator`` keeps the reference's collective API and ``CommStats``
contract (/root/reference/pkg/src/distfno/comm.py:57-104, :330-542):
``broadcast`` (B), its adjoint ``reduce_sum``, ``repartition`` (R),
``gather`` and ``allreduce_sum_scalar``, each recording calls and *off-rank*
elements / bytes per primitive, plus the hot-path primitive ``exchange`` -- the
peer-major all-to-all(v) the fused kernels pack for (recorded as a
repartition, like the reference's ``Communicator.repartition``).

Two backends carry the bytes:

* ``ProcessGroupBackend`` -- one process per GPU over ``torch.distributed``:
  NCCL over NVLink / NVSwitch on the GPU box (``all_to_all_single`` with the
  uneven split sizes of ``block_decompose``), gloo for CPU tests.
* ``ThreadWorld`` -- ranks are threads of one process sharing one device (the
  reference's in-process transport, comm.py:112-155, :555-587).  Used to run
  P-rank decompositions on a single GPU in the parity tests; collectives are
  device-to-device copies.

Collectives are blocking and must be called in identical order on every rank.
Each call carries the reference's 64-bit tag (crc32(label) << 32 | primitive
<< 24 | sequence, comm.py:343-350); the thread backend compares tags across
ranks and raises ``CollectiveMismatchError`` on disagreement and
``CollectiveTimeoutError`` when a peer never arrives.
"""

from __future__ import annotations

import copy
import threading
import zlib
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import torch

from .errors import CollectiveMismatchError, CollectiveTimeoutError, ShapeMismatchError
from .partition import Partition, repartition_plan
from .tensor import DenseTensor

BROADCAST = "broadcast"
REDUCE_SUM = "reduce_sum"
REPARTITION = "repartition"
GATHER = "gather"
ALLREDUCE_SCALAR = "allreduce_scalar"
_PRIM_CODE = {BROADCAST: 1, REDUCE_SUM: 2, REPARTITION: 3, GATHER: 4, ALLREDUCE_SCALAR: 5}
DEFAULT_TIMEOUT = 60.0
_MAX_DIMS = 8


@dataclass
class PrimitiveStats:
    calls: int = 0
    elements: int = 0
    bytes: int = 0


@dataclass
class CommStats:
    """Per-rank counters per primitive; only off-rank traffic counts
    (reference comm.py:64-92)."""

    rank: int = 0
    primitives: dict = field(default_factory=dict)

    def record(self, primitive: str, elements: int, nbytes: int) -> None:
        entry = self.primitives.setdefault(primitive, PrimitiveStats())
        entry.calls += 1
        entry.elements += int(elements)
        entry.bytes += int(nbytes)

    def get(self, primitive: str) -> PrimitiveStats:
        return self.primitives.get(primitive, PrimitiveStats())

    def snapshot(self) -> "CommStats":
        return copy.deepcopy(self)

    def minus(self, earlier: "CommStats") -> "CommStats":
        out = CommStats(rank=self.rank)
        for name, entry in self.primitives.items():
            prev = earlier.get(name)
            out.primitives[name] = PrimitiveStats(
                entry.calls - prev.calls, entry.elements - prev.elements, entry.bytes - prev.bytes
            )
        return out


def aggregate_stats(per_rank: Sequence[CommStats]) -> CommStats:
    """Sum counters over ranks (reference comm.py:95-104)."""
    out = CommStats(rank=-1)
    for stats in per_rank:
        for name, entry in stats.primitives.items():
            acc = out.primitives.setdefault(name, PrimitiveStats())
            acc.calls += entry.calls
            acc.elements += entry.elements
            acc.bytes += entry.bytes
    return out


def describe_tag(tag: int) -> str:
    names = {v: k for k, v in _PRIM_CODE.items()}
    return f"collective #{tag & 0xFFFFFF} ({names.get((tag >> 24) & 0xFF, 'unknown')}, tag {tag:#x})"


# ---------------------------------------------------------------------------
# backends: each provides rank, world_size, device and five raw operations
# ---------------------------------------------------------------------------


class ThreadWorld:
    """In-process world: rank threads meet at a barrier and read each other's
    posted tensors (reference InProcessTransport, comm.py:112-155)."""

    def __init__(self, world_size: int, device=None, timeout: float = DEFAULT_TIMEOUT):
        self.world_size = world_size
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")
        )
        self.timeout = timeout
        self._barrier = threading.Barrier(world_size)
        self._slots = [None] * world_size
        self._done = [None] * world_size

    def backend(self, rank: int) -> "ThreadBackend":
        return ThreadBackend(self, rank)


def _stream_event(device):
    """An event recorded on the calling thread's current CUDA stream (None
    without CUDA): rank threads may run on different streams, so every
    cross-rank read waits for the producer's event and every owner waits for
    its readers' events before the buffer can be reused."""
    if device.type != "cuda":
        return None
    ev = torch.cuda.Event()
    ev.record()
    return ev


def _wait(ev) -> None:
    if ev is not None:
        torch.cuda.current_stream().wait_event(ev)


def _private(obj):
    """Copy every tensor in a posted payload onto the reader's stream."""
    if isinstance(obj, torch.Tensor):
        return obj.clone()
    if isinstance(obj, tuple):
        return tuple(_private(o) for o in obj)
    if isinstance(obj, list):
        return [_private(o) for o in obj]
    return obj


class ThreadBackend:
    def __init__(self, world: ThreadWorld, rank: int):
        self.world = world
        self.rank = rank
        self.world_size = world.world_size
        self.device = world.device

    def _sync(self):
        try:
            self.world._barrier.wait(timeout=self.world.timeout)
        except threading.BrokenBarrierError:
            raise CollectiveTimeoutError(
                f"rank {self.rank} timed out at a collective; a peer likely skipped it"
            ) from None

    def _check_tags(self, tag, posted):
        for peer, entry in enumerate(posted):
            if entry[0] != tag:
                return CollectiveMismatchError(
                    f"rank {self.rank} issued {describe_tag(tag)} but rank {peer} issued {describe_tag(entry[0])}"
                )
        return None

    def post_and_collect(self, tag: int, payload, collect: bool = True) -> list:
        """Publish (tag, payload); return every rank's payload in rank order
        once all have arrived.  Tags must agree (reference comm.py:137-152).
        Peers' tensors come back as private copies made on this rank's stream
        after the producers' events, so no rank reads a buffer its owner may
        still be writing or may free afterwards.  With ``collect=False`` this
        rank only posts (peers' entries come back as None)."""
        self.world._slots[self.rank] = (tag, payload, _stream_event(self.device))
        self._sync()
        posted = list(self.world._slots)
        err = self._check_tags(tag, posted)
        out = []
        if err is None:
            for peer, (_, p, ev) in enumerate(posted):
                if peer == self.rank or not collect:
                    out.append(p if peer == self.rank else None)
                    continue
                _wait(ev)
                out.append(_private(p))
        self.world._done[self.rank] = _stream_event(self.device)
        self._sync()  # nobody overwrites a slot before everyone has read it
        for peer, ev in enumerate(self.world._done):
            if peer != self.rank:
                _wait(ev)
        if err is not None:
            raise err
        return out

    def exchange(self, tag, send, recv, send_counts, recv_counts):
        # Device-to-device copies on this rank's current stream, ordered after
        # every producer's event; the owner waits for all readers' events
        # before it may overwrite its send buffer.
        self.world._slots[self.rank] = (tag, (send, list(send_counts)), _stream_event(self.device))
        self._sync()
        posted = list(self.world._slots)
        err = self._check_tags(tag, posted)
        if err is None:
            roff = 0
            for peer in range(self.world_size):
                _, (psend, pcounts), ev = posted[peer]
                n = recv_counts[peer]
                if n != pcounts[self.rank]:
                    err = CollectiveMismatchError(
                        f"rank {self.rank} expects {n} elements from rank {peer}, which sends {pcounts[self.rank]}"
                    )
                    break
                soff = sum(pcounts[: self.rank])
                if n:
                    _wait(ev)
                    recv[roff : roff + n].copy_(psend[soff : soff + n])
                roff += n
        self.world._done[self.rank] = _stream_event(self.device)
        self._sync()
        for peer, ev in enumerate(self.world._done):
            if peer != self.rank:
                _wait(ev)
        if err is not None:
            raise err

    def close(self):
        pass


class ProcessGroupBackend:
    """torch.distributed process group (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None, device=None):
        import torch.distributed as dist

        if not dist.is_initialized():
            raise CollectiveMismatchError("torch.distributed is not initialised")
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world_size = dist.get_world_size(group)
        if device is None:
            backend = dist.get_backend(group)
            device = (
                torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
            )
        self.device = torch.device(device)

    def _global(self, r: int) -> int:
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def all_gather_tensor(self, t: torch.Tensor) -> list:
        parts = [torch.empty_like(t) for _ in range(self.world_size)]
        self.dist.all_gather(parts, t.contiguous(), group=self.group)
        return parts

    def broadcast_(self, t: torch.Tensor, root: int) -> None:
        self.dist.broadcast(t, src=self._global(root), group=self.group)

    def broadcast_header(self, t, root: int):
        """(labels, shape, dtype) of the root's tensor via one small int64
        broadcast (non-root ranks may hold None, reference comm.py:361-368)."""
        from .tensor import DimLabel, DType

        lab = list(DimLabel)
        dts = list(DType)
        hdr = torch.zeros(2 + 2 * _MAX_DIMS, dtype=torch.int64, device=self.device)
        if self.rank == root:
            if t.data.dim() > _MAX_DIMS:
                raise ShapeMismatchError(f"broadcast supports at most {_MAX_DIMS} dims")
            vals = [dts.index(t.dtype), t.data.dim()] + list(t.shape) + [0] * (_MAX_DIMS - t.data.dim())
            vals += [lab.index(l) for l in t.labels] + [0] * (_MAX_DIMS - t.data.dim())
            hdr.copy_(torch.tensor(vals, dtype=torch.int64))
        self.broadcast_(hdr, root)
        v = hdr.tolist()
        nd = v[1]
        shape = tuple(v[2 : 2 + nd])
        labels = tuple(lab[k] for k in v[2 + _MAX_DIMS : 2 + _MAX_DIMS + nd])
        return labels, shape, dts[v[0]]

    def send(self, t: torch.Tensor, dst: int):
        self.dist.send(t.contiguous(), dst=self._global(dst), group=self.group)

    def recv(self, t: torch.Tensor, src: int):
        self.dist.recv(t, src=self._global(src), group=self.group)

    def exchange(self, tag, send, recv, send_counts, recv_counts):
        self.dist.all_to_all_single(
            recv, send, output_split_sizes=list(recv_counts), input_split_sizes=list(send_counts), group=self.group
        )

    def close(self):
        pass


def _as_real_flat(t: torch.Tensor) -> torch.Tensor:
    t = t.reshape(-1)
    return torch.view_as_real(t).reshape(-1) if t.is_complex() else t


class Communicator:
    """Collectives over one rank's backend with per-primitive accounting
    (reference comm.py:330-542)."""

    def __init__(self, backend, timeout: float = DEFAULT_TIMEOUT):
        self._be = backend
        self.rank = backend.rank
        self.world_size = backend.world_size
        self.device = backend.device
        self.timeout = timeout
        self.stats = CommStats(rank=self.rank)
        self._seq = 0
        self._bcast_meta = {}

    @classmethod
    def from_process_group(cls, group=None, device=None) -> "Communicator":
        return cls(ProcessGroupBackend(group, device))

    @property
    def threaded(self) -> bool:
        return isinstance(self._be, ThreadBackend)

    def _next_tag(self, primitive: str, label: str) -> int:
        tag = (zlib.crc32(label.encode()) << 32) | (_PRIM_CODE[primitive] << 24) | (self._seq & 0xFFFFFF)
        self._seq += 1
        return tag

    def report(self) -> CommStats:
        return self.stats.snapshot()

    def close(self) -> None:
        self._be.close()

    # ---- helpers -------------------------------------------------------
    def _gather_all(self, tag: int, t: torch.Tensor, collect: bool = True) -> list:
        """Every rank's tensor, in rank order (same shape on all ranks); with
        ``collect=False`` on the thread backend this rank only contributes."""
        if self.threaded:
            return self._be.post_and_collect(tag, t, collect)
        return self._be.all_gather_tensor(t)

    # ---- collectives ---------------------------------------------------
    def broadcast(self, t: Optional[DenseTensor], root: int = 0, label: str = "") -> DenseTensor:
        """Replicate the root's tensor on every rank (reference comm.py:361-388)."""
        tag = self._next_tag(BROADCAST, label)
        if self.rank == root and t is None:
            raise CollectiveMismatchError("broadcast root holds no tensor")
        if self.world_size == 1:
            self.stats.record(BROADCAST, 0, 0)
            return t
        if self.threaded:
            payload = (t.labels, t.data) if self.rank == root else None
            posted = self._be.post_and_collect(tag, payload, collect=self.rank != root)
            labels, data = posted[root]
            received = DenseTensor(labels, data.to(self.device))
        else:
            # The (labels, shape, dtype) header is read back once per label;
            # later broadcasts under the same label reuse it, so the steady
            # state has no device -> host synchronisation.  Every rank checks
            # its own tensor against the header before any payload moves.
            meta = self._bcast_meta.get(label) if label else None
            if meta is None:
                meta = self._be.broadcast_header(t, root)
                if label:
                    self._bcast_meta[label] = meta
            labels, shape, dtype = meta
            if t is not None and (tuple(t.labels) != tuple(labels) or tuple(t.shape) != tuple(shape)
                                  or t.dtype != dtype):
                raise CollectiveMismatchError(
                    f"rank {self.rank} broadcast {label!r}: local {t.dims} {t.dtype} disagrees with the "
                    f"root's {tuple(zip(labels, shape))} {dtype}")
            if self.rank == root:
                buf = t.data.to(self.device).contiguous()
            else:
                buf = torch.empty(shape, dtype=dtype.torch_dtype, device=self.device)
            self._be.broadcast_(buf, root)
            received = DenseTensor(labels, buf)
        if self.rank == root:
            sent = t.size * (self.world_size - 1)
            self.stats.record(BROADCAST, sent, sent * t.dtype.itemsize)
            return t
        if t is not None and (t.dims != received.dims or t.dtype != received.dtype):
            raise CollectiveMismatchError(
                f"rank {self.rank} broadcast metadata {t.dims} disagrees with root's {received.dims}"
            )
        self.stats.record(BROADCAST, 0, 0)
        return received

    def reduce_sum(self, t: DenseTensor, root: int = 0, label: str = "") -> Optional[DenseTensor]:
        """Element-wise sum delivered on root, summed in rank order so the
        result is deterministic (reference comm.py:390-419)."""
        tag = self._next_tag(REDUCE_SUM, label)
        if self.world_size == 1:
            self.stats.record(REDUCE_SUM, 0, 0)
            return DenseTensor(t.labels, t.data.clone())
        parts = self._gather_all(tag, t.data.to(self.device), collect=self.rank == root)
        if self.rank != root:
            self.stats.record(REDUCE_SUM, t.size, t.size * t.dtype.itemsize)
            return None
        for src, p in enumerate(parts):
            if tuple(p.shape) != t.shape or p.dtype != t.data.dtype:
                raise CollectiveMismatchError(f"reduce_sum shapes disagree: root {t.dims}, rank {src} {tuple(p.shape)}")
        acc = parts[0].clone()
        for p in parts[1:]:
            acc += p.to(acc.device)
        self.stats.record(REDUCE_SUM, 0, 0)
        return DenseTensor(t.labels, acc)

    def allreduce_sum(self, t: torch.Tensor, label: str = "") -> torch.Tensor:
        """reduce_sum to rank 0 followed by broadcast, fused: every rank sums
        the gathered parts in rank order, so replicas are bit-identical
        (reference fno_backward d/fno.py:501-508).  Records the reference's
        two primitives."""
        tag = self._next_tag(REDUCE_SUM, label)
        n = t.numel()
        item = t.element_size()
        if self.world_size == 1:
            self.stats.record(REDUCE_SUM, 0, 0)
            self._next_tag(BROADCAST, label + ".re")
            self.stats.record(BROADCAST, 0, 0)
            return t
        parts = self._gather_all(tag, t)
        acc = parts[0].clone()
        for p in parts[1:]:
            acc += p
        self.stats.record(REDUCE_SUM, 0 if self.rank == 0 else n, 0 if self.rank == 0 else n * item)
        self._next_tag(BROADCAST, label + ".re")
        sent = n * (self.world_size - 1) if self.rank == 0 else 0
        self.stats.record(BROADCAST, sent, sent * item)
        return acc

    def allreduce_sum_many(self, tensors: Sequence[torch.Tensor], labels: Sequence[str]) -> list:
        """``reduce_sum`` to rank 0 then ``broadcast`` of several tensors in ONE
        collective: the flattened tensors travel as one all-gather and every
        rank sums the parts in rank order, so replicas are bit-identical with
        no host synchronisation (reference fno_backward d/fno.py:501-508).
        CommStats and tags are recorded exactly as the reference's sequence
        reduce_sum(t0), reduce_sum(t1), ..., broadcast(t0), broadcast(t1), ..."""
        P = self.world_size
        for t, label in zip(tensors, labels):
            self._next_tag(REDUCE_SUM, label)
            n, item = t.numel(), t.element_size()
            self.stats.record(REDUCE_SUM, 0 if self.rank == 0 or P == 1 else n, 0 if self.rank == 0 or P == 1 else n * item)
        if P == 1:
            out = list(tensors)
        else:
            sizes = [t.numel() for t in tensors]
            flat = torch.cat([t.reshape(-1) for t in tensors])
            tag = (zlib.crc32("|".join(labels).encode()) << 32) | (_PRIM_CODE[REDUCE_SUM] << 24) | (self._seq & 0xFFFFFF)
            parts = self._gather_all(tag, flat)
            acc = parts[0].clone()
            for p in parts[1:]:
                acc += p
            out, off = [], 0
            for t, n in zip(tensors, sizes):
                out.append(acc[off : off + n].view(t.shape))
                off += n
        for t, label in zip(tensors, labels):
            self._next_tag(BROADCAST, label + ".re")
            n, item = t.numel(), t.element_size()
            sent = n * (P - 1) if self.rank == 0 else 0
            self.stats.record(BROADCAST, sent, sent * item)
        return out

    def exchange(self, send: torch.Tensor, recv: torch.Tensor, send_counts: Sequence[int],
                 recv_counts: Sequence[int], label: str = "", record: bool = True) -> int:
        """Peer-major all-to-all(v) of packed buffers; counts in elements of
        ``send``'s dtype.  Recorded as one repartition with the off-rank
        element count, exactly as the reference's repartition
        (comm.py:461-482) -- unless ``record`` is false, for the chunks of a
        pipelined repartition that ``record_repartition`` accounts once.
        Returns the off-rank element count.  Runs on the current stream."""
        tag = self._next_tag(REPARTITION, label)
        if len(send_counts) != self.world_size or len(recv_counts) != self.world_size:
            raise ShapeMismatchError("one split size per rank is required")
        off_rank = sum(n for p, n in enumerate(send_counts) if p != self.rank)
        if self.world_size > 1:
            s, r = _as_real_flat(send), _as_real_flat(recv)
            k = 2 if send.is_complex() else 1
            self._be.exchange(tag, s, r, [k * n for n in send_counts], [k * n for n in recv_counts])
        elif send.data_ptr() != recv.data_ptr():
            recv.reshape(-1).copy_(send.reshape(-1))
        if record:
            self.stats.record(REPARTITION, off_rank, off_rank * send.element_size())
        return off_rank

    def record_repartition(self, off_rank_elements: int, itemsize: int) -> None:
        """Account one (chunked) repartition with its total off-rank elements."""
        self.stats.record(REPARTITION, off_rank_elements, off_rank_elements * itemsize)

    def repartition(self, t: DenseTensor, src_part: Partition, dst_part: Partition, label: str = "") -> DenseTensor:
        """Move this rank's src slab to its dst slab (reference comm.py:421-483).
        Generic labelled form: packs the routing-table blocks peer-major,
        runs ``exchange``, unpacks.  The FNO hot path packs in its kernels
        instead."""
        if src_part.num_ranks != self.world_size:
            raise ShapeMismatchError(f"partition has {src_part.num_ranks} ranks, world is {self.world_size}")
        dims = []
        for lbl, extent in t.dims:
            if lbl == src_part.dim:
                if extent != src_part.extent_of(self.rank):
                    raise ShapeMismatchError(
                        f"rank {self.rank} holds {extent} along {lbl.value!r}, partition says "
                        f"{src_part.extent_of(self.rank)}"
                    )
                dims.append((lbl, src_part.global_extent))
            else:
                dims.append((lbl, extent))
        plan = repartition_plan(src_part, dst_part, dims, self.rank)
        data = t.data.to(self.device)
        send = torch.cat([data[e.send_slices()].reshape(-1) for e in plan]) if plan else data.reshape(-1)
        out_shape = [dst_part.extent_of(self.rank) if l == dst_part.dim else e for l, e in dims]
        recv = torch.empty(sum(e.recv_element_count for e in plan), dtype=data.dtype, device=self.device)
        self.exchange(send, recv, [e.element_count for e in plan], [e.recv_element_count for e in plan], label)
        out = torch.empty(out_shape, dtype=data.dtype, device=self.device)
        off = 0
        for e in plan:
            n = e.recv_element_count
            shape = tuple(len(r) for r in e.recv)
            out[e.recv_slices()] = recv[off : off + n].reshape(shape)
            off += n
        return DenseTensor(t.labels, out)

    def gather(self, t: DenseTensor, part: Partition, root: int = 0, label: str = "") -> Optional[DenseTensor]:
        """Assemble the global tensor on root (reference comm.py:485-522)."""
        tag = self._next_tag(GATHER, label)
        axis = t.axis(part.dim)
        if t.shape[axis] != part.extent_of(self.rank):
            raise ShapeMismatchError(
                f"rank {self.rank} slab extent {t.shape[axis]} does not match partition extent "
                f"{part.extent_of(self.rank)}"
            )
        data = t.data.to(self.device).contiguous()
        if self.world_size == 1:
            self.stats.record(GATHER, 0, 0)
            return DenseTensor(t.labels, data.clone())
        shape = list(t.shape)
        if self.threaded:
            blocks = self._be.post_and_collect(tag, (t.labels, data), collect=self.rank == root)
            if self.rank != root:
                self.stats.record(GATHER, t.size, t.size * t.dtype.itemsize)
                return None
            for src, (labels, _) in enumerate(blocks):
                if labels != t.labels:
                    raise CollectiveMismatchError(f"gather labels disagree: {labels} vs {t.labels}")
            blocks = [b for _, b in blocks]
        else:
            # complex payloads travel as their real view (NCCL has no complex type)
            if self.rank != root:
                self._be.send(torch.view_as_real(data) if data.is_complex() else data, root)
                self.stats.record(GATHER, t.size, t.size * t.dtype.itemsize)
                return None
            blocks = []
            for src in range(self.world_size):
                if src == root:
                    blocks.append(data)
                    continue
                s = list(shape)
                s[axis] = part.extent_of(src)
                buf = torch.empty(s, dtype=data.dtype, device=self.device)
                self._be.recv(torch.view_as_real(buf) if buf.is_complex() else buf, src)
                blocks.append(buf)
        for src, b in enumerate(blocks):
            if b.shape[axis] != part.extent_of(src):
                raise CollectiveMismatchError(
                    f"gather slab from rank {src} has extent {b.shape[axis]}, partition says {part.extent_of(src)}"
                )
        self.stats.record(GATHER, 0, 0)
        return DenseTensor(t.labels, torch.cat([b.to(self.device) for b in blocks], dim=axis))

    def allreduce_sum_scalar(self, value: float, label: str = "") -> float:
        """float64 sum over ranks, identical on every rank (reference
        comm.py:524-542): root-ordered summation."""
        tag = self._next_tag(ALLREDUCE_SCALAR, label)
        if self.world_size == 1:
            self.stats.record(ALLREDUCE_SCALAR, 0, 0)
            return float(value)
        t = torch.tensor([float(value)], dtype=torch.float64, device=self.device)
        parts = self._gather_all(tag, t)
        total = float(parts[0].item())
        for p in parts[1:]:
            total += float(p.item())
        if self.rank == 0:
            self.stats.record(ALLREDUCE_SCALAR, self.world_size - 1, 8 * (self.world_size - 1))
        else:
            self.stats.record(ALLREDUCE_SCALAR, 1, 8)
        return total

    def barrier(self) -> None:
        if self.world_size == 1:
            return
        if self.threaded:
            self._be._sync()
        else:
            self._be.dist.barrier(group=self._be.group)


def comm_report(comm: Communicator) -> CommStats:
    return comm.report()


def run_ranks(world_size: int, fn: Callable, timeout: float = DEFAULT_TIMEOUT, device=None,
              join_timeout: float = 600.0) -> list:
    """Run ``fn(comm)`` on every rank of an in-process (threaded) world and
    return the results in rank order; the first rank exception is re-raised
    (reference comm.py:555-587).  All ranks share one CUDA device."""
    world = ThreadWorld(world_size, device=device, timeout=timeout)
    results = [None] * world_size
    errors = [None] * world_size
    dev = world.device

    def runner(rank: int) -> None:
        if dev.type == "cuda":
            torch.cuda.set_device(dev)
        comm = Communicator(world.backend(rank), timeout=timeout)
        try:
            results[rank] = fn(comm)
        except BaseException as exc:  # noqa: BLE001 - re-raised below
            errors[rank] = exc
            world._barrier.abort()

    threads = [threading.Thread(target=runner, args=(r,), daemon=True) for r in range(world_size)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=join_timeout)
        if t.is_alive():
            raise CollectiveTimeoutError("a rank thread did not finish")
    primary = [e for e in errors if e is not None and not isinstance(e, CollectiveTimeoutError)]
    if primary:
        raise primary[0]
    for e in errors:
        if e is not None:
            raise e
    return results
