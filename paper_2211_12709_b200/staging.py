"""Host -> HBM input staging for step loops (the data-loader side of the
reference's driver loops, d/bench.py:381-390 ``drive_scale`` and
d/bench.py:433-508 ``drive_train``).

The reference's inputs are host numpy arrays handed straight to
``fno_forward``.  On B200 one 64^3 x 32 x 20 fp32 slab is 671 MB -- about 13 ms
over PCIe Gen5 -- so a step loop that copies each input synchronously spends
as long on the copy as on the FNO itself.  ``InputStager`` keeps a ring of
device slots and copies step k+1's input from pinned host memory on a
dedicated copy stream while step k computes:

    stager = InputStager(shape, torch.float32, device)
    stager.put(x_host[0])
    for k in range(steps):
        x = stager.get()                    # compute stream waits for the H2D of step k
        if k + 1 < steps:
            stager.put(x_host[k + 1])       # overlaps with step k's forward + backward
        y = fno_forward(comm, x, params, config, cache)
        ...

A slot is overwritten only after every kernel enqueued on the compute stream
before the following ``get()`` -- i.e. the whole step that read it, backward
included (the forward cache keeps the input for the encoder's weight
gradient) -- has completed.
"""

from __future__ import annotations

from collections import deque

import torch

from .errors import ShapeMismatchError
from .tensor import DATA_LABELS, DenseTensor


class InputStager:
    def __init__(self, shape, dtype=torch.float32, device=None, depth: int = 2, labels=DATA_LABELS,
                 copy_streams: int = 1):
        if depth < 2:
            raise ValueError("depth must be >= 2 (one slot computing, one filling)")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.shape = tuple(shape)
        self.dtype = dtype
        self.labels = tuple(labels)
        self.slots = [torch.empty(self.shape, dtype=dtype, device=self.device) for _ in range(depth)]
        # the copy may be split over several streams (measured: one is fastest on PCIe Gen5)
        self.copy_streams = [torch.cuda.Stream(device=self.device) for _ in range(max(1, copy_streams))]
        self.copy_stream = self.copy_streams[0]
        self.filled = [[torch.cuda.Event() for _ in self.copy_streams] for _ in range(depth)]  # H2D parts done
        self.released = [None] * depth                               # compute done with the slot
        self.pending = deque()                                       # slots filled, not yet handed out
        self.in_use = None                                           # slot handed out by the last get()
        self.next_slot = 0
        self.h2d_bytes = 0

    def put(self, host) -> None:
        """Start the H2D copy of ``host`` (pinned CPU tensor or DenseTensor)
        into the next free slot, on the copy stream."""
        data = host.data if isinstance(host, DenseTensor) else host
        if tuple(data.shape) != self.shape or data.dtype != self.dtype:
            raise ShapeMismatchError(f"staged input {tuple(data.shape)} {data.dtype}, expected {self.shape} {self.dtype}")
        s = self.next_slot
        if len(self.pending) + (self.in_use is not None) >= len(self.slots):
            raise RuntimeError("InputStager: every slot is filled or in use; get() before put()")
        self.next_slot = (s + 1) % len(self.slots)
        src, dst = data.reshape(-1), self.slots[s].reshape(-1)
        n, k = src.numel(), len(self.copy_streams)
        for j, cs in enumerate(self.copy_streams):
            a, b = n * j // k, n * (j + 1) // k
            with torch.cuda.stream(cs):
                if self.released[s] is not None:
                    cs.wait_event(self.released[s])
                dst[a:b].copy_(src[a:b], non_blocking=True)
                self.filled[s][j].record(cs)
        self.h2d_bytes += data.numel() * data.element_size()
        self.pending.append(s)

    def get(self) -> DenseTensor:
        """The oldest staged input, usable on the current stream.  Also marks
        the previously handed-out slot free once the work enqueued so far
        (its whole step) completes."""
        if not self.pending:
            raise RuntimeError("InputStager: get() without a staged input")
        cur = torch.cuda.current_stream(self.device)
        if self.in_use is not None:
            ev = torch.cuda.Event()
            ev.record(cur)
            self.released[self.in_use] = ev
        s = self.pending.popleft()
        for ev in self.filled[s]:
            cur.wait_event(ev)
        self.in_use = s
        return DenseTensor(self.labels, self.slots[s])

    def synchronize(self) -> None:
        for cs in self.copy_streams:
            cs.synchronize()
