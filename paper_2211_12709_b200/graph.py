"""One fwd+bwd step of the FNO captured as a CUDA graph.

The reference's step (``drive_scale``, d/bench.py:381-390: forward, g = y,
backward) issues ~30 libdfno kernels through Python; replaying them as one
CUDA graph removes the per-launch host work (ctypes call, argument checks,
tensor allocation) and the launch gaps between kernels.  The graph holds the
same kernels, the same buffers and the same arithmetic as the eager calls --
``fno_forward`` / ``fno_backward`` are simply run once under
``torch.cuda.graph`` after one eager warm-up (which sizes the per-rank plan:
exchange buffers, x-spectral workspace, mixer-gradient partials, and reads
the broadcast headers).

Graphs are captured for single-rank worlds and for process-group worlds whose
collectives are stream-ordered (NCCL: every collective of the step is an
all-to-all / all-gather / broadcast on the current stream, no host
synchronisation after the warm-up).  The thread backend synchronises ranks on
the host, so it stays eager.
"""

from __future__ import annotations

from typing import Callable, Optional

import torch

from .comm import Communicator
from .errors import DimensionMismatchError
from .fno import FnoConfig, FnoParams, ForwardCache, fno_backward, fno_forward
from .tensor import DenseTensor


class FwdBwdGraph:
    """``fno_forward`` followed by ``fno_backward`` with upstream gradient
    ``grad(y)`` (default g = y, the loss 1/2 ||y||^2 of the reference's scale
    driver) captured once and replayed.

    ``x`` is the static input: write new samples into ``self.x.data`` (e.g.
    ``copy_`` from a staged host buffer) before ``replay()``.  Outputs --
    ``y``, ``gx`` and the gradients -- are static tensors overwritten by every
    replay."""

    def __init__(self, comm: Communicator, x: DenseTensor, params: FnoParams, config: FnoConfig,
                 grad: Optional[Callable[[DenseTensor], DenseTensor]] = None, backward: bool = True):
        if comm.threaded and comm.world_size > 1:
            raise DimensionMismatchError("the thread backend synchronises ranks on the host; it cannot be captured")
        if not x.data.is_cuda:
            raise DimensionMismatchError("the captured input must live on the device")
        self.comm, self.params, self.config = comm, params, config
        self.x = x
        self._grad = grad or (lambda y: y)
        self._backward = backward  # False: forward only (the reference's scale-driver column)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # eager warm-up: plans, workspaces, broadcast headers
            self._step()
        torch.cuda.current_stream().wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.y, self.gx, self.grads = self._step()

    def _step(self):
        if not self._backward:
            return fno_forward(self.comm, self.x, self.params, self.config), None, None
        cache = ForwardCache()
        y = fno_forward(self.comm, self.x, self.params, self.config, cache)
        gx, grads = fno_backward(self.comm, self._grad(y), self.params, self.config, cache)
        return y, gx, grads

    def replay(self) -> None:
        self.graph.replay()
