"""InputStager: pipelined pinned-host -> HBM inputs give the same step results
as synchronous copies, and a slot is never overwritten while its step runs."""

import numpy as np
import pytest
import torch

import paper_2211_12709_b200 as P
from paper_2211_12709_b200.errors import ShapeMismatchError

pytestmark = pytest.mark.gpu


def test_stager_matches_synchronous_inputs():
    cfg = P.FnoConfig(16, 16, 16, 8, 3, 2, 4, P.ModeSpec.of_xyzt(4, 4, 4, 4), 2, "gelu", "real32", 1)
    params = P.init_params(cfg, 0)
    comm = P.run_ranks(1, lambda c: c)[0]
    hosts = []
    for k in range(5):
        h = torch.empty((1, 3, 16, 16, 16, 8), dtype=torch.float32, pin_memory=True)
        h.copy_(torch.from_numpy(np.random.default_rng(k).standard_normal(h.shape).astype(np.float32)))
        hosts.append(h)
    ref = []
    for h in hosts:
        cache = P.ForwardCache()
        y = P.fno_forward(comm, P.DenseTensor(P.DATA_LABELS, h.cuda()), params, cfg, cache)
        gx, _ = P.fno_backward(comm, y, params, cfg, cache)
        ref.append((y.data.clone(), gx.data.clone()))
    stager = P.InputStager(hosts[0].shape, torch.float32)
    stager.put(hosts[0])
    for k in range(len(hosts)):
        x = stager.get()
        if k + 1 < len(hosts):
            stager.put(hosts[k + 1])
        cache = P.ForwardCache()
        y = P.fno_forward(comm, x, params, cfg, cache)
        gx, _ = P.fno_backward(comm, y, params, cfg, cache)
        assert torch.equal(y.data, ref[k][0])
        assert torch.equal(gx.data, ref[k][1])
    assert stager.h2d_bytes == 5 * hosts[0].numel() * 4
    with pytest.raises(ShapeMismatchError):
        stager.put(torch.empty((1, 3, 8, 16, 16, 8), pin_memory=True))
