"""The fwd+bwd step captured as one CUDA graph (P.FwdBwdGraph) replays the
eager step bit for bit, including after new input is written into the static
input buffer."""

import pytest
import torch

import paper_2211_12709_b200 as P

pytestmark = pytest.mark.gpu


def test_graph_replay_matches_eager_step():
    cfg = P.FnoConfig(32, 16, 16, 8, 3, 4, 6, P.ModeSpec.of_xyzt(4, 4, 4, 3), 2, "gelu", "real32", 1)
    params = P.init_params(cfg, 5, device="cuda")
    x = P.DenseTensor(P.DATA_LABELS, torch.randn((2, 3, 32, 16, 16, 8), device="cuda"))

    def eager(comm, xin):
        cache = P.ForwardCache()
        y = P.fno_forward(comm, xin, params, cfg, cache)
        gx, grads = P.fno_backward(comm, y, params, cfg, cache)
        return y.data.clone(), gx.data.clone(), [t.data.clone() for t in (grads.we, grads.wd, *grads.blocks)]

    def body(comm):
        g = P.FwdBwdGraph(comm, x, params, cfg)
        out = []
        for k in range(2):
            if k:
                x.data.copy_(torch.randn_like(x.data))
            g.replay()
            torch.cuda.synchronize()
            got = (g.y.data.clone(), g.gx.data.clone(),
                   [t.data.clone() for t in (g.grads.we, g.grads.wd, *g.grads.blocks)])
            out.append((got, eager(comm, x)))
        return out

    for got, want in P.run_ranks(1, body)[0]:
        assert torch.equal(got[0], want[0]) and torch.equal(got[1], want[1])
        assert all(torch.equal(a, b) for a, b in zip(got[2], want[2]))


def test_graph_rejects_threaded_multi_rank():
    cfg = P.FnoConfig(16, 16, 16, 8, 2, 2, 2, P.ModeSpec.of_xyzt(4, 4, 4, 3), 1, "gelu", "real32", 2)
    params = P.init_params(cfg, 1, device="cuda")

    def body(comm):
        xl = P.DenseTensor(P.DATA_LABELS, torch.zeros((1, 2, 8, 16, 16, 8), device="cuda"))
        with pytest.raises(P.DimensionMismatchError):
            P.FwdBwdGraph(comm, xl, P.shard_params(params, cfg, comm.rank), cfg)
        return True

    assert all(P.run_ranks(2, body))
