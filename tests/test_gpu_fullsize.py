"""Full-size value parity: fno_forward + fno_backward through the public API
at the headline and north-star configurations, against the float64 torch.fft
restatement of the reference (oracle/torch_ref.py), which is
itself pinned here to the numpy oracle at C1 and (on CPU,
tests/test_torch_ref.py) to the reference's own golden vectors.

  * C1 32^3 x 16, c = 20, 4 blocks: torch_ref (GPU) vs numpy oracle < 1e-12,
    and the fp32 path vs both
  * C2 64^3 x 32, c = 20, 4 blocks, GELU -- the bench headline
  * C3 128^3 x 32, c = 20, 4 blocks at P = 1 and the P = 2 strong-scaling split
  * C4 262 x 118 x 64 x 86 (the paper's CO2 grid) at P = 8 thread-ranks on one
    GPU: every rank runs the exact P = 8 geometry (x slabs of 33 / 32, the
    Nx = 262 ky-pencils of width 2); width 8 so the float64 oracle fits
  * C5 P = 2 rank geometry (128 x 64 x 64 x 32)

Tolerances (metric max|a-b| / max(max|a|, max|b|), d/bench.py:83-85):
outputs 1e-5, every gradient 1e-4 (the fp32 build runs its DFTs as 3xTF32 on
tcgen05).  The upstream gradient g is a seeded random
field, so gradient errors are not masked by the forward error.
"""

import gc

import numpy as np
import pytest
import torch

import paper_2211_12709_b200 as P
from oracle import fno_oracle as O
from oracle import torch_ref as R

pytestmark = pytest.mark.gpu

TOL_Y = 1e-5
TOL_G = 1e-4


def _config(grid, modes, c, blocks, ranks, act="gelu", cin=None, cout=None):
    return P.FnoConfig(nx=grid[0], ny=grid[1], nz=grid[2], nt=grid[3], in_channels=cin or c,
                       out_channels=cout or c, hidden_channels=c, modes=P.ModeSpec.of_xyzt(*modes),
                       num_blocks=blocks, activation=act, dtype="real32", num_ranks=ranks)


def _inputs(config, seed, batch=1):
    dev = torch.device("cuda")
    params = P.init_params(config, seed, device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    shape_in = (batch, config.in_channels) + config.grid
    shape_out = (batch, config.out_channels) + config.grid
    x = torch.randn(shape_in, generator=gen, device=dev, dtype=torch.float32)
    g = torch.randn(shape_out, generator=gen, device=dev, dtype=torch.float32)
    return params, x, g


def _ours(config, params, x, g):
    """Forward + backward on config.num_ranks thread-ranks through the public
    API; returns the gathered y, gx (device), mixer grads and the block grads
    concatenated over the ky shards."""
    xpart = config.x_partition()
    xd = P.DenseTensor(P.DATA_LABELS, x)
    gd = P.DenseTensor(P.DATA_LABELS, g)

    def worker(comm):
        lp = P.shard_params(params, config, comm.rank)
        cache = P.ForwardCache()
        y = P.fno_forward(comm, P.slice_local(xd, xpart, comm.rank), lp, config, cache=cache)
        gx, grads = P.fno_backward(comm, P.slice_local(gd, xpart, comm.rank), lp, config, cache)
        return y.data, gx.data, grads

    res = P.run_ranks(config.num_ranks, worker)
    torch.cuda.synchronize()
    y = torch.cat([r[0] for r in res], dim=2)
    gx = torch.cat([r[1] for r in res], dim=2)
    gws = [torch.cat([r[2].blocks[i].data for r in res], dim=3) for i in range(config.num_blocks)]
    out = (y, gx, res[0][2].we.data, res[0][2].wd.data, gws)
    del res
    P.clear_plans()
    gc.collect()
    torch.cuda.empty_cache()
    return out


def _reference(config, params, x, g):
    modes = config.mode_counts
    blocks = [w.data for w in params.blocks]
    ry, cache = R.forward(x, params.we.data, params.wd.data, blocks, modes, config.activation.value)
    rgx, rgwe, rgwd, rgws = R.backward(g, params.we.data, params.wd.data, blocks, modes, cache,
                                       config.activation.value)
    del cache
    return ry, rgx, rgwe, rgwd, rgws


def _compare(ours, ref):
    y, gx, gwe, gwd, gws = ours
    ry, rgx, rgwe, rgwd, rgws = ref
    errs = {"y": R.rel_err(y, ry), "gx": R.rel_err(gx, rgx), "gwe": R.rel_err(gwe, rgwe),
            "gwd": R.rel_err(gwd, rgwd)}
    for i, (a, b) in enumerate(zip(gws, rgws)):
        errs[f"gw{i}"] = R.rel_err(a, b)
    return errs


def _check(errs):
    print({k: f"{v:.2e}" for k, v in errs.items()})
    assert errs["y"] < TOL_Y, errs
    assert all(v < TOL_G for k, v in errs.items() if k != "y"), errs


def _free():
    P.clear_plans()
    gc.collect()
    torch.cuda.empty_cache()


def test_c1_torch_ref_pinned_to_numpy_oracle_and_fp32_path():
    # C1 (the reference's CPU config): the GPU float64 restatement against the
    # numpy oracle, then the fp32 path against both
    config = _config((32, 32, 32, 16), (8, 8, 8, 8), 20, 4, 1)
    params, x, g = _inputs(config, 21)
    ref = _reference(config, params, x, g)
    xn, gn = x.double().cpu().numpy(), g.double().cpu().numpy()
    we, wd = params.we.numpy().astype(np.float64), params.wd.numpy().astype(np.float64)
    blocks = [w.numpy().astype(np.complex128) for w in params.blocks]
    oy, cache = O.forward(xn, we, wd, blocks, config.mode_counts, with_cache=True)
    ogx, ogwe, ogwd, ogws = O.backward(gn, we, wd, blocks, config.mode_counts, cache)
    for a, b in ((ref[0], oy), (ref[1], ogx), (ref[2], ogwe), (ref[3], ogwd), *zip(ref[4], ogws)):
        assert O.rel_err(a.cpu().numpy(), b) < 1e-12
    _check(_compare(_ours(config, params, x, g), ref))
    _free()


def test_c2_headline_config():
    # bench.py's N = 1 workload: 64^3 x 32, c = 20, 4 blocks, m = 8, GELU
    config = _config((64, 64, 64, 32), (8, 8, 8, 8), 20, 4, 1)
    params, x, g = _inputs(config, 22)
    ours = _ours(config, params, x, g)
    _check(_compare(ours, _reference(config, params, x, g)))
    del ours
    _free()


@pytest.mark.parametrize("ranks", [1, 2])
def test_c3_128cubed(ranks):
    config = _config((128, 128, 128, 32), (8, 8, 8, 8), 20, 4, ranks)
    params, x, g = _inputs(config, 23)
    ours = _ours(config, params, x, g)
    _check(_compare(ours, _reference(config, params, x, g)))
    del ours
    _free()


@pytest.mark.parametrize("groups", [1, 2], ids=["unsplit", "pipelined"])
def test_c4_co2_grid_p8_geometry(groups, monkeypatch):
    from paper_2211_12709_b200 import fno as F

    monkeypatch.setattr(F, "PIPELINE_GROUPS_THREADED", groups)
    # 262 x 118 x 64 x 86 at P = 8: x slabs 33 x 6 + 32 x 2, ky pencils of 2,
    # Nt = 86 and Ny = 118 (not multiples of 4 / 8)
    config = _config((262, 118, 64, 86), (8, 8, 8, 8), 8, 2, 8)
    assert [len(r) for r in config.x_partition().ranges] == [33] * 6 + [32] * 2
    params, x, g = _inputs(config, 24)
    ours = _ours(config, params, x, g)
    _check(_compare(ours, _reference(config, params, x, g)))
    del ours
    _free()


def test_c4_paper_channels_1_20_1():
    # the paper-like variant: 1 input channel, width 20,
    # 1 output channel, on a 2-rank split of a 128 x 118 x 64 x 86 grid
    config = _config((128, 118, 64, 86), (8, 8, 8, 8), 20, 2, 2, cin=1, cout=1)
    params, x, g = _inputs(config, 25)
    ours = _ours(config, params, x, g)
    _check(_compare(ours, _reference(config, params, x, g)))
    del ours
    _free()


def test_c5_weak_p2_rank_geometry():
    config = _config((128, 64, 64, 32), (8, 8, 8, 8), 20, 2, 2)
    params, x, g = _inputs(config, 26)
    ours = _ours(config, params, x, g)
    _check(_compare(ours, _reference(config, params, x, g)))
    del ours
    _free()
