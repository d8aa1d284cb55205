"""The reference's public layer functions, each against the oracle on the
GPU: encoder_forward / decoder_forward (d/fno.py:292-306), fno_block_forward
(d/fno.py:309-347) and fno_block_backward (d/fno.py:426-465), at P = 1 and
across a 3-rank decomposition (block input / gradient sliced along x, weight
gradients gathered along ky)."""

import numpy as np
import pytest
import torch

import paper_2211_12709_b200 as P
from oracle import fno_oracle as O

pytestmark = pytest.mark.gpu

GRID, MODES = (12, 10, 8, 6), (3, 4, 3, 2)


def _cfg(c, ranks, dtype):
    return P.FnoConfig(*GRID, c, c, c, P.ModeSpec.of_xyzt(*MODES), 1, "gelu", dtype, ranks)


@pytest.mark.parametrize("dtype,tol", [("real64", 1e-12), ("real32", 1e-5)])
@pytest.mark.parametrize("which", ["encoder", "decoder"])
def test_mixer_forward_against_oracle(which, dtype, tol):
    rng = np.random.default_rng(4)
    x = rng.standard_normal((2, 5) + GRID)
    w = rng.standard_normal((5, 3)) / 3
    tdt = torch.float64 if dtype == "real64" else torch.float32

    def body(comm):
        xd = P.DenseTensor(P.DATA_LABELS, torch.tensor(x, dtype=tdt, device="cuda"))
        wd = P.DenseTensor((P.DimLabel.C, P.DimLabel.CO), torch.tensor(w, dtype=tdt, device="cuda"))
        f = P.encoder_forward if which == "encoder" else P.decoder_forward
        return f(comm, xd, wd, "gelu").numpy()

    got = P.run_ranks(1, body)[0]
    xr = torch.tensor(x, dtype=tdt).double().numpy()
    want = O.act("gelu", O.mix(xr, torch.tensor(w, dtype=tdt).double().numpy()))
    assert O.rel_err(got, want) < tol


@pytest.mark.parametrize("dtype,tol,tolg", [("real64", 1e-11, 1e-11), ("real32", 1e-5, 1e-4)])
@pytest.mark.parametrize("ranks", [1, 3])
def test_block_forward_backward_against_oracle(ranks, dtype, tol, tolg):
    c = 4
    cfg = _cfg(c, ranks, dtype)
    rng = np.random.default_rng(8)
    a = rng.standard_normal((1, c) + GRID)
    g = rng.standard_normal((1, c) + GRID)
    params = P.init_params(cfg, 8, device="cpu")
    w = params.blocks[0]
    tdt = torch.float64 if dtype == "real64" else torch.float32
    xpart = cfg.x_partition()

    def body(comm):
        ad = P.slice_local(P.DenseTensor(P.DATA_LABELS, torch.tensor(a, dtype=tdt, device="cuda")), xpart, comm.rank)
        gd = P.slice_local(P.DenseTensor(P.DATA_LABELS, torch.tensor(g, dtype=tdt, device="cuda")), xpart, comm.rank)
        ws = P.shard_params(params, cfg, comm.rank).blocks[0]
        cache = P.BlockCache(None, None)
        pre = P.fno_block_forward(comm, ad, ws, cfg, cache=cache)
        gin, gw = P.fno_block_backward(comm, gd, ws, cache.spec_in, cfg)
        return pre.data.double().cpu(), gin.data.double().cpu(), gw.data.cpu()

    res = P.run_ranks(ranks, body)
    pre = torch.cat([r[0] for r in res], dim=2).numpy()
    gin = torch.cat([r[1] for r in res], dim=2).numpy()
    gw = torch.cat([r[2] for r in res], dim=3).numpy()
    ar = torch.tensor(a, dtype=tdt).double().numpy()
    gr = torch.tensor(g, dtype=tdt).double().numpy()
    wr = w.numpy().astype(np.complex128)
    want_pre, spec = O.spectral_block(ar, wr, MODES)
    want_gin, want_gw = O.spectral_block_adjoint(gr, wr, spec, MODES)
    assert O.rel_err(pre, want_pre) < tol
    assert O.rel_err(gin, want_gin) < tolg
    assert O.rel_err(gw, want_gw) < tolg


@pytest.mark.parametrize("shape", [(1, 20, 16, 16, 16, 16), (2, 5, 3, 7, 2, 3), (3, 4, 4, 2, 3, 1)])
@pytest.mark.parametrize("dtype", [torch.complex64, torch.complex128])
def test_einsum_spectral_against_numpy(shape, dtype):
    """einsum_spectral (reference tensor.py:231-255): complex64 runs libdfno's
    weight-streaming contraction (even and odd flattened mode counts, batch
    1-3), complex128 the device einsum; both against numpy in float64."""
    rng = np.random.default_rng(7)
    b, c = shape[:2]
    x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    w = rng.standard_normal((c, c) + shape[2:]) + 1j * rng.standard_normal((c, c) + shape[2:])
    labels = (P.DimLabel.B, P.DimLabel.C, P.DimLabel.KX, P.DimLabel.KY, P.DimLabel.KZ, P.DimLabel.KT)
    wl = (P.DimLabel.C, P.DimLabel.CO) + labels[2:]
    xt = P.DenseTensor(labels, torch.tensor(x, dtype=dtype, device="cuda"))
    wt = P.DenseTensor(wl, torch.tensor(w, dtype=dtype, device="cuda"))
    got = P.einsum_spectral(xt, wt).data.cpu().numpy()
    xr = torch.tensor(x, dtype=dtype).to(torch.complex128).numpy()
    wr = torch.tensor(w, dtype=dtype).to(torch.complex128).numpy()
    want = np.einsum("bi...,io...->bo...", xr, wr)
    tol = 1e-6 if dtype == torch.complex64 else 1e-13
    assert np.abs(got - want).max() / np.abs(want).max() < tol
