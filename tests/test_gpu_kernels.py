"""Kernel-level parity through the C ABI (include/dfno.h) against numpy
restatements of the reference stages, at the production shapes, plus
size-independent properties at the full benchmark size (C2: 64^3 x 32,
width 20, m = 8).

Stage references: fft_dims + truncate (d/fno.py:328-329), pad + ifft + real
(d/fno.py:338-343), fft_x / einsum / ifft_x (d/fno.py:331-336), and their
adjoints (d/fno.py:445-464)."""

import ctypes

import numpy as np
import pytest
import torch

from oracle import fno_oracle as O
from paper_2211_12709_b200 import _lib
from paper_2211_12709_b200.partition import block_starts

pytestmark = pytest.mark.gpu


def geom(grid, modes, c=2, batch=1, nranks=1, rank=0, dtype=_lib.F32, act=_lib.ACT_GELU, cin=None, cout=None):
    ret = tuple(min(2 * m, n) for n, m in zip(grid, modes))
    return _lib.make_geom(batch=batch, c_in=cin or c, c=c, c_out=cout or c, grid=grid, modes=modes, retained=ret,
                          nranks=nranks, rank=rank, dtype=dtype, act=act, x_starts=block_starts(grid[0], nranks),
                          ky_starts=block_starts(ret[1], nranks))


def call(name, *args):
    lib = _lib.load()
    _lib.check(getattr(lib, name)(*args), name)


def tol(dtype):
    # fp32: SIMT fp32 or tcgen05 3xTF32 (round-to-nearest split, ~2^-22 per product)
    return 1e-12 if dtype == _lib.F64 else 5e-6


SHAPES = [((4, 64, 64, 32), (8, 8, 8, 8)), ((3, 32, 32, 16), (8, 8, 8, 8)), ((2, 30, 20, 22), (4, 8, 8, 8)),
          ((2, 16, 16, 8), (4, 4, 4, 3)), ((2, 118, 64, 86), (8, 8, 8, 8)), ((2, 20, 12, 36), (8, 4, 5, 8)),
          ((2, 13, 10, 15), (4, 4, 4, 7)), ((1, 128, 128, 32), (8, 8, 8, 8)), ((1, 118, 64, 86), (8, 8, 6, 8))]


@pytest.mark.parametrize("grid,modes", SHAPES)
@pytest.mark.parametrize("dtype", [_lib.F32, _lib.F64])
@pytest.mark.parametrize("mode", [_lib.SRC_RAW, _lib.SRC_ACT, _lib.SRC_GRAD])
def test_yzt_forward(grid, modes, dtype, mode):
    c, b = 2, 1
    g = geom(grid, modes, c=c, batch=b, dtype=dtype)
    rdt = torch.float32 if dtype == _lib.F32 else torch.float64
    cdt = torch.complex64 if dtype == _lib.F32 else torch.complex128
    rng = np.random.default_rng(0)
    a = rng.standard_normal((b, c) + grid)
    pre = rng.standard_normal((b, c) + grid)
    src = torch.tensor(a, dtype=rdt, device="cuda")
    pr = torch.tensor(pre, dtype=rdt, device="cuda")
    ry, rz, rt = g.ry, g.rz, g.rt
    out = torch.empty((b, c, grid[0], ry, rz, rt), dtype=cdt, device="cuda")
    scale = 0.37
    call("dfno_dft_yzt_fwd", ctypes.byref(g), _lib.ptr(src), _lib.ptr(pr), mode, scale, _lib.ptr(out), None)
    a64 = src.double().cpu().numpy()
    if mode == _lib.SRC_ACT:
        a64 = O.act("gelu", a64)
    elif mode == _lib.SRC_GRAD:
        a64 = a64 * O.act_grad("gelu", pr.double().cpu().numpy())
    want = scale * O.yzt_truncated(a64, modes)
    assert O.rel_err(out.cpu().numpy(), want) < tol(dtype) * (4 if mode != _lib.SRC_RAW else 1)


@pytest.mark.parametrize("grid,modes", SHAPES)
@pytest.mark.parametrize("dtype", [_lib.F32, _lib.F64])
def test_yzt_inverse(grid, modes, dtype):
    c, b = 2, 1
    g = geom(grid, modes, c=c, batch=b, dtype=dtype)
    rdt = torch.float32 if dtype == _lib.F32 else torch.float64
    cdt = torch.complex64 if dtype == _lib.F32 else torch.complex128
    ry, rz, rt = g.ry, g.rz, g.rt
    rng = np.random.default_rng(1)
    v = rng.standard_normal((b, c, grid[0], ry, rz, rt)) + 1j * rng.standard_normal((b, c, grid[0], ry, rz, rt))
    vin = torch.tensor(v, dtype=cdt, device="cuda")
    out = torch.empty((b, c) + grid, dtype=rdt, device="cuda")
    n = grid[1] * grid[2] * grid[3]
    call("dfno_dft_yzt_inv", ctypes.byref(g), _lib.ptr(vin), 1.0 / n, _lib.ptr(out), None)
    keeps = [O.keep(grid[1], modes[1]), O.keep(grid[2], modes[2]), O.keep(grid[3], modes[3])]
    full = np.zeros((b, c) + grid, dtype=complex)
    full[np.ix_(np.arange(b), np.arange(c), np.arange(grid[0]), *keeps)] = vin.cpu().numpy()
    want = np.fft.ifftn(full, axes=(3, 4, 5)).real
    assert O.rel_err(out.cpu().numpy(), want) < tol(dtype)


@pytest.mark.parametrize("nx,mx,P", [(64, 8, 1), (64, 8, 4), (512, 8, 8), (33, 8, 3), (9, 2, 3), (9, 5, 3)])
@pytest.mark.parametrize("dtype", [_lib.F32, _lib.F64])
@pytest.mark.parametrize("variant", ["fused", "workspace"])
def test_xspec_forward_backward(nx, mx, P, dtype, variant):
    c, b = 4 if variant == "fused" else 5, 2
    grid, modes = (nx, 16, 16, 16), (mx, 8, 8, 8)
    rdt = torch.float32 if dtype == _lib.F32 else torch.float64
    cdt = torch.complex64 if dtype == _lib.F32 else torch.complex128
    rng = np.random.default_rng(2)
    rank = P - 1
    g = geom(grid, modes, c=c, batch=b, nranks=P, rank=rank, dtype=dtype)
    rx, ry, rz, rt = g.rx, g.ry, g.rz, g.rt
    ks = block_starts(ry, P)
    kyl = ks[rank + 1] - ks[rank]
    xs = block_starts(nx, P)
    # global pencil Z[b][c][x][kyl][rz][rt], packed KX (peer-major over x blocks)
    z = rng.standard_normal((b, c, nx, kyl, rz, rt)) + 1j * rng.standard_normal((b, c, nx, kyl, rz, rt))
    packed = np.concatenate([z[:, :, xs[p]:xs[p + 1]].reshape(-1) for p in range(P)])
    w = rng.standard_normal((c, c, rx, kyl, rz, rt)) + 1j * rng.standard_normal((c, c, rx, kyl, rz, rt))
    kin = torch.tensor(packed, dtype=cdt, device="cuda")
    wt = torch.tensor(w, dtype=cdt, device="cuda")
    spec = torch.empty((b, c, rx, kyl, rz, rt), dtype=cdt, device="cuda")
    kout = torch.empty_like(kin)
    ws = ctypes.c_int64()
    call("dfno_xspec_workspace", ctypes.byref(g), ctypes.byref(ws))
    work = torch.empty(ws.value, dtype=torch.uint8, device="cuda")
    if variant == "fused":
        call("dfno_xspec_fwd", ctypes.byref(g), _lib.ptr(kin), _lib.ptr(wt), _lib.ptr(spec), _lib.ptr(kout), None)
    else:
        call("dfno_xspec_fwd_ws", ctypes.byref(g), _lib.ptr(kin), _lib.ptr(wt), _lib.ptr(spec), _lib.ptr(kout),
             _lib.ptr(work), None)
    kx = O.keep(nx, mx)
    s_ref = np.fft.fft(z, axis=2)[:, :, kx]
    y = np.einsum("bi...,io...->bo...", s_ref, w)
    pad = np.zeros_like(z)
    pad[:, :, kx] = y
    u = np.fft.ifft(pad, axis=2)
    u_packed = np.concatenate([u[:, :, xs[p]:xs[p + 1]].reshape(-1) for p in range(P)])
    t = tol(dtype) * 10
    assert O.rel_err(spec.cpu().numpy(), s_ref) < t
    assert O.rel_err(kout.cpu().numpy(), u_packed) < t
    # backward
    gw = torch.empty_like(wt)
    if variant == "fused":
        call("dfno_xspec_bwd", ctypes.byref(g), _lib.ptr(kin), _lib.ptr(spec), _lib.ptr(wt), _lib.ptr(gw),
             _lib.ptr(kout), None)
    else:
        call("dfno_xspec_bwd_ws", ctypes.byref(g), _lib.ptr(kin), _lib.ptr(spec), _lib.ptr(wt), _lib.ptr(gw),
             _lib.ptr(kout), _lib.ptr(work), None)
    d = np.fft.fft(z, axis=2)[:, :, kx] / nx
    gw_ref = np.einsum("bi...,bo...->io...", np.conj(spec.cpu().numpy().astype(complex)), d)
    dx = np.einsum("bo...,io...->bi...", d, np.conj(w))
    pad = np.zeros_like(z)
    pad[:, :, kx] = dx
    u = np.fft.ifft(pad, axis=2) * nx
    u_packed = np.concatenate([u[:, :, xs[p]:xs[p + 1]].reshape(-1) for p in range(P)])
    assert O.rel_err(gw.cpu().numpy(), gw_ref) < t
    assert O.rel_err(kout.cpu().numpy(), u_packed) < t


@pytest.mark.parametrize("dtype", [_lib.F32, _lib.F64])
@pytest.mark.parametrize("cin,cout", [(20, 20), (1, 20), (20, 3), (7, 5)])
def test_mix_forward_backward(dtype, cin, cout):
    rdt = torch.float32 if dtype == _lib.F32 else torch.float64
    b, npts = 2, 4099
    g = geom((8, 8, 8, 4), (2, 2, 2, 2), c=20, batch=b, dtype=dtype, cin=cin, cout=cout)
    rng = np.random.default_rng(3)
    x = torch.tensor(rng.standard_normal((b, cin, npts)), dtype=rdt, device="cuda")
    w = torch.tensor(rng.standard_normal((cin, cout)), dtype=rdt, device="cuda")
    pre = torch.empty((b, cout, npts), dtype=rdt, device="cuda")
    post = torch.empty_like(pre)
    for src_act in (0, 1):
        call("dfno_mix_fwd", ctypes.byref(g), npts, cin, cout, _lib.ptr(x), src_act, _lib.ptr(w), _lib.ptr(pre),
             _lib.ptr(post), None)
        xs = x.double().cpu().numpy()
        if src_act:
            xs = O.act("gelu", xs)
        want = np.einsum("bip,io->bop", xs, w.double().cpu().numpy())
        t = 1e-12 if dtype == _lib.F64 else 1e-5
        assert O.rel_err(pre.cpu().numpy(), want) < t
        assert O.rel_err(post.cpu().numpy(), O.act("gelu", want)) < t
        gout = torch.tensor(rng.standard_normal((b, cout, npts)), dtype=rdt, device="cuda")
        n = ctypes.c_int64()
        k = ctypes.c_int()
        call("dfno_mix_bwd_partials", ctypes.byref(g), npts, cin, cout, ctypes.byref(n), ctypes.byref(k))
        parts = torch.empty(n.value, dtype=rdt, device="cuda")
        gin = torch.empty_like(x)
        call("dfno_mix_bwd", ctypes.byref(g), npts, cin, cout, _lib.ptr(gout), _lib.ptr(pre), _lib.ptr(x), src_act,
             _lib.ptr(w), _lib.ptr(gin), _lib.ptr(parts), None)
        gw = torch.empty((cin, cout), dtype=rdt, device="cuda")
        call("dfno_reduce_partials", ctypes.byref(g), k.value, cin * cout, _lib.ptr(parts), _lib.ptr(gw), None)
        gp = gout.double().cpu().numpy() * O.act_grad("gelu", pre.double().cpu().numpy())
        assert O.rel_err(gin.cpu().numpy(), np.einsum("bop,io->bip", gp, w.double().cpu().numpy())) < t
        assert O.rel_err(gw.cpu().numpy(), np.einsum("bip,bop->io", xs, gp)) < t * 10


@pytest.mark.parametrize("cin,cout", [(20, 20), (1, 20), (20, 3)])
@pytest.mark.parametrize("with_post", [True, False])
def test_mix_forward_tma_paths(cin, cout, with_post):
    """npts % 4 == 0 selects the TMA-fed mix kernel (TMA loads, double-buffered
    TMEM accumulators, TMA stores; single-buffered staging when the output
    activation is also written); odd tails exercise the clipped last tile."""
    b, npts = 2, 4100
    g = geom((8, 8, 8, 4), (2, 2, 2, 2), c=20, batch=b, dtype=_lib.F32, cin=cin, cout=cout)
    rng = np.random.default_rng(5)
    x = torch.tensor(rng.standard_normal((b, cin, npts)), dtype=torch.float32, device="cuda")
    w = torch.tensor(rng.standard_normal((cin, cout)), dtype=torch.float32, device="cuda")
    pre = torch.full((b, cout, npts), float("nan"), device="cuda")
    post = torch.full_like(pre, float("nan")) if with_post else None
    for src_act in (0, 1):
        call("dfno_mix_fwd", ctypes.byref(g), npts, cin, cout, _lib.ptr(x), src_act, _lib.ptr(w), _lib.ptr(pre),
             _lib.ptr(post) if with_post else None, None)
        xs = x.double().cpu().numpy()
        if src_act:
            xs = O.act("gelu", xs)
        want = np.einsum("bip,io->bop", xs, w.double().cpu().numpy())
        assert O.rel_err(pre.cpu().numpy(), want) < 1e-5
        if with_post:
            assert O.rel_err(post.cpu().numpy(), O.act("gelu", want)) < 1e-5


def test_mix_backward_fused_src_activation_derivative():
    """src_act = 2: gin comes back multiplied by act'(src) (the decoder backward
    fused with the last block's activation derivative); same weight gradient
    as src_act = 1."""
    b, npts, cin, cout = 2, 4100, 20, 20
    g = geom((8, 8, 8, 4), (2, 2, 2, 2), c=20, batch=b, dtype=_lib.F32, cin=cin, cout=cout)
    rng = np.random.default_rng(6)
    src = torch.tensor(rng.standard_normal((b, cin, npts)), dtype=torch.float32, device="cuda")
    pre = torch.tensor(rng.standard_normal((b, cout, npts)), dtype=torch.float32, device="cuda")
    gout = torch.tensor(rng.standard_normal((b, cout, npts)), dtype=torch.float32, device="cuda")
    w = torch.tensor(rng.standard_normal((cin, cout)), dtype=torch.float32, device="cuda")
    n, k = ctypes.c_int64(), ctypes.c_int()
    call("dfno_mix_bwd_partials", ctypes.byref(g), npts, cin, cout, ctypes.byref(n), ctypes.byref(k))
    out = {}
    for sa in (1, 2):
        parts = torch.empty(n.value, device="cuda")
        gin = torch.empty_like(src)
        call("dfno_mix_bwd", ctypes.byref(g), npts, cin, cout, _lib.ptr(gout), _lib.ptr(pre), _lib.ptr(src), sa,
             _lib.ptr(w), _lib.ptr(gin), _lib.ptr(parts), None)
        gw = torch.empty((cin, cout), device="cuda")
        call("dfno_reduce_partials", ctypes.byref(g), k.value, cin * cout, _lib.ptr(parts), _lib.ptr(gw), None)
        out[sa] = (gin.double().cpu().numpy(), gw.cpu().numpy())
    s64 = src.double().cpu().numpy()
    gp = gout.double().cpu().numpy() * O.act_grad("gelu", pre.double().cpu().numpy())
    gin_a = np.einsum("bop,io->bip", gp, w.double().cpu().numpy())
    assert O.rel_err(out[1][0], gin_a) < 1e-5
    assert O.rel_err(out[2][0], gin_a * O.act_grad("gelu", s64)) < 1e-5
    assert np.array_equal(out[1][1], out[2][1])


def test_full_size_round_trip_and_linearity():
    """C2 geometry (64^3 x 32, c = 20): size-independent properties.
    (1) band-limited round trip: yzt_inv(yzt_fwd(u)) == u for u made of
        retained modes only; (2) linearity of the forward transform."""
    grid, modes, c = (64, 64, 64, 32), (8, 8, 8, 8), 20
    g = geom(grid, modes, c=c, dtype=_lib.F32)
    rng = np.random.default_rng(4)
    shape = (1, c, 64, 16, 16, 16)
    vn = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    # the retained set is not closed under negation (frequency N-m is kept,
    # m is not; d/spectral.py:59-66): zero position j = m on every dim so the
    # real field's spectrum stays inside the retained set
    vn[:, :, :, 8] = 0
    vn[:, :, :, :, 8] = 0
    vn[..., 8] = 0
    v = torch.tensor(vn, dtype=torch.complex64, device="cuda")
    # a real field whose yzt spectrum is supported on retained modes: u = Re(ifft(pad(v)))
    u = torch.empty((1, c) + grid, dtype=torch.float32, device="cuda")
    call("dfno_dft_yzt_inv", ctypes.byref(g), _lib.ptr(v), 1.0, _lib.ptr(u), None)
    t1 = torch.empty(shape, dtype=torch.complex64, device="cuda")
    call("dfno_dft_yzt_fwd", ctypes.byref(g), _lib.ptr(u), None, _lib.SRC_RAW, 1.0, _lib.ptr(t1), None)
    u2 = torch.empty_like(u)
    n = 64 * 64 * 32
    call("dfno_dft_yzt_inv", ctypes.byref(g), _lib.ptr(t1), 1.0 / n, _lib.ptr(u2), None)
    torch.cuda.synchronize()
    assert float((u2 - u).abs().max() / u.abs().max()) < 1e-5
    # linearity
    a = torch.randn((1, c) + grid, device="cuda")
    bb = torch.randn((1, c) + grid, device="cuda")
    outs = []
    for src in (a, bb, 2.0 * a - 3.0 * bb):
        o = torch.empty(shape, dtype=torch.complex64, device="cuda")
        call("dfno_dft_yzt_fwd", ctypes.byref(g), _lib.ptr(src), None, _lib.SRC_RAW, 1.0, _lib.ptr(o), None)
        outs.append(o)
    lin = 2.0 * outs[0] - 3.0 * outs[1]
    assert float((outs[2] - lin).abs().max() / lin.abs().max()) < 1e-5


def test_full_size_adjoint_identity():
    """C2 geometry, the whole linear network (identity activation):
    <J x, g> == <x, J^T g> with J^T g from fno_backward -- a size-independent
    check of forward/backward consistency at the benchmark size."""
    import paper_2211_12709_b200 as P

    config = P.FnoConfig(64, 64, 64, 32, 20, 20, 20, P.ModeSpec.of_xyzt(8, 8, 8, 8), 4, "identity", "real32", 1)
    params = P.init_params(config, 42)
    x = P.DenseTensor(P.DATA_LABELS, torch.randn((1, 20, 64, 64, 64, 32), device="cuda"))
    g = P.DenseTensor(P.DATA_LABELS, torch.randn((1, 20, 64, 64, 64, 32), device="cuda"))

    def body(comm):
        cache = P.ForwardCache()
        y = P.fno_forward(comm, x, params, config, cache)
        gx, _ = P.fno_backward(comm, g, params, config, cache)
        return float((y.data.double() * g.data.double()).sum()), float((x.data.double() * gx.data.double()).sum())

    lhs, rhs = P.run_ranks(1, body)[0]
    assert abs(lhs - rhs) / abs(lhs) < 1e-4
