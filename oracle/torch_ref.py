"""TEST INFRASTRUCTURE ONLY: float64 torch.fft restatement of the reference FNO
(the GPU-scale oracle).

The numpy oracle (``fno_oracle.py``) is practical up to C2 on a CPU; C3
(128^3 x 32) and the CO2 grid C4 (262 x 118 x 64 x 86) need the same
algorithm on the GPU.  This module restates the reference's algorithm with
torch.fft (cuFFT, complex128) and torch.einsum in float64, independently of
libdfno: full-length FFTs along each dim followed by the gather of the
retained modes, per-mode einsum, zero-pad, full-length inverse FFTs and the
real part -- exactly the reference's stages, run dim by dim (the 4-D DFT is
separable, so truncating after each 1-D transform equals truncating the fftn
output) and channel-chunked so C3/C4 fit in HBM.

Reference lines followed:
  * block forward  fft_dims(yzt) -> truncate -> fft_dims(x) -> truncate ->
    einsum_spectral -> pad -> ifft_dims(x) -> pad -> ifft_dims(yzt) -> .real
                                                  d/fno.py:328-343, d/oracle.py:43-58
  * retained set {0..m-1} u {N-m..N-1}            d/spectral.py:59-66
  * einsum "bixyzt,ioxyzt->boxyzt"               d/tensor.py:231-255
  * encoder / decoder mixing + activation         d/fno.py:286-306, d/tensor.py:210-228
  * erf GELU and its derivative                   d/fno.py:41-55
  * block adjoint: fft/N, truncate, gW = sum_b conj(S) D, dX = sum_o D conj(W),
    pad, N * ifft                                  d/fno.py:415-465
  * whole backward                                d/fno.py:468-509

It is pinned to the numpy oracle and to the reference-generated golden
fixtures in tests/test_torch_ref.py (CPU) and tests/test_gpu_fullsize.py (GPU,
C1 cross-check inside the same test as the C2/C3/C4 comparisons).
"""

from __future__ import annotations

import math

import torch

_INV_SQRT2 = 1.0 / math.sqrt(2.0)
_INV_SQRT2PI = 1.0 / math.sqrt(2.0 * math.pi)
F64 = torch.float64
C128 = torch.complex128


def keep(n: int, m: int, device) -> torch.Tensor:
    """Retained positions along one dim (d/spectral.py:59-66)."""
    if 2 * m >= n:
        return torch.arange(n, device=device)
    return torch.cat([torch.arange(m, device=device), torch.arange(n - m, n, device=device)])


def act(kind: str, h: torch.Tensor) -> torch.Tensor:
    """d/fno.py:41-46"""
    if kind == "gelu":
        return 0.5 * h * (1.0 + torch.special.erf(h * _INV_SQRT2))
    if kind == "relu":
        return torch.clamp_min(h, 0)
    return h.clone()


def act_grad(kind: str, h: torch.Tensor) -> torch.Tensor:
    """d/fno.py:48-55"""
    if kind == "gelu":
        return 0.5 * (1.0 + torch.special.erf(h * _INV_SQRT2)) + h * _INV_SQRT2PI * torch.exp(-0.5 * h * h)
    if kind == "relu":
        return (h > 0).to(h.dtype)
    return torch.ones_like(h)


def mix(x: torch.Tensor, w: torch.Tensor, kind: str | None = None, chunk: int = 4) -> torch.Tensor:
    """Y[b,o,...] = sum_i X[b,i,...] W[i,o] (d/tensor.py:225-227), optionally
    followed by the activation; accumulated input channel by input channel so
    no (b, c, points) temporary larger than one output is made."""
    b, ci = x.shape[:2]
    co = w.shape[1]
    out = torch.empty((b, co) + tuple(x.shape[2:]), dtype=F64, device=x.device)
    for o0 in range(0, co, chunk):
        o1 = min(co, o0 + chunk)
        acc = torch.zeros((b, o1 - o0) + tuple(x.shape[2:]), dtype=F64, device=x.device)
        for i in range(ci):
            acc += x[:, i:i + 1].to(F64) * w[i, o0:o1].to(F64).view(1, -1, *([1] * (x.dim() - 2)))
        out[:, o0:o1] = act(kind, acc) if kind else acc
    return out


def mix_weight_grad(a: torch.Tensor, g: torch.Tensor) -> torch.Tensor:
    """gW[i,o] = sum_{b,points} a[b,i] g[b,o] (d/fno.py:405-408)."""
    af = a.reshape(a.shape[0], a.shape[1], -1)
    gf = g.reshape(g.shape[0], g.shape[1], -1)
    return torch.einsum("bip,bop->io", af, gf)


def mix_input_grad(g: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """dX[b,i] = sum_o g[b,o] W[i,o] (d/fno.py:409-412)."""
    return mix(g, w.t().contiguous())


def _fft_trunc(a: torch.Tensor, modes, chunk: int) -> torch.Tensor:
    """fft over (x, y, z, t) of real a (b, c, X, Y, Z, T), keeping the retained
    set after each 1-D transform; returns (b, c, r_x, r_y, r_z, r_t) complex128."""
    dev = a.device
    ks = [keep(n, m, dev) for n, m in zip(a.shape[2:], modes)]
    outs = []
    for c0 in range(0, a.shape[1], chunk):
        z = a[:, c0:c0 + chunk].to(F64)
        for dim in (5, 4, 3, 2):  # t, z, y, x
            z = torch.fft.fft(z, dim=dim).index_select(dim, ks[dim - 2])
        outs.append(z)
    return torch.cat(outs, dim=1)


def _pad_ifft(s: torch.Tensor, full, modes, chunk: int) -> torch.Tensor:
    """Zero-pad the retained set into the full spectrum and ifft over
    (x, y, z, t) (1/N per dim); returns the real part (b, c, X, Y, Z, T)."""
    dev = s.device
    ks = [keep(n, m, dev) for n, m in zip(full, modes)]
    outs = torch.empty((s.shape[0], s.shape[1]) + tuple(full), dtype=F64, device=dev)
    for c0 in range(0, s.shape[1], chunk):
        z = s[:, c0:c0 + chunk]
        for dim in (2, 3, 4, 5):  # x, y, z, t
            shape = list(z.shape)
            shape[dim] = full[dim - 2]
            p = torch.zeros(shape, dtype=C128, device=dev)
            p.index_copy_(dim, ks[dim - 2], z)
            z = torch.fft.ifft(p, dim=dim)
            del p
        outs[:, c0:c0 + chunk] = z.real
        del z
    return outs


def spectral_block(a: torch.Tensor, w: torch.Tensor, modes, chunk: int = 2):
    """(pre_activation, spec_in) of one block on the whole domain (d/oracle.py:43-58)."""
    spec = _fft_trunc(a, modes, chunk)
    y = torch.einsum("bixyzt,ioxyzt->boxyzt", spec, w.to(C128))
    return _pad_ifft(y, a.shape[2:], modes, chunk), spec


def spectral_block_adjoint(g: torch.Tensor, w: torch.Tensor, spec_in: torch.Tensor, modes, chunk: int = 2):
    """(grad input, grad W) of one block given the gradient of its output
    (d/fno.py:426-465 with the four dims merged: fft / N, truncate, gW / dX
    (d/fno.py:415-423), pad, N * ifft)."""
    full = tuple(g.shape[2:])
    n = math.prod(full)
    d = _fft_trunc(g, modes, chunk) / n
    gw = torch.einsum("bixyzt,boxyzt->ioxyzt", spec_in.conj(), d)
    dx = torch.einsum("boxyzt,ioxyzt->bixyzt", d, w.to(C128).conj())
    return _pad_ifft(dx, full, modes, chunk) * n, gw


def forward(x, we, wd, blocks, modes, kind="gelu"):
    """Serial forward with cache (d/oracle.py:25-62 / d/fno.py:350-380).
    Caches pre-activations and spec_in only."""
    enc_pre = mix(x, we)
    a = act(kind, enc_pre)
    pres, specs = [], []
    for w in blocks:
        pre, spec = spectral_block(a, w, modes)
        del a
        pres.append(pre)
        specs.append(spec)
        a = act(kind, pre)
    dec_pre = mix(a, wd)
    del a
    y = act(kind, dec_pre)
    return y, {"x": x, "enc_pre": enc_pre, "pres": pres, "specs": specs, "dec_pre": dec_pre}


def backward(g, we, wd, blocks, modes, cache, kind="gelu"):
    """Serial reverse mode (d/fno.py:468-509): (gx, gwe, gwd, [gW per block]).
    Consumes (frees) the cache's pre-activations as it goes."""
    gd = g.to(F64) * act_grad(kind, cache.pop("dec_pre"))
    pres = cache["pres"]
    a_last = act(kind, pres[-1]) if blocks else act(kind, cache["enc_pre"])
    gwd = mix_weight_grad(a_last, gd)
    del a_last
    ga = mix_input_grad(gd, wd.to(F64))
    del gd
    gws = [None] * len(blocks)
    for i in reversed(range(len(blocks))):
        ga *= act_grad(kind, pres[i])
        pres[i] = None
        ga, gws[i] = spectral_block_adjoint(ga, blocks[i], cache["specs"][i], modes)
    ga *= act_grad(kind, cache.pop("enc_pre"))
    gwe = mix_weight_grad(cache["x"].to(F64), ga)
    gx = mix_input_grad(ga, we.to(F64))
    return gx, gwe, gwd, gws


def rel_err(a: torch.Tensor, b: torch.Tensor) -> float:
    """max|a-b| / max(max|a|, max|b|) (d/bench.py:83-85), computed on the
    device in float64."""
    a = a.to(b.device)
    if a.is_complex() or b.is_complex():
        a, b = a.to(C128), b.to(C128)
    else:
        a, b = a.to(F64), b.to(F64)
    den = max(a.abs().max().item(), b.abs().max().item())
    return 0.0 if den == 0 else (a - b).abs().max().item() / den
