"""TEST INFRASTRUCTURE ONLY: numpy oracle of the distributed FNO.

Serial (undistributed) forward and its reverse-mode adjoint, plus the staged
per-rank pipeline the reference runs on P ranks (with explicit
repartitions), used to check the GPU path's outputs, gradients, packed
exchange layouts and communication counters.

Conventions pinned to the reference:
  * data (b, c, x, y, z, t), t fastest                  d/tensor.py:1-6, d/bench.py:57
  * a0 = act(X We); a_i+1 = act(block_i(a_i)); y = act(a_L Wd)   d/fno.py:364-379
  * erf GELU and its derivative                        d/fno.py:41-55
  * unnormalised fft, 1/N per dim on the inverse       d/spectral.py:1-9
  * retained set {0..m-1} u {N-m..N-1}                 d/spectral.py:59-66
  * block output = Re(ifftn(pad(einsum(trunc(fftn))))) d/oracle.py:43-58
  * gW = sum_b conj(S) D ; dX = sum_o D conj(W)         d/fno.py:415-423
  * backward scales fft/N, ifft*N                      d/fno.py:445-464
"""

from __future__ import annotations

import math

import numpy as np
from scipy.special import erf

_INV_SQRT2 = 1.0 / math.sqrt(2.0)
_INV_SQRT2PI = 1.0 / math.sqrt(2.0 * math.pi)
AXES = (2, 3, 4, 5)


# --------------------------------------------------------------------------
# elementary pieces
# --------------------------------------------------------------------------


def keep(n: int, m: int) -> np.ndarray:
    """Retained positions along a dim (reference d/spectral.py:59-66, d/oracle.py:19-22)."""
    if 2 * m >= n:
        return np.arange(n)
    return np.concatenate([np.arange(m), np.arange(n - m, n)])


def block_ranges(extent: int, parts: int) -> list:
    """Remainder-first contiguous blocks (reference d/partition.py:47-66)."""
    q, r = divmod(extent, parts)
    out, lo = [], 0
    for k in range(parts):
        hi = lo + q + (1 if k < r else 0)
        out.append((lo, hi))
        lo = hi
    return out


def act(kind: str, h: np.ndarray) -> np.ndarray:
    """reference d/fno.py:41-46"""
    if kind == "gelu":
        return 0.5 * h * (1.0 + erf(h * _INV_SQRT2))
    if kind == "relu":
        return np.maximum(h, 0)
    return h.copy()


def act_grad(kind: str, h: np.ndarray) -> np.ndarray:
    """reference d/fno.py:48-55"""
    if kind == "gelu":
        return 0.5 * (1.0 + erf(h * _INV_SQRT2)) + h * _INV_SQRT2PI * np.exp(-0.5 * h * h)
    if kind == "relu":
        return (h > 0).astype(h.dtype)
    return np.ones_like(h)


def mix(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Y[b,o,...] = sum_i X[b,i,...] W[i,o] (reference d/tensor.py:225-227)."""
    return np.moveaxis(np.tensordot(x, w, axes=([1], [0])), -1, 1)


def _mesh(b, c, keeps):
    return np.ix_(np.arange(b), np.arange(c), *keeps)


def spectral_block(a: np.ndarray, w: np.ndarray, modes) -> tuple:
    """One block on the whole domain: returns (pre_activation, spec_in).
    reference d/oracle.py:43-58 (serial form of d/fno.py:309-347)."""
    full = a.shape[2:]
    keeps = [keep(n, m) for n, m in zip(full, modes)]
    z = np.fft.fftn(a, axes=AXES)[_mesh(a.shape[0], a.shape[1], keeps)]
    y = np.einsum("bixyzt,ioxyzt->boxyzt", z, w, optimize=True)
    padded = np.zeros(y.shape[:2] + tuple(full), dtype=y.dtype)
    padded[_mesh(y.shape[0], y.shape[1], keeps)] = y
    return np.fft.ifftn(padded, axes=AXES).real, z


def spectral_block_adjoint(g: np.ndarray, w: np.ndarray, spec_in: np.ndarray, modes) -> tuple:
    """Adjoint of spectral_block given the gradient w.r.t. its output:
    returns (grad input, grad W).  reference d/fno.py:426-465 with all four
    dims merged: fft/N, truncate, gW / dX (d/fno.py:415-423), pad, N*ifft."""
    full = g.shape[2:]
    n = int(np.prod(full))
    keeps = [keep(nd, m) for nd, m in zip(full, modes)]
    d = np.fft.fftn(g, axes=AXES)[_mesh(g.shape[0], g.shape[1], keeps)] / n
    gw = np.einsum("bixyzt,boxyzt->ioxyzt", np.conj(spec_in), d, optimize=True)
    dx = np.einsum("boxyzt,ioxyzt->bixyzt", d, np.conj(w), optimize=True)
    padded = np.zeros(dx.shape[:2] + tuple(full), dtype=dx.dtype)
    padded[_mesh(dx.shape[0], dx.shape[1], keeps)] = dx
    return np.fft.ifftn(padded, axes=AXES).real * n, gw


# --------------------------------------------------------------------------
# whole network, serial
# --------------------------------------------------------------------------


def forward(x, we, wd, blocks, modes, kind="gelu", with_cache=False):
    """Serial forward (reference d/oracle.py:25-62 / d/fno.py:350-380)."""
    enc_pre = mix(x, we)
    a = act(kind, enc_pre)
    pres, specs = [], []
    for w in blocks:
        pre, spec = spectral_block(a, w, modes)
        pres.append(pre)
        specs.append(spec)
        a = act(kind, pre)
    dec_pre = mix(a, wd)
    y = act(kind, dec_pre)
    if not with_cache:
        return y
    return y, {"x": x, "enc_pre": enc_pre, "pres": pres, "specs": specs, "dec_pre": dec_pre}


def backward(g, we, wd, blocks, modes, cache, kind="gelu"):
    """Serial reverse mode (reference d/fno.py:468-509): returns
    (gx, gwe, gwd, [gW per block])."""
    gd = g * act_grad(kind, cache["dec_pre"])
    a_last = act(kind, cache["pres"][-1]) if blocks else act(kind, cache["enc_pre"])
    gwd = np.einsum("bi...,bo...->io", a_last, gd, optimize=True)
    ga = np.moveaxis(np.tensordot(gd, wd, axes=([1], [1])), -1, 1)
    gws = [None] * len(blocks)
    for i in reversed(range(len(blocks))):
        gp = ga * act_grad(kind, cache["pres"][i])
        ga, gws[i] = spectral_block_adjoint(gp, blocks[i], cache["specs"][i], modes)
    ge = ga * act_grad(kind, cache["enc_pre"])
    gwe = np.einsum("bi...,bo...->io", cache["x"], ge, optimize=True)
    gx = np.moveaxis(np.tensordot(ge, we, axes=([1], [1])), -1, 1)
    return gx, gwe, gwd, gws


# --------------------------------------------------------------------------
# staged per-rank pipeline (what the distributed reference does on P ranks)
# --------------------------------------------------------------------------


def yzt_truncated(a_local: np.ndarray, modes) -> np.ndarray:
    """fft_dims(a,(y,z,t)) + truncate (reference d/fno.py:328-329)."""
    ny, nz, nt = a_local.shape[3:]
    z = np.fft.fftn(a_local, axes=(3, 4, 5))
    return z[np.ix_(*(np.arange(s) for s in a_local.shape[:3]), keep(ny, modes[1]), keep(nz, modes[2]),
                    keep(nt, modes[3]))]


def pack_xk(t_local: np.ndarray, ky_parts) -> np.ndarray:
    """Peer-major XK send buffer of one rank: chunk p =
    t[:, :, :, ky in ky_parts[p]] flattened (include/dfno.h layouts;
    routing of reference d/partition.py:171-187)."""
    return np.concatenate([t_local[:, :, :, lo:hi].reshape(-1) for lo, hi in ky_parts])


def staged_forward_block(a_slabs: list, w: np.ndarray, modes, nx: int) -> tuple:
    """One block across P ranks with explicit repartitions (reference
    d/fno.py:309-347).  a_slabs[r] is rank r's x slab; w is the global
    weight.  Returns (pre slabs, spec_in shards, off-rank elements per
    repartition summed over ranks)."""
    P = len(a_slabs)
    ry = len(keep(a_slabs[0].shape[3], modes[1]))
    xparts = block_ranges(nx, P)
    kyparts = block_ranges(ry, P)
    t = [yzt_truncated(a, modes) for a in a_slabs]                     # (b,c,xl,ry,rz,rt)
    # x -> ky: rank q receives every rank's x slab restricted to its ky block
    pencils = [np.concatenate([t[r][:, :, :, lo:hi] for r in range(P)], axis=2) for lo, hi in kyparts]
    moved = sum(t[r][:, :, :, lo:hi].size for r in range(P) for q, (lo, hi) in enumerate(kyparts) if q != r)
    kx = keep(nx, modes[0])
    specs, outs = [], []
    for q, (lo, hi) in enumerate(kyparts):
        s = np.fft.fft(pencils[q], axis=2)[:, :, kx]
        specs.append(s)
        y = np.einsum("bi...,io...->bo...", s, w[:, :, :, lo:hi], optimize=True)
        padded = np.zeros(y.shape[:2] + (nx,) + y.shape[3:], dtype=y.dtype)
        padded[:, :, kx] = y
        outs.append(np.fft.ifft(padded, axis=2))
    # ky -> x
    pres = []
    ny, nz, nt = a_slabs[0].shape[3:]
    keeps = (keep(ny, modes[1]), keep(nz, modes[2]), keep(nt, modes[3]))
    for r, (xlo, xhi) in enumerate(xparts):
        v = np.concatenate([outs[q][:, :, xlo:xhi] for q in range(P)], axis=3)
        full = np.zeros(v.shape[:3] + (ny, nz, nt), dtype=v.dtype)
        full[np.ix_(*(np.arange(s) for s in v.shape[:3]), *keeps)] = v
        pres.append(np.fft.ifftn(full, axes=(3, 4, 5)).real)
    return pres, specs, moved


def predicted_volume(nx, ry, P, per_pair) -> int:
    """Off-rank elements per repartition, summed over ranks
    (reference d/fno.py:227-231)."""
    xs = block_ranges(nx, P)
    ks = block_ranges(ry, P)
    return per_pair * sum((xs[r][1] - xs[r][0]) * (ry - (ks[r][1] - ks[r][0])) for r in range(P))


def rel_err(a, b) -> float:
    """max|a-b| / max(max|a|, max|b|) (reference d/bench.py:83-85)."""
    a = np.asarray(a)
    b = np.asarray(b)
    scale = max(float(np.max(np.abs(a))) if a.size else 0.0, float(np.max(np.abs(b))) if b.size else 0.0, 1e-300)
    return float(np.max(np.abs(a - b))) / scale if a.size else 0.0
