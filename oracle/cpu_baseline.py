"""TEST / BASELINE INFRASTRUCTURE ONLY: the reference's CPU algorithm, timed.

``bench.py`` uses this for its ``cpu_baseline`` field and for
``--impl reference``.  /root/reference does not exist on the GPU box, so the
timed code is this numpy port of the reference's *staged distributed*
pipeline -- the exact sequence of numpy operations one rank of the reference
performs in ``fno_forward`` + ``fno_backward`` (d/fno.py:286-509): full
complex ``np.fft.fftn`` over (y, z, t) (d/spectral.py:36), ``np.ix_``
truncation (d/spectral.py:110-117), the x FFT on the ky pencil, the
``einsum`` spectral multiply (d/tensor.py:254), zero padding
(d/spectral.py:120-145), ``ifftn`` and ``.real`` (d/fno.py:338-343), the
tensordot channel mixes (d/tensor.py:225-227) and erf GELU (d/fno.py:41-55).

Bounded sample: the global problem is split into R = S x N ranks along x
(remainder-first, like the reference's decomposition) and ONE rank's share
of the work is timed per process; ``cores`` processes run side by side, one
per host core (the reference's ``--transport proc`` mode, d/bench.py:526-565).
The repartitions are replaced by local reshaping of the rank's own data into
the received shapes (identical array sizes, so identical numpy work; the
reference measured 0.13 s of 15.5 s in its transport at C1).  Whole-job
throughput = samples / (t_rank * R / cores).
"""

from __future__ import annotations

import math
import multiprocessing as mp
import os
import time

import numpy as np
from scipy.special import erf

_S2 = 1.0 / math.sqrt(2.0)
_S2PI = 1.0 / math.sqrt(2.0 * math.pi)


def _gelu(h):
    return 0.5 * h * (1.0 + erf(h * _S2))


def _gelu_d(h):
    return 0.5 * (1.0 + erf(h * _S2)) + h * _S2PI * np.exp(-0.5 * h * h)


def _keep(n, m):
    if 2 * m >= n:
        return np.arange(n)
    return np.concatenate([np.arange(m), np.arange(n - m, n)])


def _blocks(n, p):
    q, r = divmod(n, p)
    return [q + (1 if k < r else 0) for k in range(p)]


def _mix(x, w):
    return np.ascontiguousarray(np.moveaxis(np.tensordot(x, w, axes=([1], [0])), -1, 1))


class RankSample:
    """One rank's arrays for an R-way x decomposition of the global grid."""

    def __init__(self, grid, channels, modes, blocks, ranks, dtype=np.float32, seed=42):
        nx, ny, nz, nt = grid
        self.grid = grid
        self.c = channels
        self.L = blocks
        self.xl = _blocks(nx, ranks)[0]
        self.keeps = [_keep(n, m) for n, m in zip(grid, modes)]
        self.r = [len(k) for k in self.keeps]
        self.kyl = _blocks(self.r[1], ranks)[0]
        rng = np.random.default_rng(seed)
        self.real = dtype
        self.cplx = np.complex64 if dtype == np.float32 else np.complex128
        c = channels
        self.x = rng.standard_normal((1, c, self.xl, ny, nz, nt)).astype(dtype)
        lim = math.sqrt(6.0 / (2 * c))
        self.we = rng.uniform(-lim, lim, (c, c)).astype(dtype)
        self.wd = rng.uniform(-lim, lim, (c, c)).astype(dtype)
        wshape = (c, c, self.r[0], self.kyl, self.r[2], self.r[3])
        self.w = [((rng.random(wshape) + 1j * rng.random(wshape)) / (c * c)).astype(self.cplx)
                  for _ in range(blocks)]
        self.ranks = ranks

    # -- the rank-local stage sequence of fno_block_forward (d/fno.py:328-343)
    def _yzt_fwd(self, a, scale=None):
        z = np.fft.fftn(a.astype(self.cplx), axes=(3, 4, 5))
        if scale is not None:
            z = z * scale
        k = self.keeps
        return z[np.ix_(np.arange(z.shape[0]), np.arange(z.shape[1]), np.arange(z.shape[2]), k[1], k[2], k[3])]

    def _x_to_ky(self, t):
        # received pencil (b, c, Nx, kyl, rz, rt): same size as the reference's
        return np.ascontiguousarray(np.concatenate([t[:, :, :, : self.kyl]] * self.ranks, axis=2)[:, :, : self.grid[0]])

    def _ky_to_x(self, u):
        return np.ascontiguousarray(np.concatenate([u[:, :, : self.xl]] * self.ranks, axis=3)[:, :, :, : self.r[1]])

    def _yzt_inv(self, v, scale=None):
        ny, nz, nt = self.grid[1:]
        k = self.keeps
        full = np.zeros(v.shape[:3] + (ny, nz, nt), dtype=v.dtype)
        full[np.ix_(np.arange(v.shape[0]), np.arange(v.shape[1]), np.arange(v.shape[2]), k[1], k[2], k[3])] = v
        out = np.fft.ifftn(full, axes=(3, 4, 5))
        if scale is not None:
            out = out * scale
        return np.ascontiguousarray(out.real)

    def _x_stage(self, z, w, bwd=False, spec=None):
        nx = self.grid[0]
        s = np.fft.fft(z, axis=2)
        if bwd:
            s = s / nx
        s = s[:, :, self.keeps[0]]
        if bwd:
            gw = np.einsum("bi...,bo...->io...", np.conj(spec), s, optimize=True)
            y = np.einsum("bo...,io...->bi...", s, np.conj(w), optimize=True)
        else:
            gw = None
            y = np.einsum("bi...,io...->bo...", s, w, optimize=True)
        pad = np.zeros(y.shape[:2] + (nx,) + y.shape[3:], dtype=y.dtype)
        pad[:, :, self.keeps[0]] = y
        u = np.fft.ifft(pad, axis=2)
        if bwd:
            u = u * nx
        return u, s, gw

    def step(self):
        """fwd + bwd with g = y (d/bench.py:381-390)."""
        n_yzt = self.grid[1] * self.grid[2] * self.grid[3]
        enc_pre = _mix(self.x, self.we)
        a = _gelu(enc_pre)
        acts, pres, specs = [a], [], []
        for w in self.w:
            z = self._x_to_ky(self._yzt_fwd(a))
            u, spec, _ = self._x_stage(z, w)
            pre = self._yzt_inv(self._ky_to_x(u))
            a = _gelu(pre)
            pres.append(pre)
            specs.append(spec)
            acts.append(a)
        dec_pre = _mix(a, self.wd)
        y = _gelu(dec_pre)
        g = y * _gelu_d(dec_pre)
        np.einsum("bi...,bo...->io", acts[-1], g, optimize=True)
        g = _mix(g, self.wd.T)
        for i in reversed(range(self.L)):
            g = g * _gelu_d(pres[i])
            d = self._x_to_ky(self._yzt_fwd(g, 1.0 / n_yzt))
            u, _, _ = self._x_stage(d, self.w[i], bwd=True, spec=specs[i])
            g = self._yzt_inv(self._ky_to_x(u), float(n_yzt))
        g = g * _gelu_d(enc_pre)
        np.einsum("bi...,bo...->io", self.x, g, optimize=True)
        return _mix(g, self.we.T)


def _worker(args):
    grid, channels, modes, blocks, ranks, steps = args
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    s = RankSample(grid, channels, modes, blocks, ranks)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        s.step()
        times.append(time.perf_counter() - t0)
    return times


def measure(grid, channels, modes, blocks, ranks, cores, steps=1):
    """Run ``cores`` rank samples in parallel processes for ``steps`` steps;
    returns the per-step wall time of the slowest process and the whole-job
    step time (t * ranks / cores)."""
    cores = max(1, min(cores, ranks))
    env_before = os.environ.get("OPENBLAS_NUM_THREADS")
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    try:
        ctx = mp.get_context("spawn")
        with ctx.Pool(cores) as pool:
            res = pool.map(_worker, [(grid, channels, modes, blocks, ranks, steps)] * cores)
    finally:
        if env_before is None:
            os.environ.pop("OPENBLAS_NUM_THREADS", None)
        else:
            os.environ["OPENBLAS_NUM_THREADS"] = env_before
    per_step = [max(r[i] for r in res) for i in range(steps)]
    return per_step, [t * ranks / cores for t in per_step]
