"""Pin the float64 torch.fft restatement (oracle/torch_ref.py, the GPU-scale
oracle for C2/C3/C4) to the reference's own golden vectors and to the numpy
oracle, on CPU.  The GPU tests (test_gpu_fullsize.py) repeat the C1
cross-check on the device before trusting it at full size."""

import json

import numpy as np
import pytest
import torch

from oracle import fno_oracle as O
from oracle import torch_ref as R


def _load(golden_dir, name):
    d = dict(np.load(golden_dir / f"{name}.npz"))
    meta = json.loads((golden_dir / f"{name}.json").read_text())
    return d, meta, [d[f"w{i}"] for i in range(meta["blocks"])]


def _run(x, we, wd, blocks, modes, act, g=None):
    t = lambda a: torch.as_tensor(a)  # noqa: E731
    y, cache = R.forward(t(x).double(), t(we), t(wd), [t(w) for w in blocks], modes, act)
    gx, gwe, gwd, gws = R.backward(y if g is None else t(g), t(we), t(wd), [t(w) for w in blocks], modes, cache,
                                   act)
    return y, gx, gwe, gwd, gws


@pytest.mark.parametrize("name", ["acc16_c2_l4_f64", "g8_c2_l2_f64", "odd_11x10x6x5_f64", "uneven_9864_p3"])
def test_torch_ref_matches_reference_goldens(golden_dir, name):
    # goldens are the reference's own fno_forward / fno_backward (g = y) in real64
    d, meta, blocks = _load(golden_dir, name)
    y, gx, gwe, gwd, gws = _run(d["x"], d["we"], d["wd"], blocks, meta["modes"], meta["activation"])
    assert O.rel_err(y.numpy(), d["y_p1"]) < 1e-12
    assert O.rel_err(gx.numpy(), d["gx_p1"]) < 1e-12
    assert O.rel_err(gwe.numpy(), d["gwe_p1"]) < 1e-12
    assert O.rel_err(gwd.numpy(), d["gwd_p1"]) < 1e-12
    for i, gw in enumerate(gws):
        assert O.rel_err(gw.numpy(), d[f"gw{i}_p1"]) < 1e-12


@pytest.mark.parametrize("act", ["gelu", "relu", "identity"])
def test_torch_ref_matches_numpy_oracle_production_modes(act):
    # m = 8 on every dim (r = 16), width 6, odd and even extents, random g
    rng = np.random.default_rng(7)
    grid, modes, c, nb = (18, 17, 16, 20), (8, 8, 8, 8), 6, 2
    x = rng.standard_normal((2, 3) + grid)
    we, wd = rng.standard_normal((3, c)), rng.standard_normal((c, 2))
    blocks = [rng.standard_normal((c, c, 16, 16, 16, 16)) + 1j * rng.standard_normal((c, c, 16, 16, 16, 16))
              for _ in range(nb)]
    blocks = [b / c for b in blocks]
    g = rng.standard_normal((2, 2) + grid)
    y, gx, gwe, gwd, gws = _run(x, we, wd, blocks, modes, act, g)
    ry, cache = O.forward(x, we, wd, blocks, modes, act, with_cache=True)
    rgx, rgwe, rgwd, rgws = O.backward(g, we, wd, blocks, modes, cache, act)
    for a, b in ((y, ry), (gx, rgx), (gwe, rgwe), (gwd, rgwd), *zip(gws, rgws)):
        assert O.rel_err(a.numpy(), b) < 1e-12
