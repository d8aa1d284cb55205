"""The synthetic spectral-propagator dataset (reference d/bench.py:403-430):
the host-side draws against the reference's own arrays
(tests/golden/train_ref.npz); the transforms run on libdfno's block kernels
and are checked on the GPU in test_gpu_drivers.py."""

import json

import numpy as np
import pytest

from paper_2211_12709_b200 import drivers as D
from paper_2211_12709_b200.errors import ExtensionMissingError


def test_make_dataset_draws_match_reference(golden_dir):
    # same PCG64 stream, same order: the inputs are the reference's, cast once
    meta = json.loads((golden_dir / "train_ref.json").read_text())["dataset"]
    ref = np.load(golden_dir / "train_ref.npz")
    cfg = D.config_from_opts(meta)
    rng = np.random.default_rng(meta["seed"])
    r_shape = tuple(min(n, 2 * m) for n, m in zip(cfg.grid, cfg.mode_counts))
    rng.standard_normal((cfg.out_channels, cfg.in_channels) + r_shape)
    rng.standard_normal((cfg.out_channels, cfg.in_channels) + r_shape)
    x = rng.standard_normal((meta["samples"], cfg.in_channels) + cfg.grid).astype(cfg.dtype.np_dtype)
    assert x.shape == ref["ds_x"].shape and (x == ref["ds_x"]).all()


def test_make_dataset_has_no_host_path(golden_dir):
    meta = json.loads((golden_dir / "train_ref.json").read_text())["dataset"]
    with pytest.raises(ExtensionMissingError):
        D.make_dataset(D.config_from_opts(meta), meta["samples"], meta["seed"], device="cpu")
