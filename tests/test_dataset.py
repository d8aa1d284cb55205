"""The synthetic spectral-propagator dataset (reference d/bench.py:403-430)
against the reference's own arrays (tests/golden/train_ref.npz), generated
with the host device here; the GPU run is in test_gpu_drivers.py."""

import json

import numpy as np

from paper_2211_12709_b200 import drivers as D


def test_make_dataset_host_matches_reference(golden_dir):
    meta = json.loads((golden_dir / "train_ref.json").read_text())["dataset"]
    ref = np.load(golden_dir / "train_ref.npz")
    x, y = D.make_dataset(D.config_from_opts(meta), meta["samples"], meta["seed"], device="cpu")
    assert x.shape == ref["ds_x"].shape and y.shape == ref["ds_y"].shape
    assert (x.numpy() == ref["ds_x"]).all()
    assert np.abs(y.numpy() - ref["ds_y"]).max() <= 1e-6 * np.abs(ref["ds_y"]).max()
