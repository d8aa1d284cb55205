"""The verification drivers on the device path,
with the reference's options and bars: SPEC criteria 1-4 (parity 1e-10 in
real64, adjoints 1e-12, finite-difference gradient 1e-5) and the exact
communication volume of the reference's own drive_comm_volume run
(tests/golden/commvolume_9864_p3.json)."""

import json

import pytest

import paper_2211_12709_b200 as P
from paper_2211_12709_b200 import drivers as D

pytestmark = pytest.mark.gpu


def run(driver, opts):
    return P.run_ranks(opts["workers"], lambda comm: driver(comm, opts))[0]


def test_comm_volume_equals_reference_run(golden_dir):
    want = json.loads((golden_dir / "commvolume_9864_p3.json").read_text())
    got = run(D.drive_comm_volume, {"grid": [9, 8, 6, 4], "modes": [2, 2, 2, 2], "channels": 2, "blocks": 2,
                                    "dtype": "real64", "seed": 0, "batch": 2, "activation": "gelu", "workers": 3})
    assert got == want


def _oracle_serial_forward(x_global, params, cfg):
    """The reference's serial_fno_forward slot filled by the float64 numpy
    oracle (all-at-once FFTs, oracle/fno_oracle.py)."""
    from oracle import fno_oracle as O

    blocks = [w.numpy().astype("complex128") for w in params.blocks]
    return O.forward(x_global.numpy().astype("float64"), params.we.numpy().astype("float64"),
                     params.wd.numpy().astype("float64"), blocks, cfg.mode_counts, cfg.activation.value)


@pytest.mark.parametrize("dtype,tol", [("real64", 1e-10), ("real32", 1e-5)])
def test_parity_against_serial_oracle(dtype, tol):
    # SPEC criterion 1 as the reference runs it: distributed forward vs the
    # serial all-at-once oracle (d/bench.py:100-124)
    opts = {"grid": [16, 16, 16, 8], "modes": [4, 4, 4, 3], "channels": 2, "blocks": 4, "dtype": dtype, "seed": 7,
            "workers": 8}
    res = P.run_ranks(8, lambda comm: D.drive_parity_forward(comm, opts, serial_forward=_oracle_serial_forward))[0]
    assert res["max_rel_err"] < tol


@pytest.mark.parametrize("dtype,tol", [("real64", 1e-10), ("real32", 1e-5)])
def test_parity_decomposition_invariance(dtype, tol):
    res = run(D.drive_parity_forward, {"grid": [16, 16, 16, 8], "modes": [4, 4, 4, 3], "channels": 2, "blocks": 4,
                                       "dtype": dtype, "seed": 7, "workers": 8})
    assert res["max_rel_err"] < tol
    assert res["repart_calls_per_rank"] == 8
    cfg = D.config_from_opts({"grid": [16, 16, 16, 8], "modes": [4, 4, 4, 3], "channels": 2, "blocks": 4,
                              "dtype": dtype, "workers": 8})
    assert res["repart_elements_total"] == P.predicted_block_volume(cfg, 1).per_forward_elements


def test_adjoint_identities():
    res = run(D.drive_adjoint, {"seed": 3, "pairs": 5, "workers": 3})
    assert res["broadcast_reduce_max_err"] < 1e-12 and res["repartition_max_err"] < 1e-12


def test_finite_difference_gradient():
    res = run(D.drive_gradient, {"grid": [8, 8, 8, 4], "modes": [2, 2, 2, 2], "channels": 2, "blocks": 2,
                                 "dtype": "real64", "seed": 11, "directions": 5, "workers": 2})
    assert res["max_rel_err"] < 1e-5, res["errors"]


@pytest.fixture(scope="module")
def train_ref(golden_dir):
    import numpy as np

    return json.loads((golden_dir / "train_ref.json").read_text()), np.load(golden_dir / "train_ref.npz")


def test_make_dataset_matches_reference(train_ref):
    meta, arrays = train_ref
    d = meta["dataset"]
    x, y = D.make_dataset(D.config_from_opts(d), d["samples"], d["seed"])
    assert x.is_cuda and x.dtype == y.dtype
    assert (x.cpu().numpy() == arrays["ds_x"]).all()  # same PCG64 draws, cast once
    err = abs(y.cpu().numpy() - arrays["ds_y"]).max() / abs(arrays["ds_y"]).max()
    assert err < 1e-6  # float64 transforms on the device vs numpy, then one float32 rounding


@pytest.mark.parametrize("workers", [1, 2])
def test_drive_train_matches_reference(train_ref, workers, tmp_path):
    meta, _ = train_ref
    opts = dict(meta["opts"], workers=workers, checkpoint=str(tmp_path / "ckpt"))
    got = run(D.drive_train, opts)
    want = meta[f"train_p{workers}"]
    assert got["epochs_run"] == want["epochs_run"] == len(want["metrics"]) - 1
    for g, w in zip(got["metrics"], want["metrics"]):
        assert g["epoch"] == w["epoch"]
        for k in ("test_mse", "test_mae", "test_r2", "train_mse_median"):
            if w[k] is None:
                assert g[k] is None
            else:  # float32 training, 4 epochs of Adam: agreement to ~1e-6 relative
                assert abs(g[k] - w[k]) <= 1e-4 * max(abs(w[k]), 1e-2), (k, g[k], w[k])
    assert got["metrics"][-1]["test_mse"] < 0.7 * got["metrics"][0]["test_mse"]  # it learns
    params, cfg, seed = P.load_checkpoint(str(tmp_path / "ckpt"))
    assert seed == opts["seed"] and cfg.num_ranks == workers
