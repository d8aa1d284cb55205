"""Pin the numpy oracle to the reference: every golden fixture written by the
reference itself (tests/golden/make_golden.py) is replayed through
oracle/fno_oracle.py.  This is what lets the GPU parity tests trust the
oracle at sizes the fixtures do not cover."""

import json

import numpy as np
import pytest

from oracle import fno_oracle as O

CASES = ["g8_c2_l2_f64", "acc16_c2_l4_f64", "uneven_9864_p3", "odd_11x10x6x5_f64"]


def load(golden_dir, name):
    data = dict(np.load(golden_dir / f"{name}.npz"))
    meta = json.loads((golden_dir / f"{name}.json").read_text())
    blocks = [data[f"w{i}"] for i in range(meta["blocks"])]
    return data, meta, blocks


@pytest.mark.parametrize("name", CASES)
def test_oracle_forward_matches_reference(golden_dir, name):
    d, meta, blocks = load(golden_dir, name)
    y = O.forward(d["x"], d["we"], d["wd"], blocks, meta["modes"], meta["activation"])
    assert O.rel_err(y, d["y_serial"]) < 1e-12
    for P in meta["ranks"]:
        assert O.rel_err(y, d[f"y_p{P}"]) < 1e-10


@pytest.mark.parametrize("name", CASES)
def test_oracle_backward_matches_reference(golden_dir, name):
    d, meta, blocks = load(golden_dir, name)
    y, cache = O.forward(d["x"], d["we"], d["wd"], blocks, meta["modes"], meta["activation"], with_cache=True)
    gx, gwe, gwd, gws = O.backward(y, d["we"], d["wd"], blocks, meta["modes"], cache, meta["activation"])
    for P in meta["ranks"]:
        assert O.rel_err(gx, d[f"gx_p{P}"]) < 1e-10
        assert O.rel_err(gwe, d[f"gwe_p{P}"]) < 1e-10
        assert O.rel_err(gwd, d[f"gwd_p{P}"]) < 1e-10
        for i, gw in enumerate(gws):
            assert O.rel_err(gw, d[f"gw{i}_p{P}"]) < 1e-10


def test_oracle_fp32_reference_within_its_own_bar(golden_dir):
    # the reference's real32 run vs real64 oracle: the reference's own 1e-4 bar
    d32, meta, blocks = load(golden_dir, "acc16_c2_l4_f32")
    d64, _, b64 = load(golden_dir, "acc16_c2_l4_f64")
    y64 = O.forward(d64["x"], d64["we"], d64["wd"], b64, meta["modes"])
    assert O.rel_err(d32["y_p1"], y64) < 1e-4
    assert O.rel_err(d32["y_p8"], y64) < 1e-4


def test_staged_pipeline_and_volume(golden_dir):
    # the per-rank staged pipeline with explicit repartitions equals the
    # serial block, and its moved-element count equals the reference's
    # measured counters (repartition elements per rank, summed)
    d, meta, blocks = load(golden_dir, "uneven_9864_p3")
    P = 3
    nx = meta["grid"][0]
    a = O.act(meta["activation"], O.mix(d["x"], d["we"]))
    serial, _ = O.spectral_block(a, blocks[0], meta["modes"])
    slabs = [a[:, :, lo:hi] for lo, hi in O.block_ranges(nx, P)]
    pres, _, moved = O.staged_forward_block(slabs, blocks[0], meta["modes"], nx)
    assert O.rel_err(np.concatenate(pres, axis=2), serial) < 1e-12
    counters = meta[f"counters_fwd_p{P}"]
    measured = sum(r["repartition"][1] for r in counters)
    blocks_n = meta["blocks"]
    assert measured == 2 * blocks_n * moved
    assert moved == meta[f"predicted_p{P}"][0]


def test_retained_indices_known_answer():
    # t/test_spectral.py:80-81
    assert list(O.keep(8, 2)) == [0, 1, 6, 7]
    assert list(O.keep(4, 2)) == [0, 1, 2, 3]
