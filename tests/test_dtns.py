"""DTNS tensor files and checkpoints against the
reference's own bytes (tests/golden/dtns_ref.npz, tests/golden/ckpt_ref/,
made by tests/golden/make_golden.py from distfno.tensor / distfno.training):
byte-identical serialisation, round trips, the reference's error cases
(d/tensor.py:282-312) and checkpoint interop both ways."""

import filecmp
import io

import numpy as np
import pytest
import torch

import paper_2211_12709_b200 as P

LABELS = {"r32": ("b", "c", "x", "y", "z", "t"), "r64": ("c", "co"), "c64": ("c", "co", "kx", "ky"),
          "c128": ("kz", "kt")}


@pytest.fixture(scope="module")
def ref(golden_dir):
    return np.load(golden_dir / "dtns_ref.npz")


@pytest.mark.parametrize("key", sorted(LABELS))
def test_bytes_identical_to_reference(ref, key):
    t = P.DenseTensor(LABELS[key], torch.from_numpy(ref[f"{key}_data"]))
    assert P.tensor_to_bytes(t) == ref[f"{key}_bytes"].tobytes()
    back = P.tensor_from_bytes(ref[f"{key}_bytes"].tobytes())
    assert P.bit_equal(back, t)
    assert P.serialized_size(t.labels, t.shape, t.dtype) == len(ref[f"{key}_bytes"])
    sink = io.BytesIO()
    assert P.tensor_write(t, sink) == len(ref[f"{key}_bytes"])
    assert P.bit_equal(P.tensor_read(io.BytesIO(sink.getvalue())), t)


def test_malformed_streams(ref):
    good = ref["c64_bytes"].tobytes()
    with pytest.raises(P.MalformedHeaderError):
        P.tensor_from_bytes(b"XXXX" + good[4:])
    with pytest.raises(P.MalformedHeaderError):
        P.tensor_from_bytes(good[:4] + bytes([2]) + good[5:])
    with pytest.raises(P.UnknownDTypeError):
        P.tensor_from_bytes(good[:5] + bytes([9]) + good[6:])
    with pytest.raises(P.TruncatedPayloadError):
        P.tensor_from_bytes(good[:-1])
    with pytest.raises(P.TruncatedPayloadError):
        P.tensor_from_bytes(good[:12])
    assert issubclass(P.TruncatedPayloadError, P.SerializationError)


def test_checkpoint_interop_both_ways(golden_dir, tmp_path):
    params, cfg, seed = P.load_checkpoint(str(golden_dir / "ckpt_ref"))
    assert seed == 5 and cfg.grid == (8, 8, 8, 4) and cfg.num_ranks == 2
    assert (cfg.in_channels, cfg.hidden_channels, cfg.out_channels, cfg.num_blocks) == (1, 2, 3, 2)
    mine = P.init_params(cfg, 5, device="cpu")
    for k, v in mine.named().items():
        assert P.bit_equal(v, params.named()[k]), k
    P.save_checkpoint(str(tmp_path), mine, cfg, 5)
    for name in ("manifest.txt", "we.dtns", "wd.dtns", "block0.dtns", "block1.dtns"):
        assert filecmp.cmp(tmp_path / name, golden_dir / "ckpt_ref" / name, shallow=False), name
    with pytest.raises(ValueError):
        P.save_checkpoint(str(tmp_path / "s"), P.shard_params(mine, cfg, 0), cfg, 5)


@pytest.mark.gpu
def test_checkpoint_to_device_and_gather_params(golden_dir):
    params, cfg, _ = P.load_checkpoint(str(golden_dir / "ckpt_ref"), device="cuda")
    assert params.we.data.is_cuda

    def worker(comm):
        full = P.gather_params(comm, P.shard_params(params, cfg, comm.rank), cfg)
        return full

    res = P.run_ranks(2, worker)
    assert res[1] is None
    for k, v in params.named().items():
        assert P.bit_equal(res[0].named()[k], v), k
