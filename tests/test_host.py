"""Host-side logic of the drop-in (no GPU needed): configuration rules,
bit-identical parameter init, sharding, volume prediction, labelled tensors,
spectral bookkeeping -- each against the reference's fixtures or its
documented behaviour."""

import hashlib
import json

import numpy as np
import pytest
import torch

import paper_2211_12709_b200 as P
from paper_2211_12709_b200 import (
    DATA_LABELS,
    DenseTensor,
    DimensionMismatchError,
    DimLabel,
    DType,
    FnoConfig,
    InfeasiblePartitionError,
    ModeSpec,
    init_params,
    predicted_block_volume,
    shard_params,
)


def cfg(grid=(8, 8, 8, 4), modes=(2, 2, 2, 2), c=2, blocks=2, dtype="real64", P_=1, act="gelu", cin=None, cout=None):
    return FnoConfig(nx=grid[0], ny=grid[1], nz=grid[2], nt=grid[3], in_channels=cin or c, out_channels=cout or c,
                     hidden_channels=c, modes=ModeSpec.of_xyzt(*modes), num_blocks=blocks, activation=act,
                     dtype=dtype, num_ranks=P_)


def test_config_feasibility():
    # t/test_fno.py:57-61
    with pytest.raises(InfeasiblePartitionError):
        cfg(grid=(3, 4, 5, 2), modes=(1, 1, 1, 1), P_=4)
    with pytest.raises(InfeasiblePartitionError):
        cfg(grid=(16, 8, 8, 4), P_=9)
    with pytest.raises(DimensionMismatchError):
        cfg(dtype="complex64")
    with pytest.raises(DimensionMismatchError):
        cfg(blocks=0)


def test_retained_extents():
    c = cfg(grid=(16, 16, 16, 8), modes=(4, 4, 4, 3))
    assert (c.retained_x, c.retained_y, c.retained_z, c.retained_t) == (8, 8, 8, 6)


def test_init_params_bit_identical_to_reference(golden_dir):
    digests = json.loads((golden_dir / "init_digests.json").read_text())
    for key, want in digests.items():
        grid, modes, c, blocks, dtype, seed, cin, cout = json.loads(key)
        config = cfg(tuple(grid), tuple(modes), c, blocks, dtype, cin=cin, cout=cout)
        p = init_params(config, seed, device="cpu")
        for name, t in p.named().items():
            got = hashlib.sha256(t.data.numpy().tobytes()).hexdigest()
            assert got == want[name], (key, name)


def test_shard_params_slices_ky():
    config = cfg(grid=(9, 12, 8, 4), modes=(2, 3, 2, 2), c=3, P_=3)
    p = init_params(config, 0, device="cpu")
    for rank in range(3):
        lp = shard_params(p, config, rank)
        r = config.ky_partition().range_of(rank)
        assert torch.equal(lp.blocks[0].data, p.blocks[0].data[:, :, :, r.start:r.stop])
    with pytest.raises(DimensionMismatchError):
        shard_params(shard_params(p, config, 0), config, 0)


def test_predicted_volume_matches_reference(golden_dir):
    for name in ["g8_c2_l2_f64", "uneven_9864_p3", "acc16_c2_l4_f64", "odd_11x10x6x5_f64"]:
        meta = json.loads((golden_dir / f"{name}.json").read_text())
        for Pn in meta["ranks"]:
            c = cfg(tuple(meta["grid"]), tuple(meta["modes"]), meta["channels"], meta["blocks"], meta["dtype"], Pn,
                    meta["activation"], meta["in_channels"], meta["out_channels"])
            v = predicted_block_volume(c, meta["batch"])
            got = [v.per_repartition_elements, v.per_block_elements, v.per_forward_elements,
                   v.naive_per_repartition_elements, v.reduction_ratio, v.bytes_per_element]
            assert got == meta[f"predicted_p{Pn}"]


def test_predicted_volume_known_answers():
    # t/test_fno.py:232-244
    assert predicted_block_volume(cfg(grid=(10, 10, 10, 10), modes=(1, 1, 1, 1), c=1, P_=2)).reduction_ratio == 125.0
    v = predicted_block_volume(cfg(grid=(16, 16, 16, 8), modes=(4, 4, 4, 3), P_=4), batch_size=3)
    closed = 3 * 2 * 16 * 8 * 8 * 6 * 3 // 4
    assert v.per_repartition_elements == closed and v.bytes_per_element == 16


def test_dense_tensor_rules():
    with pytest.raises(DimensionMismatchError):
        DenseTensor(("b", "b"), np.zeros((1, 1)))
    with pytest.raises(DimensionMismatchError):
        DenseTensor(("kx",), np.zeros(3))
    t = DenseTensor(DATA_LABELS, np.zeros((1, 2, 3, 4, 5, 6), dtype=np.float32))
    assert t.dtype == DType.REAL32 and t.extent("z") == 5 and t.axis(DimLabel.T) == 5
    with pytest.raises(AttributeError):
        t.labels = ()
    src = np.ones(3)
    t2 = DenseTensor(("x",), src)
    src[0] = 7  # the tensor owns its bytes (reference tensor.py:145-148)
    assert float(t2.data[0]) == 1.0


def test_modespec_and_retained():
    assert list(P.retained_indices(8, 2)) == [0, 1, 6, 7]
    assert P.retained_extent(5, 3) == 5
    m = ModeSpec.of_xyzt(1, 2, 3, 4).restrict(("kx", "kz"))
    assert m.labels() == (DimLabel.KX, DimLabel.KZ)


def test_truncate_pad_adjoint_host_tensors():
    # pad_modes is the exact adjoint of truncate_modes (t/test_spectral.py:138-161)
    spec = ModeSpec({DimLabel.KY: 2, DimLabel.KZ: 2})
    rng = np.random.default_rng(0)
    x = DenseTensor(("ky", "kz"), rng.standard_normal((9, 6)) + 1j * rng.standard_normal((9, 6)))
    y = DenseTensor(("ky", "kz"), rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4)))
    lhs = np.vdot(P.truncate_modes(x, spec).numpy(), y.numpy())
    rhs = np.vdot(x.numpy(), P.pad_modes(y, spec, {"ky": 9, "kz": 6}).numpy())
    assert abs(lhs - rhs) < 1e-12 * max(abs(lhs), 1)


def test_channel_envelope_rejected_before_any_kernel():
    # real64 keeps a channel row per thread in its fused x-spectral kernel:
    # widths above 32 are refused when the plan is built; real32 takes any width
    import paper_2211_12709_b200 as P
    from paper_2211_12709_b200 import fno as F

    F.check_envelope(P.FnoConfig(8, 8, 8, 4, 3, 3, 64, P.ModeSpec.of_xyzt(2, 2, 2, 2), 1, "gelu", "real32", 1))
    F.check_envelope(P.FnoConfig(8, 8, 8, 4, 32, 32, 32, P.ModeSpec.of_xyzt(2, 2, 2, 2), 1, "gelu", "real64", 1))
    wide = P.FnoConfig(8, 8, 8, 4, 3, 3, 40, P.ModeSpec.of_xyzt(2, 2, 2, 2), 1, "gelu", "real64", 1)
    with pytest.raises(P.DimensionMismatchError, match="hidden_channels"):
        F.check_envelope(wide)
