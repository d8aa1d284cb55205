"""Partition / routing integer logic: bit-exact against the reference's own
tables (tests/golden/partitions.json, written by the reference's
block_decompose and repartition_plan, d/partition.py:47-66, :135-188)."""

import json

import pytest

from paper_2211_12709_b200 import (
    BlockRange,
    DimLabel,
    InfeasiblePartitionError,
    Partition,
    ShapeMismatchError,
    block_decompose,
    range_intersection,
    repartition_plan,
)


@pytest.fixture(scope="module")
def tables(golden_dir):
    return json.loads((golden_dir / "partitions.json").read_text())


def test_block_decompose_matches_reference(tables):
    for key, ranges in tables["block_decompose"].items():
        n, P = map(int, key.split("/"))
        got = [[r.start, r.stop] for r in block_decompose(n, P)]
        assert got == ranges, key


def test_block_decompose_exhaustive_properties():
    # t/test_partition.py:32-44: remainder-first, balanced, tiling, all extents <= 300
    for n in range(1, 301):
        for P in range(1, min(n, 8) + 1):
            blocks = block_decompose(n, P)
            sizes = [len(b) for b in blocks]
            assert sum(sizes) == n
            assert max(sizes) - min(sizes) <= 1
            assert sizes == sorted(sizes, reverse=True)
            assert blocks[0].start == 0 and blocks[-1].stop == n
            for a, b in zip(blocks, blocks[1:]):
                assert a.stop == b.start


def test_infeasible():
    with pytest.raises(InfeasiblePartitionError):
        block_decompose(3, 4)
    with pytest.raises(InfeasiblePartitionError):
        block_decompose(3, 0)
    with pytest.raises(ShapeMismatchError):
        BlockRange(3, 2)
    with pytest.raises(InfeasiblePartitionError):
        Partition(DimLabel.X, 4, (BlockRange(0, 4), BlockRange(4, 4)))
    with pytest.raises(ShapeMismatchError):
        Partition(DimLabel.X, 5, (BlockRange(0, 2), BlockRange(3, 5)))


def test_intersection():
    assert range_intersection(BlockRange(0, 4), BlockRange(2, 9)) == BlockRange(2, 4)
    assert range_intersection(BlockRange(0, 2), BlockRange(2, 9)) is None


def test_repartition_plan_matches_reference(tables):
    for key, entries in tables["plans"].items():
        nx, ry, P, rank = map(int, key.split("/"))
        src = Partition.block(DimLabel.X, nx, P)
        dst = Partition.block(DimLabel.KY, ry, P)
        dims = [(DimLabel.B, 2), (DimLabel.C, 3), (DimLabel.X, nx), (DimLabel.KY, ry), (DimLabel.KZ, 4),
                (DimLabel.KT, 3)]
        plan = repartition_plan(src, dst, dims, rank)
        got = [[e.peer, [[r.start, r.stop] for r in e.send], [[r.start, r.stop] for r in e.recv]] for e in plan]
        assert got == entries, key


def test_plan_tiles_slabs():
    # t/test_partition.py:134-154: send blocks tile the local slab
    for nx, ry, P in [(9, 4, 3), (262, 16, 8), (7, 7, 7), (10, 6, 4)]:
        src = Partition.block("x", nx, P)
        dst = Partition.block("ky", ry, P)
        dims = [("b", 1), ("c", 2), ("x", nx), ("ky", ry)]
        for rank in range(P):
            plan = repartition_plan(src, dst, dims, rank)
            assert sum(e.element_count for e in plan) == 2 * src.extent_of(rank) * ry
            assert sum(e.recv_element_count for e in plan) == 2 * nx * dst.extent_of(rank)


def test_plan_errors():
    src = Partition.block("x", 8, 2)
    with pytest.raises(ShapeMismatchError):
        repartition_plan(src, Partition.block("x", 8, 2), [("x", 8)], 0)
    with pytest.raises(ShapeMismatchError):
        repartition_plan(src, Partition.block("ky", 4, 4), [("x", 8), ("ky", 4)], 0)
    with pytest.raises(ShapeMismatchError):
        repartition_plan(src, Partition.block("ky", 4, 2), [("x", 9), ("ky", 4)], 0)
