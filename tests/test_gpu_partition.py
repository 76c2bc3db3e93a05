"""bc_reduce_partition on the GPU (bulge.py:348-385): the relayed chase over several workers is
bit-identical to the whole-band chase (the reference's tests/test_bulge.py:59-91 property), and
the protocol errors of bulge.py:335-361 are raised."""
import numpy as np
import pytest

from paper_2511_16174_b200 import (BandMatrix, BulgeReflectorSet, OverlapBlock, ProtocolError,
                                   bc_reduce, partition)
from paper_2511_16174_b200.stages import bc_reduce_partition


def _rand_band(rng, n, b):
    g = rng.standard_normal((n, n))
    a = (g + g.T) / 2
    a[np.abs(np.subtract.outer(np.arange(n), np.arange(n))) > b] = 0.0
    return BandMatrix.from_dense(a, b)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(6))
def test_partitioned_chase_matches_single_worker(seed):
    rng = np.random.default_rng(200 + seed)
    b = int(rng.integers(2, 6))
    n = int(rng.integers(4 * b, 72))
    workers = int(rng.integers(2, 5))
    band = _rand_band(rng, n, b)
    t_ref, u_ref = bc_reduce(band)
    d_parts, e_parts, refl_parts = [], [], []
    tail, overlap = band, None
    for i, (c0, c1) in enumerate(partition(n, workers)):
        last = i == workers - 1
        res = bc_reduce_partition(tail, b, c0, c1, overlap, last)
        d_parts.append(res.d_part)
        e_parts.append(res.e_part)
        refl_parts.append(res.reflectors)
        tail, overlap = res.tail, res.outgoing
    merged = BulgeReflectorSet.merge(refl_parts)
    np.testing.assert_array_equal(np.concatenate(d_parts), t_ref.d)
    np.testing.assert_array_equal(np.concatenate(e_parts), t_ref.e)
    assert len(merged) == len(u_ref)
    for f in ("i_idx", "j_idx", "row0", "length", "tau", "v"):
        np.testing.assert_array_equal(getattr(merged, f), getattr(u_ref, f))


@pytest.mark.gpu
def test_partitioned_chase_b32_large():
    rng = np.random.default_rng(7)
    n, b = 700, 32
    band = _rand_band(rng, n, b)
    t_ref, u_ref = bc_reduce(band)
    tail, overlap, d_parts = band, None, []
    for i, (c0, c1) in enumerate(partition(n, 3)):
        res = bc_reduce_partition(tail, b, c0, c1, overlap, i == 2)
        d_parts.append(res.d_part)
        tail, overlap = res.tail, res.outgoing
    np.testing.assert_array_equal(np.concatenate(d_parts), t_ref.d)


def test_partition_protocol_errors():
    band = BandMatrix(8, 2, np.zeros((3, 8)))
    with pytest.raises(ProtocolError):            # interior worker without an overlap block
        bc_reduce_partition(band, 2, 4, 8, None, True)
    ov = OverlapBlock(values=np.zeros((4, 2)), offset=0, b=2)
    with pytest.raises(ProtocolError):            # first worker must not receive one
        bc_reduce_partition(band, 2, 0, 4, ov, False)
    with pytest.raises(ProtocolError):            # wrong boundary
        bc_reduce_partition(band, 2, 4, 8, OverlapBlock(values=np.zeros((4, 2)), offset=3, b=2),
                            True)
    bad = np.zeros((4, 2))
    bad[2, 0] = 1.0
    with pytest.raises(ProtocolError):            # fill outside the bridge entry
        bc_reduce_partition(band, 2, 4, 8, OverlapBlock(values=bad, offset=4, b=2), True)
