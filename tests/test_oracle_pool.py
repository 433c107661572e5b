"""Pins for the oracle's query pooling (Eq. 2) and bf16 rounding.

Each pin is fixed by something other than the oracle itself: SPEC.md worked
examples, hand-computed RNE ties, and torch's own fp32->bf16 RNE.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc


def test_pool_identity_pq1():
    # S:116 "Pq=1 -> output equals Q exactly"
    rng = np.random.default_rng(0)
    q = orc.round_bf16(rng.standard_normal((37, 8)))
    np.testing.assert_array_equal(orc.pool(q, 1), q)


def test_pool_worked_example():
    # S:117 "Q=[[1,3],[3,5]], Pq=2 -> [[2,4]]"
    np.testing.assert_array_equal(orc.pool(np.array([[1.0, 3.0], [3.0, 5.0]]), 2), [[2.0, 4.0]])


def test_pool_ragged_last_block():
    # S:118 / S:113: 10x4 with Pq=4 -> 3 rows; last = mean of rows 8-9 (true height)
    rng = np.random.default_rng(1)
    q = rng.standard_normal((10, 4))
    qp = orc.pool(q, 4, round_to_bf16=False)
    assert qp.shape == (3, 4)
    np.testing.assert_allclose(qp[2], (q[8] + q[9]) / 2.0, rtol=0, atol=1e-15)
    np.testing.assert_allclose(qp[0], q[0:4].sum(0) / 4.0, rtol=0, atol=1e-15)


@pytest.mark.parametrize("rows,expect", [
    # exact midpoint between 1.0 (even mantissa) and 1+2^-7 (odd) -> ties to even -> 1.0
    ([1.0, 1.0078125], 1.0),
    # midpoint between 1+2^-7 (odd) and 1+2^-6 (even) -> 1+2^-6
    ([1.0078125, 1.015625], 1.015625),
    # 1.005859375 lies above the midpoint 1.00390625 -> rounds up to 1+2^-7
    ([1.0, 1.0078125, 1.0078125, 1.0078125], 1.0078125),
    # negative tie: -(1 + 2^-8) -> -1.0
    ([-1.0, -1.0078125], -1.0),
])
def test_pool_rne_ties(rows, expect):
    q = np.array(rows, np.float64).reshape(-1, 1)
    qp = orc.pool(q, len(rows))
    assert qp.shape == (1, 1) and qp[0, 0] == expect


def test_round_bf16_matches_torch_rne():
    # torch's float32 -> bfloat16 conversion is IEEE RNE; for fp32-representable
    # inputs, fp64 -> bf16 RNE must agree with it bit for bit.
    rng = np.random.default_rng(2)
    x32 = np.concatenate([
        rng.standard_normal(100_000).astype(np.float32),
        (rng.standard_normal(10_000) * 1e-30).astype(np.float32),
        (rng.standard_normal(10_000) * 1e30).astype(np.float32),
        np.array([1.00390625, 1.01171875, -1.00390625, 2.0 ** -133, 3 * 2.0 ** -134], np.float32),
    ])
    ours = orc.round_bf16(x32.astype(np.float64))
    ref = torch.from_numpy(x32).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(ours, ref)


def test_pool_bf16_inputs_against_numpy_mean():
    # For bf16 inputs the fp64 block sum is exact; compare with numpy's mean then
    # torch RNE (valid when the fp64 mean is exactly representable in fp32).
    g = torch.Generator().manual_seed(3)
    qb = torch.randn(1000, 16, generator=g).to(torch.bfloat16)
    q = qb.to(torch.float64).numpy()
    pq = 64
    qp = orc.pool(q, pq)
    Np = (1000 + pq - 1) // pq
    for i in range(Np):
        m = q[i * pq:min(1000, (i + 1) * pq)].mean(0)
        m32 = m.astype(np.float32)
        if not np.array_equal(m32.astype(np.float64), m):
            continue
        ref = torch.from_numpy(m32).to(torch.bfloat16).to(torch.float64).numpy()
        np.testing.assert_array_equal(qp[i], ref)


def test_bf16_bits_roundtrip():
    g = torch.Generator().manual_seed(4)
    t = torch.randn(333, generator=g).to(torch.bfloat16)
    bits = t.view(torch.int16).numpy().view(np.uint16)
    x = orc.bf16_bits_to_f64(bits)
    np.testing.assert_array_equal(x, t.to(torch.float64).numpy())
    np.testing.assert_array_equal(orc.f64_to_bf16_bits(x), bits)
