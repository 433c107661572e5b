"""Pins for the oracle's attention: dense Eq. 1 and vector-sparse Eq. 5
(P:320-341 / Alg. 2).

Pins: torch's float64 scaled_dot_product_attention on CPU (a library routine,
with an explicit boolean mask for Eq. 5), closed forms,
the full-selection reduction Eq. 5 -> Eq. 1, key-permutation equivariance
(S:70), torch.logsumexp for LSE, and the degenerate-row reading R6.
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import oracle as orc


def rand_qkv(N, D, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    return [orc.round_bf16(rng.standard_normal((N, D)) * scale) for _ in range(3)]


def sdpa(q, k, v, mask=None, causal=False, scale=None):
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))[None, None]
    o = F.scaled_dot_product_attention(t(q), t(k), t(v), attn_mask=None if mask is None else t(mask),
                                       is_causal=causal, scale=scale)
    return o[0, 0].numpy()


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("N,D", [(1, 8), (37, 16), (200, 64)])
def test_dense_matches_torch_sdpa_fp64(causal, N, D):
    q, k, v = rand_qkv(N, D, 1)
    o, lse = orc.dense_attn(q, k, v, causal=causal)
    np.testing.assert_allclose(o, sdpa(q, k, v, causal=causal), rtol=0, atol=1e-12)
    s = torch.from_numpy(q @ k.T / math.sqrt(D))
    if causal:
        s = s.masked_fill(torch.triu(torch.ones(N, N, dtype=torch.bool), 1), float("-inf"))
    np.testing.assert_allclose(lse, torch.logsumexp(s, 1).numpy(), rtol=0, atol=1e-12)


def test_dense_identity_closed_form():
    # Q=K=V=I2, scale 1/sqrt(2): row 0 = softmax([1/sqrt2, 0])
    I = np.eye(2)
    o, _ = orc.dense_attn(I, I, I)
    p = math.exp(1 / math.sqrt(2)) / (math.exp(1 / math.sqrt(2)) + 1.0)
    np.testing.assert_allclose(o, [[p, 1 - p], [1 - p, p]], rtol=0, atol=1e-15)


def test_dense_single_key_broadcasts_v():
    # one key -> A is all ones, O = V broadcast
    rng = np.random.default_rng(2)
    q = rng.standard_normal((5, 4))
    k = rng.standard_normal((1, 4))
    v = rng.standard_normal((1, 4))
    # Eq. 1 with N_k=1: emulate by dense over a 1-row problem per query row
    for r in range(5):
        o, lse = orc.dense_attn(q[r:r + 1], k, v)
        np.testing.assert_array_equal(o[0], v[0])


def _full_csr(Np, N):
    off = np.arange(0, (Np + 1) * N, N, dtype=np.int64)
    idx = np.tile(np.arange(N, dtype=np.int32), Np)
    return off, idx


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("N,pq", [(256, 64), (300, 64), (130, 128)])
def test_sparse_full_selection_equals_dense(causal, N, pq):
    # Eq. 5 with Idx(i) = all keys reduces to Eq. 1
    q, k, v = rand_qkv(N, 32, 3)
    Np = (N + pq - 1) // pq
    off, idx = _full_csr(Np, N)
    o, lse = orc.sparse_attn(q, k, v, off, idx, pq, causal=causal)
    od, lsed = orc.dense_attn(q, k, v, causal=causal)
    np.testing.assert_allclose(o[:N], od, rtol=0, atol=1e-12)
    np.testing.assert_allclose(lse[:N], lsed, rtol=0, atol=1e-12)
    if Np * pq > N:
        assert np.all(o[N:] == 0) and np.all(np.isnan(lse[N:]))


def test_sparse_one_key_per_block_gives_v_row():
    # one selected key j per block, non-causal -> each output row equals V[j]
    N, pq = 256, 64
    q, k, v = rand_qkv(N, 16, 4)
    picks = np.array([7, 200, 31, 99], np.int32)
    off = np.arange(5, dtype=np.int64)
    o, _ = orc.sparse_attn(q, k, v, off, picks, pq)
    for i, j in enumerate(picks):
        np.testing.assert_array_equal(o[i * pq:(i + 1) * pq], np.broadcast_to(v[j], (pq, 16)))


@pytest.mark.parametrize("causal", [False, True])
def test_sparse_matches_masked_sdpa(causal):
    # Eq. 5 == SDPA with the boolean mask M[r,j] = (j in Idx(i)) & (j <= r if causal)
    N, D, pq = 320, 32, 64
    q, k, v = rand_qkv(N, D, 5)
    rng = np.random.default_rng(6)
    Np = (N + pq - 1) // pq
    sets = []
    for i in range(Np):
        hi = min(N, (i + 1) * pq) if causal else N
        m = rng.random(hi) < 0.3
        m[rng.integers(0, hi)] = True
        if causal:
            m[i * pq] = True  # every row sees >= 1 key
        sets.append(np.nonzero(m)[0].astype(np.int32))
    off = np.zeros(Np + 1, np.int64)
    off[1:] = np.cumsum([s.size for s in sets])
    idx = np.concatenate(sets)
    o, lse = orc.sparse_attn(q, k, v, off, idx, pq, causal=causal)
    mask = np.zeros((N, N), bool)
    for i, s in enumerate(sets):
        mask[i * pq:min(N, (i + 1) * pq), s] = True
    if causal:
        mask &= np.tril(np.ones((N, N), bool))
    np.testing.assert_allclose(o[:N], sdpa(q, k, v, mask=mask), rtol=0, atol=1e-12)
    sc = torch.from_numpy(q @ k.T / math.sqrt(D)).masked_fill(torch.from_numpy(~mask), float("-inf"))
    np.testing.assert_allclose(lse[:N], torch.logsumexp(sc, 1).numpy(), rtol=0, atol=1e-12)
    # rows of P sum to 1 <=> O of V=ones is ones
    o1, _ = orc.sparse_attn(q, k, np.ones_like(v), off, idx, pq, causal=causal)
    np.testing.assert_allclose(o1[:N], 1.0, rtol=0, atol=1e-13)


def test_sparse_permutation_equivariance_noncausal():
    # permuting K and V rows (and remapping indices) leaves O unchanged
    N, D, pq = 192, 16, 64
    q, k, v = rand_qkv(N, D, 7)
    rng = np.random.default_rng(8)
    sets = [np.sort(rng.choice(N, 40, replace=False)).astype(np.int32) for _ in range(3)]
    off = np.array([0, 40, 80, 120], np.int64)
    o, _ = orc.sparse_attn(q, k, v, off, np.concatenate(sets), pq)
    perm = rng.permutation(N)
    inv = np.argsort(perm)
    kp, vp = k[perm], v[perm]
    sets2 = [np.sort(inv[s]).astype(np.int32) for s in sets]
    o2, _ = orc.sparse_attn(q, kp, vp, off, np.concatenate(sets2), pq)
    np.testing.assert_allclose(o, o2, rtol=0, atol=1e-13)


def test_sparse_causal_degenerate_rows_take_own_value():
    # Reading R6: a causal row with no visible selected key outputs V_r and
    # LSE_r = scale*<q_r,k_r>.
    N, D, pq = 128, 16, 64
    q, k, v = rand_qkv(N, D, 9)
    off = np.array([0, 1, 2], np.int64)
    idx = np.array([63, 64], np.int32)  # block 0 selects only its last key
    o, lse = orc.sparse_attn(q, k, v, off, idx, pq, causal=True)
    for r in range(63):
        np.testing.assert_array_equal(o[r], v[r])
        assert lse[r] == pytest.approx(float(q[r] @ k[r]) / 4.0, abs=1e-14)
    np.testing.assert_array_equal(o[63], v[63])
    np.testing.assert_array_equal(o[64:], np.broadcast_to(v[64], (64, D)))


def test_shift_invariance_of_softmax():
    # adding a constant to all scores of a row leaves A unchanged.  With
    # k_j -> k_j + c*q_r/|q_r|^2 * sqrt(D) for one query row, every score of that
    # row shifts by c.
    N, D = 64, 8
    q, k, v = rand_qkv(N, D, 10)
    r = 5
    c = 3.0
    shift = c * q[r] / float(q[r] @ q[r]) * math.sqrt(D)
    o1, l1 = orc.dense_attn(q, k, v, rows=[r])
    o2, l2 = orc.dense_attn(q, k + shift, v, rows=[r])
    np.testing.assert_allclose(o1, o2, rtol=0, atol=1e-12)
    assert l2[0] == pytest.approx(l1[0] + c, abs=1e-12)
