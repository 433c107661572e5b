"""Pins for the oracle's important-vector selection.

  MINS_ALG1  Alg. 1, P:788-831 (running row max, reset per group of G_K tiles)
  MINS_EXACT Eq. 3
  TOPK       P:213-214 ("exactly the k largest"), ties -> lowest index

Scores are injected exactly: with D=4 (scale 1/2) and Q_p row i = 2*e_i, the
pooled score of key j for row i is s_ij = K[j, i].  Pins: SPEC.md worked
examples, examples hand-derived from the
Alg. 1 listing (tests/golden/alg1_examples.json), brute-force subset
enumeration, torch.topk, and invariants.
"""
import itertools
import json
import os

import numpy as np
import pytest
import torch

from oracle import oracle as orc

GOLD = os.path.join(os.path.dirname(__file__), "golden", "alg1_examples.json")


def inject(score_rows):
    """Q_p, K such that oracle scores equal score_rows exactly (<= 4 rows)."""
    s = np.asarray(score_rows, np.float64)
    R, N = s.shape
    assert R <= 4
    qp = np.zeros((R, 4))
    for i in range(R):
        qp[i, i] = 2.0
    k = np.zeros((N, 4))
    k[:, :R] = s.T
    return qp, k


def sel_sets(offsets, indices):
    return [set(indices[offsets[r]:offsets[r + 1]].tolist()) for r in range(len(offsets) - 1)]


def run(scores, **kw):
    qp, k = inject(scores)
    kw.setdefault("pq", 1)
    off, idx = orc.select(qp, k, **kw)
    return sel_sets(off, idx)


def test_injection_is_exact():
    qp, k = inject([[5.0, 3.0, 4.9, 1.0]])
    np.testing.assert_array_equal(orc.scores_row(qp, k, 0), [5.0, 3.0, 4.9, 1.0])


def test_mins_exact_spec_example():
    # S:126 "s=[5,3,4.9,1], alpha=0.5 -> selected=[0,2]"
    assert run([[5, 3, 4.9, 1]], mode=orc.SEL_MINS_EXACT, alpha=0.5) == [{0, 2}]


def test_mins_alpha_zero_is_argmax():
    # S:127 "alpha=0 with unique maximum -> exactly the argmax column"
    assert run([[5, 3, 4.9, 1]], mode=orc.SEL_MINS_EXACT, alpha=0.0) == [{0}]


def test_mins_large_alpha_selects_all():
    # S:128 "alpha >= rowmax-rowmin -> all columns"
    assert run([[5, 3, 4.9, 1]], mode=orc.SEL_MINS_EXACT, alpha=4.0) == [{0, 1, 2, 3}]


def test_alg1_golden_examples():
    cases = json.load(open(GOLD))["cases"]
    assert len(cases) >= 4
    for c in cases:
        mode = {"ALG1": orc.SEL_MINS_ALG1, "EXACT": orc.SEL_MINS_EXACT}[c["mode"]]
        got = run([c["scores"]], mode=mode, bk=c["bk"], gk=c["gk"], alpha=c["alpha"])
        assert got == [set(c["expect"])], c["name"]


def test_alg1_strict_vs_nonstrict_comparator():
    # Reading R1: '>=' (Eq. 3) -- with alpha=0 the tile max itself is kept.  Alg. 1's
    # literal '>' would select nothing here.
    assert run([[1.0, 1.0, 0.5, 0.2]], mode=orc.SEL_MINS_ALG1, bk=2, gk=2, alpha=0.0) == [{0, 1}]


def test_alg1_group_reset():
    # G_K=1: every tile is its own group (m reset per tile) -> each tile keeps its max
    s = [4, 1, 3, 2.5, 0.5, 0.2]
    assert run([s], mode=orc.SEL_MINS_ALG1, bk=2, gk=1, alpha=0.1) == [{0, 2, 4}]


def _random_scores(rng, R, N):
    return np.round(rng.standard_normal((R, N)) * 4) / 4  # many ties, exact in fp64


@pytest.mark.parametrize("seed", range(5))
def test_superset_chain_alg1_contains_exact(seed):
    # running max <= global max -> ALG1 selection contains EXACT's
    rng = np.random.default_rng(seed)
    s = _random_scores(rng, 4, 200)
    for bk, gk in [(4, 4), (16, 1), (8, 100), (3, 7)]:
        a = run(s, mode=orc.SEL_MINS_ALG1, bk=bk, gk=gk, alpha=0.75)
        e = run(s, mode=orc.SEL_MINS_EXACT, alpha=0.75)
        for x, y in zip(a, e):
            assert y <= x


def test_single_group_max_in_first_tile_equals_exact():
    # Gk*Bk >= N and the row max in the first tile -> ALG1 == EXACT
    rng = np.random.default_rng(7)
    s = _random_scores(rng, 4, 64)
    s[:, 0] = 100.0
    a = run(s, mode=orc.SEL_MINS_ALG1, bk=8, gk=8, alpha=99.0)
    e = run(s, mode=orc.SEL_MINS_EXACT, alpha=99.0)
    assert a == e


@pytest.mark.parametrize("seed", range(3))
def test_mins_monotone_in_alpha_and_nonempty(seed):
    # S:161-162
    rng = np.random.default_rng(seed)
    s = _random_scores(rng, 4, 128)
    for mode in (orc.SEL_MINS_ALG1, orc.SEL_MINS_EXACT):
        prev = None
        for a in [0.0, 0.25, 0.5, 1.0, 2.0, 8.0]:
            cur = run(s, mode=mode, bk=16, gk=2, alpha=a)
            assert all(len(x) >= 1 for x in cur)
            if prev is not None:
                assert all(p <= c for p, c in zip(prev, cur))
            prev = cur


def test_topk_spec_examples():
    # S:136-137
    assert run([[1, 2, 3]], mode=orc.SEL_TOPK, topk=1) == [{2}]
    assert run([[2, 2, 1]], mode=orc.SEL_TOPK, topk=1) == [{0}]


@pytest.mark.parametrize("seed", range(8))
def test_topk_brute_force(seed):
    # Brute force over all C(n,k) subsets: the chosen set maximises sum(s) and is
    # the lexicographically smallest maximiser (= ties to the lowest index).
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(3, 13))
    s = rng.integers(-3, 4, size=n).astype(np.float64)   # heavy ties
    for k in range(1, n + 1):
        best = None
        for sub in itertools.combinations(range(n), k):
            key = (-s[list(sub)].sum(), sub)
            if best is None or key < best:
                best = key
        got = run([s], mode=orc.SEL_TOPK, topk=k)
        assert got == [set(best[1])], (s, k)


def test_topk_matches_torch_topk_distinct():
    rng = np.random.default_rng(9)
    s = rng.standard_normal((4, 300))
    got = run(s, mode=orc.SEL_TOPK, topk=37)
    ref = torch.topk(torch.from_numpy(s), 37, dim=1).indices.numpy()
    assert got == [set(r.tolist()) for r in ref]


def test_topk_keep_frac_budget():
    # north_star toy "keep 25%": k_i = round(0.25*|V_i|) -> 256 of 1024; counts = budget
    rng = np.random.default_rng(10)
    qp = rng.standard_normal((3, 16))
    k = rng.standard_normal((1024, 16))
    off, idx = orc.select(qp, k, pq=64, mode=orc.SEL_TOPK, keep_frac=0.25)
    assert np.all(np.diff(off) == 256)
    # causal: budget follows the visible count |V_i| = (i+1)*64
    off, idx = orc.select(qp, k, pq=64, causal=True, mode=orc.SEL_TOPK, keep_frac=0.25)
    assert np.diff(off).tolist() == [16, 32, 48]


@pytest.mark.parametrize("mode", [orc.SEL_MINS_ALG1, orc.SEL_MINS_EXACT, orc.SEL_TOPK])
def test_causal_safety_and_canonical_form(mode):
    # no selected index exceeds L_i; indices ascending & unique (R9)
    rng = np.random.default_rng(11)
    N, D, pq = 500, 16, 64
    q = orc.round_bf16(rng.standard_normal((N, D)))
    k = orc.round_bf16(rng.standard_normal((N, D)))
    qp = orc.pool(q, pq)
    off, idx = orc.select(qp, k, pq, causal=True, mode=mode, bk=16, gk=2, alpha=0.3, keep_frac=0.3)
    for i in range(qp.shape[0]):
        seg = idx[off[i]:off[i + 1]]
        assert seg.size >= 1
        assert np.all(np.diff(seg) > 0)
        assert seg.max() <= min(N, (i + 1) * pq) - 1


def test_causal_invisible_keys_do_not_raise_max():
    # A huge score on a causally invisible key must not affect ALG1/EXACT thresholds.
    s = np.array([[1.0, 0.5, 100.0, 100.0]])
    qp, k = inject(s)
    # pq=2 rows: block 0 sees keys {0,1}; block 1 sees all four.  Use a 2-row Q_p
    # whose second row scores are the same vector.
    qp2 = np.vstack([qp, qp])
    for mode in (orc.SEL_MINS_ALG1, orc.SEL_MINS_EXACT):
        off, idx = orc.select(qp2, k, pq=2, causal=True, mode=mode, bk=4, gk=1, alpha=0.6)
        assert sel_sets(off, idx)[0] == {0, 1}


def test_thresholds_detail_alg1():
    # thr reports theta = running max - alpha per tile (golden case 1)
    qp, k = inject([[1, 0.5, 3, 2.6, 4, 1]])
    off, idx, thr, js = orc.select(qp, k, pq=1, mode=orc.SEL_MINS_ALG1, bk=2, gk=3, alpha=1.0,
                                   detail=True)
    np.testing.assert_array_equal(thr[0], [0.0, 2.0, 3.0])
    np.testing.assert_array_equal(js[0], [0, 2, 4])


def test_sparsity_full_selection_zero():
    N, pq = 256, 64
    off = np.arange(0, 5 * N, N, dtype=np.int64)
    idx = np.tile(np.arange(N, dtype=np.int32), 4)
    assert orc.sparsity(off, idx, N, pq, causal=False) == 0.0


def test_sparsity_hand_computed():
    """Reading R15, worked by hand.  N = 4, P_q = 2.
    Non-causal, Idx(0) = {1}, Idx(1) = {0, 2, 3}: kept pairs 2*1 + 2*3 = 8 of 16 -> rho = 1/2.
    Causal, Idx(0) = {0, 1}, Idx(1) = {0, 3}: row 0 sees {0}, row 1 {0, 1}, row 2 {0} (3 > 2),
    row 3 {0, 3}: 6 visible pairs of N(N+1)/2 = 10 -> rho = 0.4 (a count of C_i * h_i would
    give 8 and rho = 0.2: it over-counts the diagonal block).
    Ragged, N = 5, P_q = 2, non-causal, Idx = {0} | {1, 4} | {2, 3}: 2*1 + 2*2 + 1*2 = 8 of 25."""
    assert orc.sparsity([0, 1, 4], [1, 0, 2, 3], 4, 2, causal=False) == 0.5
    assert abs(orc.sparsity([0, 2, 4], [0, 1, 0, 3], 4, 2, causal=True) - 0.4) < 1e-15
    assert abs(orc.sparsity([0, 1, 3, 5], [0, 1, 4, 2, 3], 5, 2, causal=False) - (1 - 8 / 25)) < 1e-15
    # full causal selection (every visible key) -> 0
    N, pq = 7, 3
    off, idx = [0], []
    for i in range(3):
        keys = list(range(min(N, (i + 1) * pq)))
        idx += keys
        off.append(len(idx))
    assert orc.sparsity(off, idx, N, pq, causal=True) == 0.0
