"""Pins for the oracle's topP (cumulative-mass) selection of the naive approach.

  topP  P:203-216 ("elements are selected such that their cumulative attention scores
        exceed a threshold p"), SPEC S:140-148 (smallest prefix in descending probability,
        ties -> lowest index, p = 1 -> every nonzero-probability column).

Scores are injected exactly as in test_oracle_select.py (D = 4, scale 1/2, Q_p row i =
2 e_i, so s_ij = K[j, i]); probabilities are softmax(s).  Pins: the SPEC worked example,
brute-force enumeration of every key subset (minimal cardinality reaching mass p, and
top-by-probability among those), p = 1, monotonicity in p, the relation to the oracle's
independent TOPK mode, and causal safety.
"""
import itertools

import numpy as np
import pytest

from oracle import oracle as orc
from tests.test_oracle_select import inject, sel_sets


def probs(s):
    s = np.asarray(s, np.float64)
    e = np.exp(s - s.max())
    return e / e.sum()


def topp(score_rows, p, causal=False, pq=1):
    qp, k = inject(score_rows)
    off, idx, mass = orc.select_topp(qp, k, pq, p, causal=causal, scale=0.5, detail=True)
    return sel_sets(off, idx), mass


def test_spec_example():
    # probs = [0.7, 0.2, 0.1], p = 0.7 -> [0]   (s = log probs).  The probability
    # 0.7 is recomputed by softmax in fp64 and lands within an ulp of p, so the exact
    # boundary is pinned from both sides: p just below 0.7 -> {0}, just above -> {0, 1}.
    s = [np.log([0.7, 0.2, 0.1])]
    sets, mass = topp(s, 0.7 - 1e-9)
    assert sets[0] == {0}
    assert abs(mass[0] - 0.7) < 1e-12
    assert topp(s, 0.7 + 1e-9)[0][0] == {0, 1}
    assert topp(s, 0.9 - 1e-9)[0][0] == {0, 1}
    assert topp(s, 0.9 + 1e-9)[0][0] == {0, 1, 2}


def test_p_one_selects_every_nonzero_probability_column():
    s = [0.3, -1.0, 2.0, 0.0, -2000.0]       # exp(-2002) underflows to probability 0
    sets, _ = topp([s], 1.0)
    assert sets[0] == {0, 1, 2, 3}


@pytest.mark.parametrize("seed", range(6))
def test_brute_force_minimal_top_set(seed):
    rng = np.random.default_rng(seed)
    n = 9
    s = rng.normal(size=n) * 1.5
    s[3] = s[5]                                # a tie (lowest index wins)
    a = probs(s)
    for p in (0.2, 0.5, 0.77, 0.9, 0.99):
        sel, mass = topp([s], p)
        sel = sel[0]
        # minimal cardinality among all subsets reaching p
        kmin = min(len(c) for r in range(1, n + 1) for c in itertools.combinations(range(n), r)
                   if a[list(c)].sum() >= p)
        assert len(sel) == kmin
        assert a[list(sel)].sum() >= p and abs(mass[0] - a[list(sel)].sum()) < 1e-12
        # top by probability, ties -> lowest index: the chosen set is the first kmin of the
        # (descending probability, ascending index) order
        order = sorted(range(n), key=lambda j: (-a[j], j))
        assert sel == set(order[:kmin])


@pytest.mark.parametrize("seed", range(3))
def test_monotone_in_p_and_contains_argmax(seed):
    rng = np.random.default_rng(100 + seed)
    s = rng.normal(size=40) * 2.0
    prev = set()
    for p in np.linspace(0.05, 1.0, 20):
        sel = topp([s], float(p))[0][0]
        assert int(np.argmax(s)) in sel
        assert prev <= sel
        prev = sel


@pytest.mark.parametrize("seed", range(3))
def test_equals_topk_of_the_same_size(seed):
    # Independent code path: the oracle's TOPK mode sorts raw scores, topP sorts softmax
    # probabilities; softmax is monotone, so topP(p) == TOPK(k = |topP(p)|).
    rng = np.random.default_rng(200 + seed)
    s = rng.normal(size=(3, 50)) * 1.7
    qp, k = inject(s)
    for p in (0.3, 0.6, 0.95):
        off, idx = orc.select_topp(qp, k, 1, p, scale=0.5)
        for r in range(3):
            kk = int(off[r + 1] - off[r])
            o2, i2 = orc.select(qp, k, 1, mode=orc.SEL_TOPK, topk=kk, scale=0.5, rows=[r])
            assert set(idx[off[r]:off[r + 1]].tolist()) == set(i2.tolist())


def test_causal_excludes_invisible_keys():
    rng = np.random.default_rng(7)
    s = rng.normal(size=(4, 16)) * 3.0
    s[0, 15] = 50.0                            # huge but invisible for row 0 (pq = 2: L_0 = 1)
    qp, k = inject(s)
    off, idx = orc.select_topp(qp, k, 2, 0.9, causal=True, scale=0.5)
    for r in range(4):
        sel = idx[off[r]:off[r + 1]]
        assert sel.size >= 1 and sel.max() <= min(16, (r + 1) * 2) - 1
        assert np.all(np.diff(sel) > 0)
