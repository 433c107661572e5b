"""Pins for the brute-force oracle of the per-head filter-ratio search (Eq. 4):
hand-solved cases, the unconstrained optimum, infeasible targets and monotonicity."""
import numpy as np
import pytest

from oracle.alpha_dp import alpha_search_brute, quantise


def test_hand_solved_two_heads():
    # head 0: alpha in {a0: sp .9 perf .5, a1: sp .5 perf .9}; head 1: {sp .8 perf .6, sp .4 perf .95}
    sp = [[0.9, 0.5], [0.8, 0.4]]
    perf = [[0.5, 0.9], [0.6, 0.95]]
    # target 0.7: (a0,a0)=.85 ok perf 1.1; (a0,a1)=.65 no; (a1,a0)=.65 no; (a1,a1)=.45 no
    c, v = alpha_search_brute(sp, perf, 0.7)
    assert list(c) == [0, 0] and abs(v - 1.1) < 1e-12
    # target 0.65: (a0,a1) perf 1.45 and (a1,a0) perf 1.5 both reach .65 -> (1, 0)
    c, v = alpha_search_brute(sp, perf, 0.65)
    assert list(c) == [1, 0] and abs(v - 1.5) < 1e-12
    # target 0.4: everything feasible -> the unconstrained best (1, 1)
    c, v = alpha_search_brute(sp, perf, 0.4)
    assert list(c) == [1, 1] and abs(v - 1.85) < 1e-12


def test_infeasible_target():
    c, v = alpha_search_brute([[0.5, 0.6]], [[1.0, 0.5]], 0.7)
    assert c is None and v == -np.inf


@pytest.mark.parametrize("seed", range(4))
def test_monotone_in_target_and_feasible(seed):
    rng = np.random.default_rng(seed)
    H, C = 3, 4
    sp = np.sort(rng.uniform(0.3, 0.95, size=(H, C)), axis=1)[:, ::-1]   # larger alpha -> lower sparsity
    perf = np.sort(rng.uniform(0.2, 1.0, size=(H, C)), axis=1)          # ... and higher performance
    prev = np.inf
    for rho in np.linspace(0.3, 0.95, 14):
        c, v = alpha_search_brute(sp, perf, rho)
        if c is None:
            continue
        assert quantise(sp, 1000)[np.arange(H), c].sum() >= int(np.floor(rho * 1000 * H + 0.5))
        assert v <= prev + 1e-12     # a stricter target never helps
        prev = v


def test_quantisation_rounds_half_up():
    assert list(quantise([0.0005, 0.0004999, 0.9995], 1000)) == [1, 0, 1000]
