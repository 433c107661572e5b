"""The library's Eq. 4 dynamic program (vecattn_alpha_dp, host-only C ABI) against the
brute-force oracle (oracle/alpha_dp.py) on random small instances, plus its error cases."""
import numpy as np
import pytest

from oracle.alpha_dp import alpha_search_brute


@pytest.fixture(scope="module")
def va():
    import paper_2603_29494_b200.vecattn as _va
    _va.load()
    return _va


@pytest.mark.parametrize("seed", range(12))
def test_dp_matches_brute_force(va, seed):
    rng = np.random.default_rng(1000 + seed)
    H = int(rng.integers(1, 5))
    C = int(rng.integers(1, 5))
    sp = rng.uniform(0.2, 0.98, size=(H, C)).astype(np.float32)
    perf = rng.uniform(0.0, 1.0, size=(H, C)).astype(np.float32)
    for rho in (0.3, 0.6, 0.75, 0.9):
        ref_c, ref_v = alpha_search_brute(sp.astype(np.float64), perf.astype(np.float64), rho, grid=1000)
        if ref_c is None:
            with pytest.raises(va.VecAttnError):
                va.alpha_dp(sp, perf, rho, 1000)
            continue
        c, v = va.alpha_dp(sp, perf, rho, 1000)
        assert abs(v - ref_v) < 1e-9
        assert list(c) == list(ref_c)


def test_dp_larger_instance_against_brute_force(va):
    rng = np.random.default_rng(7)
    H, C = 6, 5                                 # 15625 assignments
    sp = np.sort(rng.uniform(0.4, 0.97, size=(H, C)), axis=1)[:, ::-1].astype(np.float32)
    perf = np.sort(rng.uniform(0.5, 1.0, size=(H, C)), axis=1).astype(np.float32)
    for rho in (0.6, 0.7, 0.8):
        ref_c, ref_v = alpha_search_brute(sp.astype(np.float64), perf.astype(np.float64), rho, grid=200)
        c, v = va.alpha_dp(sp, perf, rho, 200)
        assert abs(v - ref_v) < 1e-9 and list(c) == list(ref_c)


def test_dp_argument_errors(va):
    sp = np.full((2, 2), 0.5, np.float32)
    with pytest.raises(va.VecAttnError):
        va.alpha_dp(sp, sp, 1.5)
    with pytest.raises(va.VecAttnError):
        va.alpha_dp(sp * 3.0, sp, 0.5)             # sparsity out of [0, 1]
    with pytest.raises(va.VecAttnError):
        va.alpha_dp(sp, np.full((2, 2), np.nan, np.float32), 0.5)
