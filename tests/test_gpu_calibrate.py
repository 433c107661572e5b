"""GPU checks of the filter-ratio calibration tool (paper_2603_29494_b200/calibrate.py;
Eq. 4): bisection reaches the target sparsity; per-head tables are reproduced
exactly when the DP's per-head alphas are applied (selection is per head and
deterministic); the DP's recall is never below the best uniform alpha that meets the target
(a uniform assignment is one of the DP's feasible assignments)."""
import numpy as np
import pytest
import torch

from paper_2603_29494_b200 import synth

pytestmark = pytest.mark.gpu


def test_calibration_uniform_and_dp():
    import paper_2603_29494_b200.vecattn as va
    from paper_2603_29494_b200 import calibrate as cal
    va.load()
    q, k, v = synth.make_inputs("video", 1, 4, 4, 4096, 128, cfg_id=21, device="cpu")
    q, k, v = q.cuda(), k.cuda(), v.cuda()
    cfg = va.SelectConfig(mode="alg1", pq=64, gk=8192)
    rho = 0.8
    a = cal.calibrate_uniform(q, k, cfg, rho, causal=False)
    lse_d = cal._dense_lse(q, k, v, False)
    sp_u, rec_u = cal.evaluate(q, k, v, cfg, False, lse_d, alpha=a)
    assert abs(sp_u - rho) < 0.0025
    assert 0.0 < rec_u <= 1.0 + 1e-4
    alphas = list(np.linspace(0.25 * a, 3.0 * a, 9))
    prof = cal.profile_heads(q, k, v, alphas, cfg)
    assert np.all(np.diff(prof.sparsity, axis=1) <= 1e-12)      # larger alpha keeps more keys
    assert np.all(np.diff(prof.recall, axis=1) >= -1e-6)        # ... and more attention mass
    a_h, rec_pred, sp_pred = cal.per_head_alphas(prof, rho)
    sp_m, rec_m = cal.evaluate(q, k, v, cfg, False, prof.extra["lse_dense"], alpha_per_head=a_h)
    assert abs(sp_m - sp_pred) < 1e-9 and abs(rec_m - rec_pred) < 1e-6
    assert sp_m >= rho - 1e-3
    feasible = [c for c in range(len(alphas)) if prof.sparsity[:, c].mean() >= rho - 5e-4]
    if feasible:
        assert rec_m >= max(prof.recall[:, c].mean() for c in feasible) - 1e-6
