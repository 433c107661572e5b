"""Parity helpers shared by the GPU tests (test code, not product code).

Selection parity rule: GPU and oracle index sets
must be equal for every block except documented near-ties.  A disagreement at
(i, j) is a near-tie iff |s_ij - theta| <= 2^-20 (a_ij + a_ij*) + ulp_fp32(theta),
where theta is the oracle's threshold in force for j's B_K tile (ALG1: running
max - alpha; EXACT: max - alpha; TOPK: k-th largest), j* the key defining it,
and a_ij = scale * sum_d |Q_p[i,d] K[j,d]| (the dot product's absolute scale).
Attention parity is checked on the GPU's own index sets (north_star tolerances:
max-abs 2e-2, mean-abs 2e-3 vs the fp64 oracle; LSE abs 1e-3).
"""
from __future__ import annotations

import numpy as np

from oracle import oracle as orc

ATOL_MAX = 2e-2
ATOL_MEAN = 2e-3
LSE_ATOL = 1e-3
TIE_REL = 2.0 ** -20


def bf16_np(t) -> np.ndarray:
    """torch bf16 tensor -> exact float64 numpy array."""
    return t.detach().float().cpu().double().numpy()


def compare_selection(gpu_off, gpu_idx, qp, k, pq, rows, *, causal, mode, bk=16, gk=16, alpha=0.0, topk=0,
                      keep_frac=0.0, scale=None, row_base=0):
    """Compare GPU CSR rows (absolute row ids row_base + i) with the oracle on rows `rows`
    of one head.  Returns (n_rows, n_keys_compared, n_near_ties); raises on real mismatches."""
    N, D = k.shape
    scale = orc.default_scale(D) if scale is None else scale
    ro, ri, thr, js = orc.select(qp, k, pq, causal=causal, mode=mode, bk=bk, gk=gk, alpha=alpha, topk=topk,
                                 keep_frac=keep_frac, scale=scale, rows=rows, detail=True)
    ties = 0
    nkeys = 0
    for t, i in enumerate(rows):
        g = gpu_idx[gpu_off[row_base + i]:gpu_off[row_base + i + 1]]
        o = ri[ro[t]:ro[t + 1]]
        assert np.all(np.diff(g) > 0), f"row {i}: GPU indices not ascending/unique"
        nkeys += o.size
        if mode == orc.SEL_TOPK:
            assert g.size == o.size, f"row {i}: TOPK count {g.size} != budget {o.size}"
        diff = np.setxor1d(g, o)
        if diff.size == 0:
            continue
        for j in diff:
            tile = j // bk
            theta = thr[t, tile]
            jstar = js[t, tile]
            s_ij = scale * float(qp[i] @ k[j])
            a_ij = scale * float(np.abs(qp[i] * k[j]).sum())
            a_js = scale * float(np.abs(qp[i] * k[jstar]).sum()) if jstar >= 0 else 0.0
            band = TIE_REL * (a_ij + a_js) + float(np.spacing(np.float32(abs(theta))))
            assert abs(s_ij - theta) <= band, (
                f"row {i} key {j}: not a near-tie (s={s_ij!r}, theta={theta!r}, band={band:.3e}, "
                f"gpu_has={j in set(g.tolist())})")
            ties += 1
    return len(rows), nkeys, ties


def check_attn(o_gpu, lse_gpu, o_ref, lse_ref, what=""):
    err = np.abs(o_gpu - o_ref)
    assert np.isfinite(o_gpu).all(), f"{what}: non-finite output"
    assert err.max() <= ATOL_MAX, f"{what}: max-abs {err.max():.3e}"
    assert err.mean() <= ATOL_MEAN, f"{what}: mean-abs {err.mean():.3e}"
    if lse_gpu is not None:
        le = np.abs(lse_gpu - lse_ref)
        assert le.max() <= LSE_ATOL, f"{what}: LSE max-abs {le.max():.3e}"
    return float(err.max()), float(err.mean())
