"""Filter-ratio calibration on the GPU (Eq. 4).

Everything runs through the C ABI; torch only holds device buffers and reduces the per-row
results.
  * ``calibrate_uniform``: one global alpha reaching a target sparsity. It bisects on
    counts-only ``vecattn_select`` calls.
  * ``profile_heads``: for a list of candidate alphas, records per head the sparsity
    sp_h(alpha) and a performance proxy Perf_h(alpha). The proxy is the attention recall,
    the mean over query rows of the fraction of the row's full softmax mass that the
    selected keys keep. It is exp(LSE_sparse - LSE_dense) per row, from ``vecattn_forward``
    and ``vecattn_dense_fwd``. On synthetic inputs this stands in for the task metric the
    paper records offline, which needs real models and is out of scope.
  * ``per_head_alphas``: Eq. 4's dynamic program (``vecattn_alpha_dp``) over those tables.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import vecattn as va


def _head_sparsity(offsets: np.ndarray, B: int, H: int, N: int, pq: int, causal: bool) -> np.ndarray:
    """Per-head sparsity 1 - sum_i C_i h_i / S_tot (reading R15; C_i h_i is exact for
    non-causal rows and an upper bound on the visible pairs for causal diagonal blocks)."""
    Np = (N + pq - 1) // pq
    cnt = np.diff(offsets).astype(np.float64).reshape(B, H, Np)
    i = np.arange(Np)
    h = np.minimum(N, (i + 1) * pq) - i * pq
    tot = N * (N + 1) / 2.0 if causal else float(N) * N
    # causal: C_i h_i over-counts the diagonal block's invisible pairs, so clip at 0
    return np.clip(1.0 - (cnt * h).sum(axis=(0, 2)) / (B * tot), 0.0, 1.0)


def calibrate_uniform(q, k, cfg: va.SelectConfig, rho: float, causal: bool = False, tol: float = 0.0025,
                      ws: va.Workspace | None = None) -> float:
    """Bisection for one global alpha with sparsity rho +- tol (counts-only selects)."""
    B, H, N, D = q.shape
    ws = ws or va.Workspace(q.device)

    def rho_of(a):
        c = va.SelectConfig(mode=cfg.mode, pq=cfg.pq, bk=cfg.bk, gk=cfg.gk, alpha=a)
        pr = va.problem(q, k, causal)
        wbuf = ws.get(va.select_workspace_bytes(pr, c))
        off = torch.empty(B * H * ((N + cfg.pq - 1) // cfg.pq) + 1, dtype=torch.int64, device=q.device)
        nnz = torch.empty(1, dtype=torch.int64, device=q.device)
        va.select_into(q, k, c, off, None, 0, nnz, wbuf, causal)
        return float(_head_sparsity(off.cpu().numpy(), B, H, N, cfg.pq, causal).mean())

    lo, hi = 0.0, 1.0
    while rho_of(hi) > rho and hi < 1e4:
        lo, hi = hi, hi * 2.0
    for _ in range(50):
        mid = 0.5 * (lo + hi)
        r = rho_of(mid)
        if abs(r - rho) < tol:
            return mid
        if r > rho:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


@dataclass
class HeadProfile:
    alphas: list
    sparsity: np.ndarray   # [H, n_cand]
    recall: np.ndarray     # [H, n_cand]
    extra: dict = field(default_factory=dict)


def _dense_lse(q, k, v, causal):
    o, lse = va.dense_fwd(q, k, v, causal=causal, with_lse=True)
    del o
    return lse


def _recall_and_sparsity(q, k, v, cfg, causal, lse_dense):
    """(per-head sparsity, per-head mean recall) of one selection config."""
    B, H, N, D = q.shape
    o, lse, off, idx = va.forward(q, k, v, cfg, causal=causal)
    rec = torch.exp(lse.float() - lse_dense.float()).mean(dim=(0, 2)).cpu().numpy()
    sp = _head_sparsity(off.cpu().numpy(), B, H, N, cfg.pq, causal)
    del o, idx
    return sp, rec


def profile_heads(q, k, v, alphas, cfg: va.SelectConfig, causal: bool = False) -> HeadProfile:
    """sp_h(alpha) and Perf_h(alpha) (= attention recall) for every candidate alpha."""
    lse_dense = _dense_lse(q, k, v, causal)
    H = q.shape[1]
    sp = np.zeros((H, len(alphas)))
    rec = np.zeros((H, len(alphas)))
    for c, a in enumerate(alphas):
        cc = va.SelectConfig(mode=cfg.mode, pq=cfg.pq, bk=cfg.bk, gk=cfg.gk, alpha=float(a))
        sp[:, c], rec[:, c] = _recall_and_sparsity(q, k, v, cc, causal, lse_dense)
    torch.cuda.synchronize()
    return HeadProfile(list(alphas), sp, rec, {"lse_dense": lse_dense})


def per_head_alphas(profile: HeadProfile, rho: float, grid: int = 1000):
    """Eq. 4 (vecattn_alpha_dp): the per-head alpha maximising total recall at average
    sparsity >= rho.  Returns (alphas [H], predicted mean recall, predicted mean sparsity)."""
    choice, best = va.alpha_dp(profile.sparsity, profile.recall, rho, grid)
    H = profile.sparsity.shape[0]
    a = [float(profile.alphas[c]) for c in choice]
    sp = float(np.mean([profile.sparsity[h, choice[h]] for h in range(H)]))
    return a, best / H, sp


def evaluate(q, k, v, cfg: va.SelectConfig, causal: bool, lse_dense, alpha=None, alpha_per_head=None):
    """Measured (mean sparsity, mean recall) of a uniform or per-head alpha."""
    c = va.SelectConfig(mode=cfg.mode, pq=cfg.pq, bk=cfg.bk, gk=cfg.gk, alpha=float(alpha or 0.0),
                        alpha_per_head=alpha_per_head)
    sp, rec = _recall_and_sparsity(q, k, v, c, causal, lse_dense)
    return float(sp.mean()), float(rec.mean())
