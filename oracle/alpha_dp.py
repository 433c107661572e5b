"""ORACLE (test infrastructure only): per-head filter-ratio search of Eq. 4 (PAPER.md
P:245-266, "Dynamic Programming for Offline Search of Per-Head Filter Ratios"), written as
its plain definition: among all assignments of one candidate alpha per head, the one with
the largest total performance sum_h Perf_h(alpha_h) whose average sparsity
(1/H) sum_h sp_h(alpha_h) reaches the target rho_T.  Enumerates every assignment
(n_cand ** H), so it is for small cases only.

Reading (R17b): DP[h][rho] of Eq. 4 is "the optimal performance of the first h heads
under an average sparsity of rho"; the state is the running sparsity sum rho*h
(P:258-262), and the target is read as a floor (average sparsity >= rho_T).  Sparsities
are quantised to 1/grid before summing; ties in performance go to the assignment that is
smallest in lexicographic candidate order.

Only tests/ may import this module.
"""
from __future__ import annotations

import itertools

import numpy as np


def quantise(sp, grid: int) -> np.ndarray:
    """Sparsity -> integer units of 1/grid (round half up), as the DP state uses."""
    return np.floor(np.asarray(sp, np.float64) * grid + 0.5).astype(np.int64)


def alpha_search_brute(sp, perf, rho_target: float, grid: int = 1000):
    """sp, perf: [H, n_cand].  Returns (choice [H] int, best_perf) or (None, -inf) if no
    assignment reaches the target."""
    sp = np.asarray(sp, np.float64)
    perf = np.asarray(perf, np.float64)
    H, C = sp.shape
    q = quantise(sp, grid)
    need = int(np.floor(rho_target * grid * H + 0.5))
    best, arg = -np.inf, None
    for combo in itertools.product(range(C), repeat=H):   # lexicographic order
        tot = sum(q[h, c] for h, c in enumerate(combo))
        if tot < need:
            continue
        val = sum(perf[h, c] for h, c in enumerate(combo))
        if val > best:
            best, arg = val, np.array(combo, np.int64)
    return arg, best
