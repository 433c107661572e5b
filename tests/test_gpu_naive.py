"""GPU parity of the naive materialise-then-filter selection baselines (vecattn_select_naive,
P:203-216, Fig. 5).

  naive minS  must give exactly the fused MINS_EXACT index sets (same tcgen05 accumulators,
              same fp32 threshold) and match the oracle's Eq. 3 up to documented near-ties.
  naive topP  is checked against the fp64 oracle (oracle.select_topp) on the same bf16
              inputs.  The GPU ranks fp32 scores and sums fp32 terms, so sets may differ from
              the oracle's only at the cut: every GPU set must reach mass p, be minimal and be
              a top set under the oracle's fp64 probabilities within 1e-5, and almost all rows
              must agree exactly.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2603_29494_b200 import synth
from tests.parity import bf16_np, compare_selection

pytestmark = pytest.mark.gpu

va = None


@pytest.fixture(scope="module", autouse=True)
def _lib():
    global va
    import paper_2603_29494_b200.vecattn as _va
    _va.load()
    va = _va


def dev():
    return torch.device("cuda:0")


def make(kind, B, Hq, Hkv, N, D, cfg_id=11):
    q, k, v = synth.make_inputs(kind, B, Hq, Hkv, N, D, cfg_id=cfg_id, device="cpu")
    return q, k, q.to(dev()), k.to(dev())


CASES = [  # kind, B, Hq, Hkv, N, D, pq, causal, alpha
    ("gauss", 1, 2, 2, 2048 + 80, 128, 64, False, 0.35),
    ("video", 1, 2, 1, 4096, 128, 64, True, 1.2),
    ("gauss", 2, 2, 1, 3000, 64, 128, False, 0.3),
    ("video", 1, 3, 3, 1024 + 16, 128, 64, True, 0.9),
    ("gauss", 1, 1, 1, 1024 + 3, 128, 64, False, 0.3),   # N % 4 != 0: scalar paths of the filters
]


@pytest.mark.parametrize("case", CASES)
def test_naive_mins_equals_fused_exact(case):
    kind, B, Hq, Hkv, N, D, pq, causal, alpha = case
    q, k, qd, kd = make(kind, B, Hq, Hkv, N, D)
    off_n, idx_n = va.select_naive(qd, kd, "mins", pq=pq, alpha=alpha, causal=causal)
    cfg = va.SelectConfig(mode="exact", pq=pq, alpha=alpha)
    off_f, idx_f = va.select(qd, kd, cfg, causal=causal)
    torch.cuda.synchronize()
    assert torch.equal(off_n, off_f)
    assert torch.equal(idx_n, idx_f)
    # and the oracle (Eq. 3) on one head
    qp = va.pool(qd, pq)
    Np = (N + pq - 1) // pq
    n, nk, ties = compare_selection(off_n.cpu().numpy(), idx_n.cpu().numpy(), bf16_np(qp[0, 0]), bf16_np(k[0, 0]),
                                    pq, np.arange(Np), causal=causal, mode=orc.SEL_MINS_EXACT, alpha=alpha)
    assert ties <= 4


TOPP_CASES = [  # kind, B, Hq, Hkv, N, D, pq, causal, p
    ("gauss", 1, 2, 2, 2048 + 80, 128, 64, False, 0.9),
    ("video", 1, 2, 1, 4096, 128, 64, False, 0.5),
    ("video", 1, 2, 1, 4096 + 40, 128, 64, True, 0.9),
    ("gauss", 1, 1, 1, 3000, 64, 128, True, 0.7),
    ("gauss", 1, 1, 1, 1024 + 3, 128, 64, False, 0.8),   # N % 4 != 0
]


@pytest.mark.parametrize("case", TOPP_CASES)
def test_naive_topp_matches_oracle(case):
    kind, B, Hq, Hkv, N, D, pq, causal, p = case
    q, k, qd, kd = make(kind, B, Hq, Hkv, N, D)
    off, idx = va.select_naive(qd, kd, "topp", pq=pq, top_p=p, causal=causal)
    qp = va.pool(qd, pq)
    torch.cuda.synchronize()
    off_h, idx_h = off.cpu().numpy(), idx.cpu().numpy()
    assert va.validate_selection(off, idx, tuple(qd.shape), pq, causal) == 0
    Np = (N + pq - 1) // pq
    scale = orc.default_scale(D)
    same = rows = 0
    for h in range(Hq):
        kv = h // (Hq // Hkv)
        qph, kh = bf16_np(qp[0, h]), bf16_np(k[0, kv])
        ro, ri = orc.select_topp(qph, kh, pq, p, causal=causal)
        for i in range(Np):
            vend = min(N, (i + 1) * pq) if causal else N
            s = scale * (kh[:vend] @ qph[i])
            a = np.exp(s - s.max())
            a /= a.sum()
            g = idx_h[off_h[h * Np + i]:off_h[h * Np + i + 1]]
            o = ri[ro[i]:ro[i + 1]]
            assert g.size >= 1 and g.max() < vend
            mg = a[g].sum()
            assert mg >= p - 1e-5, f"h{h} row {i}: mass {mg} < p"
            assert mg - a[g].min() < p + 1e-5, f"h{h} row {i}: not minimal"
            out = np.setdiff1d(np.arange(vend), g)
            if out.size:
                assert a[g].min() >= a[out].max() * (1 - 1e-5) - 1e-12, f"h{h} row {i}: not a top set"
            rows += 1
            same += int(np.array_equal(g, o))
    assert same >= 0.95 * rows, f"only {same}/{rows} rows identical to the oracle"


def test_naive_topp_p_one_selects_all_visible():
    q, k, qd, kd = make("gauss", 1, 1, 1, 1024, 128)
    off, idx = va.select_naive(qd, kd, "topp", pq=64, top_p=1.0)
    torch.cuda.synchronize()
    # GAUSS pooled scores are O(1): every key has a nonzero fp32 probability
    assert int(off[-1]) == 16 * 1024


def test_naive_argument_errors():
    q, k, qd, kd = make("gauss", 1, 1, 1, 256, 128)
    with pytest.raises(va.VecAttnError):
        va.select_naive(qd, kd, "topp", top_p=0.0)
    with pytest.raises(va.VecAttnError):
        va.select_naive(qd, kd, "topp", top_p=1.5)
    with pytest.raises(va.VecAttnError):
        va.select_naive(qd, kd, "mins", alpha=-1.0)
