"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

Inputs are built by bench.build_inputs on the bench's workloads with bench's alpha. The
workloads are dit128k (N = 131072, 24 heads, non-causal, the headline), vlm128k
(N = 131072, 28/4 heads, causal) and hy (N = 118800, 24 heads, non-causal; the last query
block and key tile are ragged) and wan (N = 75600, 40 heads, ρ ≈ 0.52). One fused vecattn_forward produces the outputs, and the
dense kernel is checked too.

The oracle computes sampled outputs one at a time:
  * selection: sampled pooled rows of several heads, Alg. 1 with the parity rule's near-tie
    tolerance;
  * attention: sampled query blocks (first, last, random) on the GPU's own index sets, at
    the north-star tolerances;
  * dense: sampled query rows.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2603_29494_b200 import synth
from tests.parity import ATOL_MAX, ATOL_MEAN, LSE_ATOL, bf16_np, compare_selection

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("wl_name,alpha", [("dit128k", 1.0039), ("vlm128k", None),
                                            ("hy", 1.0020),   # HY: N = 118800, a 16-row last block
                                            ("wan", 1.2070)])  # WAN: 40 heads, N = 75600, rho ~ 0.52
def test_full_size_forward_sampled(wl_name, alpha):
    import bench
    import paper_2603_29494_b200.vecattn as va
    va.load()
    wl = synth.WORKLOADS[wl_name]
    dev = torch.device("cuda:0")
    q, k, v = bench.build_inputs(wl, "video", dev, 0, wl.Hq)
    pq = 64
    Np = (wl.N + pq - 1) // pq
    if alpha is None:  # calibrated like bench.py (global alpha for rho = 0.785)
        from paper_2603_29494_b200 import calibrate as cal
        alpha = cal.calibrate_uniform(q, k, va.SelectConfig(mode="alg1", pq=pq, gk=wl.gk), 0.785, causal=wl.causal)
    cfg = va.SelectConfig(mode="alg1", pq=pq, bk=16, gk=wl.gk, alpha=alpha)
    o, lse, off, idx = va.forward(q, k, v, cfg, causal=wl.causal)
    qp = va.pool(q, pq)
    torch.cuda.synchronize()
    off_h, idx_h = off.cpu().numpy(), idx.cpu().numpy()
    assert va.validate_selection(off, idx, tuple(q.shape), pq, wl.causal) == 0
    rng = np.random.default_rng(5)
    rep = wl.Hq // wl.Hkv
    for h in (0, wl.Hq // 2, wl.Hq - 1):
        kv = h // rep
        kh = bf16_np(k[0, kv])
        vh = bf16_np(v[0, kv])
        qh = bf16_np(q[0, h])
        # ---- selection on sampled pooled rows
        rows = np.unique(np.concatenate([[0, Np - 1], rng.choice(Np, 6, replace=False)]))
        n, nk, ties = compare_selection(off_h, idx_h, bf16_np(qp[0, h]), kh, pq, rows, causal=wl.causal,
                                        mode=orc.SEL_MINS_ALG1, bk=16, gk=wl.gk, alpha=alpha, row_base=h * Np)
        assert ties <= 4
        # ---- attention on sampled blocks, on the GPU's own index sets
        hoff = off_h[h * Np:(h + 1) * Np + 1] - off_h[h * Np]
        hidx = idx_h[off_h[h * Np]:off_h[(h + 1) * Np]]
        blocks = np.unique(np.concatenate([[0, Np - 1], rng.choice(Np, 3, replace=False)]))
        oo, ol = orc.sparse_attn(qh, kh, vh, hoff, hidx, pq, causal=wl.causal, blocks=blocks)
        rows_q = (blocks[:, None] * pq + np.arange(pq)[None, :]).reshape(-1)
        ok = rows_q < wl.N
        og = o[0, h].float().cpu().numpy()[rows_q[ok]]
        err = np.abs(og - oo[ok])
        assert err.max() <= ATOL_MAX and err.mean() <= ATOL_MEAN, (wl_name, h, err.max(), err.mean())
        assert np.abs(lse[0, h].cpu().numpy()[rows_q[ok]] - ol[ok]).max() <= LSE_ATOL
    # ---- dense kernel on sampled rows of one head
    od, ld = va.dense_fwd(q[:, :1].contiguous(), k[:, :1].contiguous(), v[:, :1].contiguous(), causal=wl.causal)
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([[0, wl.N - 1], rng.choice(wl.N, 14, replace=False)]))
    do, dl = orc.dense_attn(bf16_np(q[0, 0]), bf16_np(k[0, 0]), bf16_np(v[0, 0]), causal=wl.causal, rows=rows)
    err = np.abs(od[0, 0].float().cpu().numpy()[rows] - do)
    assert err.max() <= ATOL_MAX and err.mean() <= ATOL_MEAN, (wl_name, "dense", err.max(), err.mean())
    assert np.abs(ld[0, 0].cpu().numpy()[rows] - dl).max() <= LSE_ATOL


@pytest.mark.parametrize("mode", ["exact", "topk"])
def test_full_size_exact_and_topk_sampled(mode):
    """dit128k (24 heads, N = 131072) with MINS_EXACT (Eq. 3, alpha calibrated to rho = 0.785)
    and TOPK (keep 21.5% of the keys of every block): sampled pooled rows of three heads vs
    the oracle under the near-tie rule (TOPK: counts equal the budget), and sampled blocks of
    attention on the GPU's own index sets."""
    import bench
    import paper_2603_29494_b200.vecattn as va
    va.load()
    wl = synth.WORKLOADS["dit128k"]
    dev = torch.device("cuda:0")
    q, k, v = bench.build_inputs(wl, "video", dev, 0, wl.Hq)
    pq = 64
    Np = (wl.N + pq - 1) // pq
    if mode == "exact":
        from paper_2603_29494_b200 import calibrate as cal
        alpha = cal.calibrate_uniform(q, k, va.SelectConfig(mode="exact", pq=pq), 0.785, causal=False)
        cfg = va.SelectConfig(mode="exact", pq=pq, alpha=alpha)
        omode, kw = orc.SEL_MINS_EXACT, dict(alpha=alpha)
    else:
        cfg = va.SelectConfig(mode="topk", pq=pq, keep_frac=0.215)
        omode, kw = orc.SEL_TOPK, dict(keep_frac=0.215)
    o, lse, off, idx = va.forward(q, k, v, cfg, causal=False)
    qp = va.pool(q, pq)
    torch.cuda.synchronize()
    off_h, idx_h = off.cpu().numpy(), idx.cpu().numpy()
    assert va.validate_selection(off, idx, tuple(q.shape), pq, False) == 0
    if mode == "topk":
        budget = int(np.floor(0.215 * wl.N + 0.5))
        assert np.all(np.diff(off_h) == budget)
    rng = np.random.default_rng(11)
    for h in (0, 11, 23):
        kh, vh, qh = bf16_np(k[0, h]), bf16_np(v[0, h]), bf16_np(q[0, h])
        rows = np.unique(np.concatenate([[0, Np - 1], rng.choice(Np, 4, replace=False)]))
        n, nk, ties = compare_selection(off_h, idx_h, bf16_np(qp[0, h]), kh, pq, rows, causal=False, mode=omode,
                                        bk=16, gk=wl.gk, row_base=h * Np, **kw)
        assert ties <= 4
        hoff = off_h[h * Np:(h + 1) * Np + 1] - off_h[h * Np]
        hidx = idx_h[off_h[h * Np]:off_h[(h + 1) * Np]]
        blocks = np.unique(np.concatenate([[0, Np - 1], rng.choice(Np, 2, replace=False)]))
        oo, ol = orc.sparse_attn(qh, kh, vh, hoff, hidx, pq, causal=False, blocks=blocks)
        rows_q = (blocks[:, None] * pq + np.arange(pq)[None, :]).reshape(-1)
        og = o[0, h].float().cpu().numpy()[rows_q]
        err = np.abs(og - oo)
        assert err.max() <= ATOL_MAX and err.mean() <= ATOL_MEAN, (mode, h, err.max(), err.mean())
        assert np.abs(lse[0, h].cpu().numpy()[rows_q] - ol).max() <= LSE_ATOL


@pytest.mark.parametrize("causal", [False, True])
def test_worklist_multi_stripe_beyond_262144_keys(causal):
    """N = 300000 > 262144 keys: vecattn_sparse_fwd builds its plan from the CSR in two key
    stripes with a counting pre-pass (worklist_kernel); the fused path builds it from the bitmask
    (plan_kernel).  Both must give the same O bit for bit, and sampled blocks match the oracle."""
    import paper_2603_29494_b200.vecattn as va
    va.load()
    N, D, pq = 300000, 128, 64
    q, k, v = synth.make_inputs("gauss", 1, 1, 1, N, D, cfg_id=23, device="cpu")
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    cfg = va.SelectConfig(mode="topk", pq=pq, keep_frac=0.01)
    o_f, l_f, off, idx = va.forward(qd, kd, vd, cfg, causal=causal)
    o_s, l_s = va.sparse_fwd(qd, kd, vd, off, idx, pq=pq, causal=causal)
    torch.cuda.synchronize()
    assert torch.equal(o_f, o_s) and torch.equal(l_f, l_s)
    Np = (N + pq - 1) // pq
    off_h, idx_h = off.cpu().numpy(), idx.cpu().numpy()
    blocks = np.array([0, 1, Np // 2, Np - 2, Np - 1], np.int64)
    oo, ol = orc.sparse_attn(bf16_np(q[0, 0]), bf16_np(k[0, 0]), bf16_np(v[0, 0]), off_h, idx_h, pq, causal=causal,
                             blocks=blocks)
    rows = (blocks[:, None] * pq + np.arange(pq)[None, :]).reshape(-1)
    ok = rows < N
    err = np.abs(o_s[0, 0].float().cpu().numpy()[rows[ok]] - oo[ok])
    assert err.max() <= ATOL_MAX and err.mean() <= ATOL_MEAN, (err.max(), err.mean())
    assert np.abs(l_s[0, 0].cpu().numpy()[rows[ok]] - ol[ok]).max() <= LSE_ATOL


def test_full_size_work_windows_equal_full_call():
    """dit128k (2 heads, the bench's inputs and alpha): two work windows of
    vecattn_forward_replicated that cut head 0 mid-way write exactly the full call's O into one
    replica, with the per-head longest-first order inside each window."""
    import bench
    import paper_2603_29494_b200.vecattn as va
    va.load()
    wl = synth.WORKLOADS["dit128k"]
    dev = torch.device("cuda:0")
    H = 2
    q, k, v = bench.build_inputs(wl, "video", dev, 0, H)
    cfg = va.SelectConfig(mode="alg1", pq=64, bk=16, gk=wl.gk, alpha=1.0039)
    o_ref, lse_ref, off_ref, _ = va.forward(q, k, v, cfg, causal=False)
    torch.cuda.synchronize()
    T = H * ((wl.N + 255) // 256)
    cap = int(off_ref[-1].item()) + 1024
    offsets = torch.empty_like(off_ref)
    indices = torch.empty(cap, dtype=torch.int32, device=dev)
    d_nnz = torch.empty(1, dtype=torch.int64, device=dev)
    pr = va.problem(q, k, False)
    ws = torch.empty(va.forward_workspace_bytes(pr, cfg, cap), dtype=torch.uint8, device=dev)
    full = torch.zeros_like(q)
    lse = torch.zeros_like(lse_ref)
    for lo, hi in ((0, 301), (301, T)):
        va.forward_replicated_into(q, k, v, cfg, offsets, indices, cap, d_nnz, cap, None, lse,
                                   va.replica([full.data_ptr()], 0, 0, H, lo, hi), ws, False)
    torch.cuda.synchronize()
    assert torch.equal(full, o_ref) and torch.equal(lse, lse_ref)


def test_item_order_fallback_beyond_2048_items_per_head():
    """N > 524288 (more than kLptMaxItems = 2048 items per head): the item order falls back to
    position order inside lpt_order_kernel.  The fused forward still equals the two-call path,
    and two work windows still tile the full call."""
    import paper_2603_29494_b200.vecattn as va
    va.load()
    dev = torch.device("cuda:0")
    N, D = 524288 + 300, 64
    q, k, v = (t.to(dev) for t in synth.make_inputs("gauss", 1, 1, 1, N, D, cfg_id=9, device="cpu"))
    cfg = va.SelectConfig(mode="alg1", pq=64, gk=16, alpha=0.3)
    o, lse, off, idx = va.forward(q, k, v, cfg, causal=False)
    o2, lse2 = va.sparse_fwd(q, k, v, off, idx, pq=64, causal=False)
    torch.cuda.synchronize()
    assert torch.equal(o, o2) and torch.equal(lse, lse2)
    T = (N + 255) // 256
    cap = int(off[-1].item()) + 1024
    offsets = torch.empty_like(off)
    indices = torch.empty(cap, dtype=torch.int32, device=dev)
    d_nnz = torch.empty(1, dtype=torch.int64, device=dev)
    ws = torch.empty(va.forward_workspace_bytes(va.problem(q, k, False), cfg, cap), dtype=torch.uint8, device=dev)
    full = torch.zeros_like(q)
    for lo, hi in ((0, 777), (777, T)):
        va.forward_replicated_into(q, k, v, cfg, offsets, indices, cap, d_nnz, cap, None, None,
                                   va.replica([full.data_ptr()], 0, 0, 1, lo, hi), ws, False)
    torch.cuda.synchronize()
    assert torch.equal(full, o)
