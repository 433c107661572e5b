"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the
same seeded inputs.  Sizes span several 128-row / 256-key tiles plus ragged
tails; edge cases cover empty-visibility causal rows, GQA, P_q=128, D=64.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2603_29494_b200 import synth
from tests.parity import bf16_np, check_attn, compare_selection

pytestmark = pytest.mark.gpu

va = None


@pytest.fixture(scope="module", autouse=True)
def _lib():
    global va
    import paper_2603_29494_b200.vecattn as _va
    _va.load()  # fails loudly if the CUDA library is missing
    va = _va
    torch.manual_seed(0)


def dev():
    return torch.device("cuda:0")


def make(kind, B, Hq, Hkv, N, D, cfg_id=7):
    q, k, v = synth.make_inputs(kind, B, Hq, Hkv, N, D, cfg_id=cfg_id, device="cpu")
    return q, k, v, q.to(dev()), k.to(dev()), v.to(dev())


# ------------------------------------------------------------------------ pooling
@pytest.mark.parametrize("N,D,pq", [(1024, 64, 64), (4096 + 80, 128, 64), (3000, 128, 128), (64, 64, 64),
                                    (37, 128, 64)])
def test_pool_bit_exact(N, D, pq):
    q, k, v, qd, kd, vd = make("gauss", 2, 3, 1, N, D)
    qp = va.pool(qd, pq)
    torch.cuda.synchronize()
    for b in range(2):
        for h in range(3):
            ref = orc.pool(bf16_np(q[b, h]), pq)
            np.testing.assert_array_equal(bf16_np(qp[b, h]), ref)


def test_pool_bit_exact_video_wide_range():
    q, k, v, qd, kd, vd = make("video", 1, 2, 1, 64 * 50 + 17, 128)
    q = q * torch.tensor(1e3, dtype=torch.bfloat16)
    qp = va.pool(q.to(dev()), 64)
    torch.cuda.synchronize()
    for h in range(2):
        np.testing.assert_array_equal(bf16_np(qp[0, h]), orc.pool(bf16_np(q[0, h]), 64))


# --------------------------------------------------------------- selection GEMM
@pytest.mark.parametrize("N,D,pq", [(1024, 64, 64), (5000, 128, 64), (2048 + 64, 128, 128)])
def test_pooled_scores_gemm(N, D, pq):
    q, k, v, qd, kd, vd = make("gauss", 1, 2, 1, N, D)
    s = va.debug_scores(qd, kd, pq).cpu().numpy().astype(np.float64)
    qp = va.pool(qd, pq)
    Np = (N + pq - 1) // pq
    for h in range(2):
        qph = bf16_np(qp[0, h])
        ref = qph @ bf16_np(k[0, 0]).T
        scale_abs = np.abs(qph) @ np.abs(bf16_np(k[0, 0])).T
        got = s[h * Np:(h + 1) * Np]
        assert np.all(np.isfinite(got))
        assert np.all(np.abs(got - ref) <= 1e-5 * scale_abs + 1e-30)


# ---------------------------------------------------------------------- selection
SEL_CASES = [
    # kind, B, Hq, Hkv, N, D, pq, causal, mode, bk, gk, alpha, topk, keep_frac
    ("gauss", 1, 2, 1, 1024, 64, 64, False, "topk", 16, 16, 0.0, 0, 0.25),
    ("gauss", 1, 2, 2, 4096 + 96, 128, 64, False, "alg1", 16, 16, 0.4, 0, 0.0),
    ("video", 1, 4, 2, 8192 + 100, 128, 64, True, "alg1", 16, 16, 1.0, 0, 0.0),
    ("video", 1, 2, 1, 6000, 128, 64, False, "alg1", 16, 8192, 1.5, 0, 0.0),
    ("gauss", 2, 2, 1, 3000, 128, 64, False, "exact", 16, 16, 0.3, 0, 0.0),
    ("video", 1, 2, 2, 5000, 128, 128, True, "exact", 16, 16, 1.2, 0, 0.0),
    ("gauss", 1, 2, 1, 4100, 128, 64, True, "topk", 16, 16, 0.0, 0, 0.3),
    ("gauss", 1, 1, 1, 2048, 64, 64, False, "topk", 16, 16, 0.0, 100, 0.0),
    ("video", 1, 2, 1, 4096, 128, 64, False, "alg1", 32, 4, 1.0, 0, 0.0),
    ("video", 1, 2, 1, 4096, 128, 64, True, "alg1", 64, 3, 1.0, 0, 0.0),
    # B_K below and above one 64-key TMEM chunk (B_K > 64: sub-tile max read ahead across chunks)
    ("video", 1, 2, 1, 5000 + 33, 128, 64, True, "alg1", 8, 5, 1.0, 0, 0.0),
    ("video", 1, 2, 2, 5000 + 33, 128, 64, False, "alg1", 128, 3, 1.0, 0, 0.0),
    ("video", 1, 2, 1, 6000 + 7, 64, 64, True, "alg1", 256, 2, 1.0, 0, 0.0),
    ("video", 1, 1, 1, 40000 + 37, 128, 64, False, "alg1", 128, 8192, 1.0, 0, 0.0),
    # TOPK rows longer than one 16K-key histogram segment: per-segment histograms are summed
    ("video", 1, 1, 1, 40000 + 37, 128, 64, True, "topk", 16, 16, 0.0, 0, 0.2),
    ("gauss", 1, 1, 1, 33000, 128, 64, False, "topk", 16, 16, 0.0, 500, 0.0),
]


@pytest.mark.parametrize("case", SEL_CASES, ids=[f"{c[0]}-N{c[4]}-{c[8]}-{'c' if c[7] else 'nc'}-pq{c[6]}"
                                                 for c in SEL_CASES])
def test_selection_matches_oracle(case):
    kind, B, Hq, Hkv, N, D, pq, causal, mode, bk, gk, alpha, topk, keep_frac = case
    q, k, v, qd, kd, vd = make(kind, B, Hq, Hkv, N, D)
    cfg = va.SelectConfig(mode=mode, pq=pq, bk=bk, gk=gk, alpha=alpha, topk=topk, keep_frac=keep_frac)
    off, idx = va.select(qd, kd, cfg, causal=causal)
    qp = va.pool(qd, pq)
    torch.cuda.synchronize()
    off_h, idx_h = off.cpu().numpy(), idx.cpu().numpy()
    assert va.validate_selection(off, idx, tuple(qd.shape), pq, causal) == 0
    Np = (N + pq - 1) // pq
    omode = {"alg1": orc.SEL_MINS_ALG1, "exact": orc.SEL_MINS_EXACT, "topk": orc.SEL_TOPK}[mode]
    total_ties = 0
    for b in range(B):
        for h in range(Hq):
            kv = h // (Hq // Hkv)
            rows = np.arange(Np)
            n, nk, ties = compare_selection(off_h, idx_h, bf16_np(qp[b, h]), bf16_np(k[b, kv]), pq, rows,
                                            causal=causal, mode=omode, bk=bk, gk=gk, alpha=alpha, topk=topk,
                                            keep_frac=float(np.float32(keep_frac)), row_base=(b * Hq + h) * Np)
            total_ties += ties
    assert total_ties <= max(4, int(1e-4 * idx_h.size))


def test_selection_capacity_protocol():
    q, k, v, qd, kd, vd = make("gauss", 1, 1, 1, 2048, 128)
    cfg = va.SelectConfig(mode="alg1", pq=64, alpha=0.4)
    pr = va.problem(qd, kd, False)
    ws = torch.empty(va.select_workspace_bytes(pr, cfg), dtype=torch.uint8, device=dev())
    off = torch.empty(33, dtype=torch.int64, device=dev())
    nnz = torch.empty(1, dtype=torch.int64, device=dev())
    va.select_into(qd, kd, cfg, off, None, 0, nnz, ws, False)       # counts-only call
    n = int(nnz.item())
    small = torch.full((max(1, n // 2),), -7, dtype=torch.int32, device=dev())
    va.select_into(qd, kd, cfg, off, small, small.numel(), nnz, ws, False)  # too small: untouched
    assert int(nnz.item()) == n and int(off[-1].item()) == n
    assert bool((small == -7).all())
    full = torch.empty(n, dtype=torch.int32, device=dev())
    va.select_into(qd, kd, cfg, off, full, n, nnz, ws, False)
    off2, idx2 = va.select(qd, kd, cfg)
    assert torch.equal(full, idx2) and torch.equal(off, off2)


# ---------------------------------------------------------------------- attention
def _rows_sample(N, n=256, seed=0):
    rng = np.random.default_rng(seed)
    rows = set([0, 1, N - 1, N // 2]) | set(rng.integers(0, N, n).tolist())
    return np.array(sorted(rows), np.int64)


@pytest.mark.parametrize("N,D,causal,Hq,Hkv", [(1024, 64, False, 1, 1), (4096 + 80, 128, False, 2, 1),
                                               (3000, 128, True, 4, 2), (300, 64, True, 1, 1),
                                               (128, 128, False, 1, 1)])
def test_dense_matches_oracle(N, D, causal, Hq, Hkv):
    q, k, v, qd, kd, vd = make("gauss", 1, Hq, Hkv, N, D)
    o, lse = va.dense_fwd(qd, kd, vd, causal=causal)
    torch.cuda.synchronize()
    rows = _rows_sample(N)
    for h in range(Hq):
        kv = h // (Hq // Hkv)
        ro, rl = orc.dense_attn(bf16_np(q[0, h]), bf16_np(k[0, kv]), bf16_np(v[0, kv]), causal=causal, rows=rows)
        check_attn(bf16_np(o[0, h])[rows], lse[0, h].cpu().numpy()[rows], ro, rl, f"dense h{h}")


SPARSE_CASES = [
    ("gauss", 1, 1, 1, 1024, 64, 64, False, dict(mode="topk", keep_frac=0.25)),
    ("gauss", 1, 2, 1, 4096 + 96, 128, 64, False, dict(mode="alg1", alpha=0.4, gk=16)),
    ("video", 1, 4, 2, 8192 + 100, 128, 64, True, dict(mode="alg1", alpha=1.0, gk=16)),
    ("video", 1, 2, 2, 5000, 128, 128, True, dict(mode="exact", alpha=1.2)),
    ("video", 1, 2, 1, 6000, 64, 64, False, dict(mode="alg1", alpha=1.5, gk=8192)),
    ("gauss", 2, 2, 2, 2000, 128, 64, True, dict(mode="topk", keep_frac=0.2)),
    # kernel coverage: 128-key gather kernel at D=64 (causal), double-buffered kernel at
    # P_q=128 and with B=2 (non-causal)
    ("video", 1, 2, 1, 3000 + 40, 64, 64, True, dict(mode="alg1", alpha=1.2, gk=16)),
    ("gauss", 1, 2, 2, 4096 + 40, 128, 128, False, dict(mode="alg1", alpha=0.3, gk=8192)),
    ("video", 2, 2, 1, 3000, 128, 64, False, dict(mode="exact", alpha=1.4)),
    # tiny / ragged problems: one partial item, last block of 1 row
    ("gauss", 1, 1, 1, 65, 128, 64, False, dict(mode="alg1", alpha=0.5, gk=16)),
    ("gauss", 1, 2, 1, 100, 64, 64, True, dict(mode="alg1", alpha=0.5, gk=16)),
    ("gauss", 1, 1, 1, 200, 128, 128, True, dict(mode="topk", keep_frac=0.5)),
]


@pytest.mark.parametrize("case", SPARSE_CASES, ids=[f"{c[0]}-N{c[4]}-D{c[5]}-pq{c[6]}-{'c' if c[7] else 'nc'}"
                                                    for c in SPARSE_CASES])
def test_sparse_attention_matches_oracle(case):
    kind, B, Hq, Hkv, N, D, pq, causal, sel = case
    q, k, v, qd, kd, vd = make(kind, B, Hq, Hkv, N, D)
    cfg = va.SelectConfig(pq=pq, **sel)
    off, idx = va.select(qd, kd, cfg, causal=causal)
    o, lse = va.sparse_fwd(qd, kd, vd, off, idx, pq=pq, causal=causal)
    torch.cuda.synchronize()
    off_h, idx_h = off.cpu().numpy(), idx.cpu().numpy()
    Np = (N + pq - 1) // pq
    rng = np.random.default_rng(1)
    blocks = sorted(set([0, 1, Np - 1, Np - 2]) | set(rng.integers(0, Np, 12).tolist()))
    blocks = np.array([b_ for b_ in blocks if 0 <= b_ < Np], np.int64)
    for b in range(B):
        for h in range(Hq):
            kv = h // (Hq // Hkv)
            r0 = (b * Hq + h) * Np
            ho = off_h[r0:r0 + Np + 1] - off_h[r0]
            hi = idx_h[off_h[r0]:off_h[r0 + Np]]
            ro, rl = orc.sparse_attn(bf16_np(q[b, h]), bf16_np(k[b, kv]), bf16_np(v[b, kv]), ho, hi, pq,
                                     causal=causal, blocks=blocks)
            rows = (blocks[:, None] * pq + np.arange(pq)[None, :]).reshape(-1)
            ok = rows < N
            got = bf16_np(o[b, h])[rows[ok]]
            gl = lse[b, h].cpu().numpy()[rows[ok]]
            check_attn(got, gl, ro[ok], rl[ok], f"sparse b{b} h{h}")


def test_sparse_full_selection_equals_dense():
    N, D = 2048 + 64, 128
    q, k, v, qd, kd, vd = make("gauss", 1, 2, 1, N, D)
    for causal in (False, True):
        cfg = va.SelectConfig(mode="exact", pq=64, alpha=1e6)  # keeps every visible key
        off, idx = va.select(qd, kd, cfg, causal=causal)
        o, lse = va.sparse_fwd(qd, kd, vd, off, idx, pq=64, causal=causal)
        od, lsed = va.dense_fwd(qd, kd, vd, causal=causal)
        torch.cuda.synchronize()
        assert (o.float() - od.float()).abs().max().item() <= 1.6e-2
        assert (lse - lsed).abs().max().item() <= 1e-3


@pytest.mark.parametrize("scale", [None, 2e-3])
def test_sparse_degenerate_rows_and_empty_blocks(scale):
    # causal block 0 selects only its last key -> rows 0..62 see nothing -> O_r = V_r (R6);
    # a non-causal block with an empty list -> all its rows take V_r.  A small caller scale
    # (2e-3 < 0.0055) checks that degenerate rows are still detected (the masked
    # score is -2^100 * scale, so the threshold must scale with it).
    N, D, pq = 256, 128, 64
    q, k, v, qd, kd, vd = make("gauss", 1, 1, 1, N, D)
    sets = [[63], [5, 64, 100], [], [0, 200, 255]]
    off = torch.tensor(np.concatenate([[0], np.cumsum([len(s) for s in sets])]), dtype=torch.int64, device=dev())
    idx = torch.tensor(sum(sets, []), dtype=torch.int32, device=dev())
    for causal in (True, False):
        o, lse = va.sparse_fwd(qd, kd, vd, off, idx, pq=pq, causal=causal, scale=scale)
        torch.cuda.synchronize()
        ro, rl = orc.sparse_attn(bf16_np(q[0, 0]), bf16_np(k[0, 0]), bf16_np(v[0, 0]), off.cpu().numpy(),
                                 idx.cpu().numpy(), pq, causal=causal, scale=scale)
        check_attn(bf16_np(o[0, 0]), lse[0, 0].cpu().numpy(), ro, rl, f"degenerate causal={causal} scale={scale}")


# ------------------------------------------------------------------ fused forward
FWD_CASES = [
    ("video", 1, 4, 2, 8192 + 100, 128, 64, True, dict(mode="alg1", alpha=1.0, gk=16)),
    ("gauss", 1, 2, 1, 4096 + 96, 128, 64, False, dict(mode="alg1", alpha=0.4, gk=16)),
    ("video", 1, 2, 2, 5000, 128, 128, True, dict(mode="exact", alpha=1.2)),
    ("gauss", 1, 1, 1, 1024, 64, 64, False, dict(mode="topk", keep_frac=0.25)),
    ("video", 1, 2, 1, 6000, 64, 64, False, dict(mode="alg1", alpha=1.5, gk=8192)),
]


@pytest.mark.parametrize("case", FWD_CASES, ids=[f"{c[0]}-N{c[4]}-D{c[5]}-pq{c[6]}-{'c' if c[7] else 'nc'}"
                                                 for c in FWD_CASES])
def test_fused_forward_equals_two_call_path_and_oracle(case):
    kind, B, Hq, Hkv, N, D, pq, causal, sel = case
    q, k, v, qd, kd, vd = make(kind, B, Hq, Hkv, N, D)
    cfg = va.SelectConfig(pq=pq, **sel)
    o, lse, off, idx = va.forward(qd, kd, vd, cfg, causal=causal)
    off2, idx2 = va.select(qd, kd, cfg, causal=causal)
    o2, lse2 = va.sparse_fwd(qd, kd, vd, off2, idx2, pq=pq, causal=causal)
    torch.cuda.synchronize()
    assert torch.equal(off, off2) and torch.equal(idx, idx2)      # same selection, same CSR
    assert torch.equal(o, o2) and torch.equal(lse, lse2)          # same plan order -> bit-identical
    off_h, idx_h = off.cpu().numpy(), idx.cpu().numpy()
    Np = (N + pq - 1) // pq
    blocks = np.array(sorted(set([0, Np // 2, Np - 1])), np.int64)
    for h in range(Hq):
        kv = h // (Hq // Hkv)
        r0 = h * Np
        ro, rl = orc.sparse_attn(bf16_np(q[0, h]), bf16_np(k[0, kv]), bf16_np(v[0, kv]),
                                 off_h[r0:r0 + Np + 1] - off_h[r0], idx_h[off_h[r0]:off_h[r0 + Np]], pq,
                                 causal=causal, blocks=blocks)
        rows = (blocks[:, None] * pq + np.arange(pq)[None, :]).reshape(-1)
        ok = rows < N
        check_attn(bf16_np(o[0, h])[rows[ok]], lse[0, h].cpu().numpy()[rows[ok]], ro[ok], rl[ok], f"fwd h{h}")


def test_fused_forward_capacity_protocol():
    q, k, v, qd, kd, vd = make("gauss", 1, 1, 1, 2048, 128)
    cfg = va.SelectConfig(mode="alg1", pq=64, alpha=0.4)
    pr = va.problem(qd, kd, False)
    off = torch.empty(33, dtype=torch.int64, device=dev())
    nnz = torch.empty(1, dtype=torch.int64, device=dev())
    o = torch.full_like(qd, 7.0)
    lse = torch.empty(1, 1, 2048, device=dev())
    small = 16
    ws = torch.empty(va.forward_workspace_bytes(pr, cfg, small), dtype=torch.uint8, device=dev())
    va.forward_into(qd, kd, vd, cfg, off, None, 0, nnz, small, o, lse, ws, False)
    n = int(nnz.item())
    assert n > small and bool((o == 7.0).all())   # plan capacity too small: attention skipped
    o2, lse2, off2, idx2 = va.forward(qd, kd, vd, cfg, nnz_cap=small)  # binding retries with nnz
    assert idx2.numel() == n


@pytest.mark.parametrize("nsplit", [2, 3, 8])
def test_alg1_k_split_equals_sequential(nsplit, monkeypatch):
    """a single-group ALG1 row split into key segments (segment maxima, then each
    segment starts from the max of the earlier ones) gives exactly the sequential result."""
    q, k, v, qd, kd, vd = make("video", 1, 2, 1, 4096 + 300, 128)
    cfg = va.SelectConfig(mode="alg1", pq=64, gk=8192, alpha=1.1)
    monkeypatch.setenv("VECATTN_SELECT_SPLIT", "1")
    off1, idx1 = va.select(qd, kd, cfg)
    monkeypatch.setenv("VECATTN_SELECT_SPLIT", str(nsplit))
    off2, idx2 = va.select(qd, kd, cfg)
    o2, lse2, off3, idx3 = va.forward(qd, kd, vd, cfg)
    torch.cuda.synchronize()
    assert torch.equal(off1, off2) and torch.equal(idx1, idx2)
    assert torch.equal(off1, off3) and torch.equal(idx1, idx3)
