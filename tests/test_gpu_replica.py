"""GPU: the fused attention -> all-gather (vecattn_forward_replicated).

The attention epilogue stores every O row into the full-size O buffer of every rank.  On one
GPU the "ranks" are several local buffers (the P2P store path is the same instructions with
local addresses), plus a one-rank torch symmetric-memory buffer (the bench's allocation path).
Checks: the call's heads land at rows head0.. of every replica, bit-identical to
vecattn_forward's O; rows of other heads are untouched; degenerate rows (O_r = V_r) too.
"""
import pytest
import torch

from paper_2603_29494_b200 import synth

pytestmark = pytest.mark.gpu

va = None


@pytest.fixture(scope="module", autouse=True)
def _lib():
    global va
    import paper_2603_29494_b200.vecattn as _va
    _va.load()
    va = _va


CASES = [
    # kind, B, Hq, Hkv, N, D, pq, causal, selection
    ("video", 1, 4, 2, 4096 + 100, 128, 64, False, dict(mode="alg1", alpha=1.0, gk=8192)),
    ("video", 1, 4, 1, 4096 + 36, 128, 64, True, dict(mode="alg1", alpha=1.0, gk=16)),
    ("gauss", 2, 2, 2, 1000, 64, 128, False, dict(mode="exact", alpha=0.5)),
    ("gauss", 1, 2, 1, 1024, 128, 64, True, dict(mode="topk", topk=1)),  # many degenerate causal rows
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}-B{c[1]}-N{c[4]}-D{c[5]}-{'c' if c[7] else 'nc'}-{c[8]['mode']}"
                                             for c in CASES])
def test_replicated_forward_lands_in_every_replica(case):
    kind, B, Hq, Hkv, N, D, pq, causal, sel = case
    dev = torch.device("cuda:0")
    q, k, v = (t.to(dev) for t in synth.make_inputs(kind, B, Hq, Hkv, N, D, cfg_id=3, device="cpu"))
    cfg = va.SelectConfig(pq=pq, **sel)
    o_ref, lse_ref, off_ref, _ = va.forward(q, k, v, cfg, causal=causal)
    torch.cuda.synchronize()
    head0, Htot = 3, Hq + 5
    sentinel = torch.tensor(-7.25, dtype=torch.bfloat16)
    bufs = [torch.full((B, Htot, N, D), sentinel.item(), dtype=torch.bfloat16, device=dev) for _ in range(3)]
    nnz = int(off_ref[-1].item())
    cap = nnz + 1024
    offsets = torch.empty_like(off_ref)
    indices = torch.empty(cap, dtype=torch.int32, device=dev)
    d_nnz = torch.empty(1, dtype=torch.int64, device=dev)
    lse = torch.empty(B, Hq, N, dtype=torch.float32, device=dev)
    pr = va.problem(q, k, causal)
    ws = torch.empty(va.forward_workspace_bytes(pr, cfg, cap), dtype=torch.uint8, device=dev)
    rep = va.replica([b.data_ptr() for b in bufs], 0, head0, Htot)
    va.forward_replicated_into(q, k, v, cfg, offsets, indices, cap, d_nnz, cap, None, lse, rep, ws, causal)
    torch.cuda.synchronize()
    assert torch.equal(lse, lse_ref)
    for b in bufs:
        assert torch.equal(b[:, head0:head0 + Hq], o_ref)
        rest = torch.cat([b[:, :head0], b[:, head0 + Hq:]], dim=1)
        assert bool((rest == sentinel.to(dev)).all()), "rows of other heads were written"
    # with a local output as well
    o = torch.empty_like(q)
    va.forward_replicated_into(q, k, v, cfg, offsets, indices, cap, d_nnz, cap, o, lse, rep, ws, causal)
    torch.cuda.synchronize()
    assert torch.equal(o, o_ref)


def test_replica_argument_errors():
    dev = torch.device("cuda:0")
    q, k, v = (t.to(dev) for t in synth.make_inputs("gauss", 1, 2, 1, 512, 128, cfg_id=3, device="cpu"))
    cfg = va.SelectConfig(pq=64, mode="alg1", alpha=1.0, gk=16)
    pr = va.problem(q, k, False)
    cap = 2 * 512 * 512
    offsets = torch.empty(2 * 8 + 1, dtype=torch.int64, device=dev)
    indices = torch.empty(cap, dtype=torch.int32, device=dev)
    d_nnz = torch.empty(1, dtype=torch.int64, device=dev)
    ws = torch.empty(va.forward_workspace_bytes(pr, cfg, cap), dtype=torch.uint8, device=dev)
    full = torch.empty(1, 4, 512, 128, dtype=torch.bfloat16, device=dev)
    bad = [va.replica([full.data_ptr()], 0, 3, 4),        # head0 + Hq > heads_total
           va.replica([full.data_ptr() + 2], 0, 0, 4),    # misaligned peer
           va.replica([], 0, 0, 4)]                       # no replica and no local output
    for rep in bad:
        with pytest.raises(va.VecAttnError):
            va.forward_replicated_into(q, k, v, cfg, offsets, indices, cap, d_nnz, cap, None, None, rep, ws, False)


def test_symmetric_memory_one_rank():
    """The bench's allocation path: a torch symmetric-memory O over a one-rank NCCL group,
    written through its peer pointers (and its multicast address if the box exposes one)."""
    import os
    import torch.distributed as dist
    import bench
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29561")
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        dev = torch.device("cuda:0")
        B, H, Hkv, N, D = 1, 4, 2, 2048 + 64, 128
        q, k, v = (t.to(dev) for t in synth.make_inputs("video", B, H, Hkv, N, D, cfg_id=5, device="cpu"))
        cfg = va.SelectConfig(pq=64, mode="alg1", alpha=1.0, gk=8192)
        o_ref, _, _, _ = va.forward(q, k, v, cfg, causal=False)
        sg = bench.SymmGather(H, Hkv, B, N, D, 1, 0, torch.bfloat16, dev)
        assert sg.ok, sg.why
        pr = va.problem(q, k, False)
        cap = B * H * ((N + 63) // 64) * N
        offsets = torch.empty(B * H * ((N + 63) // 64) + 1, dtype=torch.int64, device=dev)
        indices = torch.empty(cap, dtype=torch.int32, device=dev)
        d_nnz = torch.empty(1, dtype=torch.int64, device=dev)
        lse = torch.empty(B, H, N, dtype=torch.float32, device=dev)
        ws = torch.empty(va.forward_workspace_bytes(pr, cfg, cap), dtype=torch.uint8, device=dev)

        def compute(g, rng, rep):
            q0, q1, k0, k1 = rng
            va.forward_replicated_into(q[:, q0:q1].contiguous(), k[:, k0:k1].contiguous(), v[:, k0:k1].contiguous(),
                                       cfg, offsets, indices, cap, d_nnz, cap, None, lse[:, q0:q1].contiguous(), rep,
                                       ws, False)
        sg.run(compute)
        torch.cuda.synchronize()
        assert torch.equal(sg.assemble(), o_ref)
    finally:
        if own:
            dist.destroy_process_group()


WIN_CASES = [
    # kind, B, Hq, Hkv, N, D, pq, causal, selection, window cuts (fractions of all items)
    ("video", 1, 4, 2, 4096 + 100, 128, 64, False, dict(mode="alg1", alpha=1.0, gk=8192), (0.3, 0.55)),
    ("video", 2, 3, 1, 3000, 128, 64, True, dict(mode="alg1", alpha=1.0, gk=16), (0.2, 0.71)),
    ("gauss", 1, 2, 2, 2048 + 64, 64, 128, False, dict(mode="exact", alpha=0.5), (0.5, 0.51)),
]


@pytest.mark.parametrize("case", WIN_CASES, ids=[f"{c[0]}-B{c[1]}-H{c[2]}-N{c[4]}-{'c' if c[7] else 'nc'}"
                                                 for c in WIN_CASES])
def test_work_windows_partition_the_items(case):
    """Flattened (head, block) partition: three calls with work windows that cut
    heads mid-way fill exactly the rows of their items -- together the full O and LSE, bit for
    bit -- and leave every other row untouched."""
    kind, B, Hq, Hkv, N, D, pq, causal, sel, cuts = case
    dev = torch.device("cuda:0")
    q, k, v = (t.to(dev) for t in synth.make_inputs(kind, B, Hq, Hkv, N, D, cfg_id=4, device="cpu"))
    cfg = va.SelectConfig(pq=pq, **sel)
    o_ref, lse_ref, off_ref, _ = va.forward(q, k, v, cfg, causal=causal)
    torch.cuda.synchronize()
    n_mt = (N + 255) // 256
    T = B * Hq * n_mt
    b1 = max(1, int(cuts[0] * T))
    bounds = [0, b1, max(b1 + 1, int(cuts[1] * T)), T]
    nnz = int(off_ref[-1].item())
    cap = nnz + 1024
    offsets = torch.empty_like(off_ref)
    indices = torch.empty(cap, dtype=torch.int32, device=dev)
    d_nnz = torch.empty(1, dtype=torch.int64, device=dev)
    pr = va.problem(q, k, causal)
    ws = torch.empty(va.forward_workspace_bytes(pr, cfg, cap), dtype=torch.uint8, device=dev)
    full = torch.full((B, Hq, N, D), -3.5, dtype=torch.bfloat16, device=dev)
    lse_all = torch.full((B, Hq, N), -9.0, dtype=torch.float32, device=dev)
    row_item = (torch.arange(B * Hq, device=dev)[:, None] * n_mt + torch.arange(N, device=dev)[None, :] // 256)
    row_item = row_item.view(B, Hq, N)
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        o_w = torch.full((B, Hq, N, D), 11.0, dtype=torch.bfloat16, device=dev)
        lse_w = torch.full((B, Hq, N), 5.0, dtype=torch.float32, device=dev)
        rep = va.replica([full.data_ptr()], 0, 0, Hq, lo, hi)
        va.forward_replicated_into(q, k, v, cfg, offsets, indices, cap, d_nnz, cap, o_w, lse_w, rep, ws, causal)
        torch.cuda.synchronize()
        assert torch.equal(offsets, off_ref)  # the selection covers every row
        inside = (row_item >= lo) & (row_item < hi)
        assert torch.equal(o_w[inside], o_ref[inside]) and torch.equal(lse_w[inside], lse_ref[inside])
        assert bool((o_w[~inside] == 11.0).all()) and bool((lse_w[~inside] == 5.0).all())
        lse_all[inside] = lse_w[inside]
    assert torch.equal(full, o_ref) and torch.equal(lse_all, lse_ref)


def test_work_window_argument_errors():
    dev = torch.device("cuda:0")
    q, k, v = (t.to(dev) for t in synth.make_inputs("gauss", 1, 2, 1, 512, 128, cfg_id=3, device="cpu"))
    cfg = va.SelectConfig(pq=64, mode="alg1", alpha=1.0, gk=16)
    pr = va.problem(q, k, False)
    cap = 2 * 512 * 512
    offsets = torch.empty(2 * 8 + 1, dtype=torch.int64, device=dev)
    indices = torch.empty(cap, dtype=torch.int32, device=dev)
    d_nnz = torch.empty(1, dtype=torch.int64, device=dev)
    ws = torch.empty(va.forward_workspace_bytes(pr, cfg, cap), dtype=torch.uint8, device=dev)
    o = torch.empty_like(q)
    T = 2 * 2
    for lo, hi in ((2, 2), (3, 1), (-1, 2), (0, T + 1)):
        with pytest.raises(va.VecAttnError):
            va.forward_replicated_into(q, k, v, cfg, offsets, indices, cap, d_nnz, cap, o, None,
                                       va.replica([], 0, 0, 2, lo, hi), ws, False)


def test_item_order_does_not_change_results(tmp_path):
    """The per-head longest-first item order only changes which SM computes an item: O and LSE
    equal the position-order run (VECATTN_ITEM_ORDER=0, read once per process, so the
    reference runs in a subprocess) bit for bit."""
    import os
    import subprocess
    import sys
    dev = torch.device("cuda:0")
    args = ("video", 1, 3, 3, 8192 + 77, 128, 64)
    q, k, v = (t.to(dev) for t in synth.make_inputs(*args[:6], cfg_id=6, device="cpu"))
    cfg = va.SelectConfig(pq=64, mode="alg1", alpha=1.0, gk=8192)
    o, lse, _, _ = va.forward(q, k, v, cfg, causal=False)
    torch.cuda.synchronize()
    out = tmp_path / "ref.pt"
    code = (
        "import torch, sys\n"
        "from paper_2603_29494_b200 import synth\n"
        "import paper_2603_29494_b200.vecattn as va\n"
        f"q, k, v = (t.to('cuda:0') for t in synth.make_inputs(*{args[:6]!r}, cfg_id=6, device='cpu'))\n"
        "cfg = va.SelectConfig(pq=64, mode='alg1', alpha=1.0, gk=8192)\n"
        "o, lse, _, _ = va.forward(q, k, v, cfg, causal=False)\n"
        f"torch.save((o.cpu(), lse.cpu()), {str(out)!r})\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, VECATTN_ITEM_ORDER="0", PYTHONPATH=root)
    subprocess.run([sys.executable, "-c", code], check=True, env=env, cwd=root, timeout=300)
    o_ref, lse_ref = torch.load(out)
    assert torch.equal(o.cpu(), o_ref) and torch.equal(lse.cpu(), lse_ref)
