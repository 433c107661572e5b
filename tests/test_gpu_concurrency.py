"""Concurrent vecattn_forward calls on two streams (the pattern of bench.py's end-to-end step).

bench.py's e2e step runs KV-head groups whose sizes ramp up and down (bench.e2e_groups).
Consecutive groups alternate between two compute streams, each with its own offsets,
indices and workspace buffers. The library's shared state is its per-device cache of TMA
descriptors and kernel attributes and, for non-causal calls, the per-device side stream on
which the CSR emission runs beside the attention kernel (include/vecattn.h). Its kernels are
deterministic, so the grouped, concurrent outputs -- O, LSE and every group's CSR, copied out
on the group's stream before its buffers are reused -- must equal one full call bit for bit.
"""
import pytest
import torch

from paper_2603_29494_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("causal,Hq,Hkv", [(False, 8, 8), (True, 8, 2)])
def test_grouped_two_stream_forward_equals_single_call(causal, Hq, Hkv):
    import bench
    import paper_2603_29494_b200.vecattn as va
    va.load()
    dev = torch.device("cuda:0")
    N, D = 4096 + 64, 128
    q, k, v = synth.make_inputs("video", 1, Hq, Hkv, N, D, cfg_id=21, device="cpu")
    q, k, v = q.to(dev), k.to(dev), v.to(dev)
    cfg = va.SelectConfig(mode="alg1", pq=64, gk=16 if causal else 8192, alpha=0.9 if causal else 1.0)
    o_ref, lse_ref, off_ref, idx_ref = va.forward(q, k, v, cfg, causal=causal)
    torch.cuda.synchronize()

    Np = (N + 63) // 64
    cap = Hq * Np * N  # every (block, key) pair: an upper bound on the selection
    rep = Hq // Hkv
    o = torch.zeros_like(q)
    lse = torch.zeros(q.shape[:3], dtype=torch.float32, device=dev)
    main, s2 = torch.cuda.current_stream(), torch.cuda.Stream(device=dev)
    sets = []
    for st in (main, s2):
        pr = va.problem(q[:, :rep * 3], k[:, :3], causal)
        sets.append((st, torch.empty(Hq * Np + 1, dtype=torch.int64, device=dev),
                     torch.empty(cap, dtype=torch.int32, device=dev), torch.empty(1, dtype=torch.int64, device=dev),
                     torch.empty(va.forward_workspace_bytes(pr, cfg, cap), dtype=torch.uint8, device=dev)))
    s2.wait_stream(main)
    h0 = 0
    saved = []
    for gi, g in enumerate(bench.e2e_groups(Hkv)):
        st, off, idx, nnz, ws = sets[gi % 2]
        k0, k1 = h0, h0 + g
        with torch.cuda.stream(st):
            va.forward_into(q[:, k0 * rep:k1 * rep], k[:, k0:k1], v[:, k0:k1], cfg, off, idx, cap, nnz, cap,
                            o[:, k0 * rep:k1 * rep], lse[:, k0 * rep:k1 * rep], ws, causal)
            # the group's CSR (written partly on the library's side stream, joined into st)
            saved.append((k0 * rep, k1 * rep, off[:g * rep * Np + 1].clone(), idx.clone(), nnz.clone()))
        h0 = k1
    main.wait_stream(s2)
    torch.cuda.synchronize()
    assert torch.equal(o, o_ref)
    assert torch.equal(lse, lse_ref)
    for q0, q1, off_g, idx_g, nnz_g in saved:
        base = int(off_ref[q0 * Np])
        ref_off = off_ref[q0 * Np:q1 * Np + 1] - base
        assert torch.equal(off_g, ref_off)
        n = int(nnz_g.item())
        assert n == int(ref_off[-1])
        assert torch.equal(idx_g[:n], idx_ref[base:base + n])
        assert va.validate_selection(off_g, idx_g[:n], (1, q1 - q0, N, D), 64, causal) == 0
