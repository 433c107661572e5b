"""Host logic of bench.py on CPU: head partition and the GQA alignment of per-rank inputs."""
import torch

import bench
from paper_2603_29494_b200 import synth


def test_head_range_covers_all_heads():
    for H, ws in ((24, 8), (28, 8), (40, 8), (28, 3)):
        got = []
        for r in range(ws):
            h0, h1, hmax = bench.head_range(H, ws, r)
            assert h1 - h0 <= hmax
            got.extend(range(h0, h1))
        assert got == list(range(H))


def test_build_inputs_gqa_mapping_for_unaligned_ranges():
    wl = synth.Workload("tiny_vlm", 1, 28, 4, 256, 64, True, 16, (1, 16, 16), 900)
    full_q, full_k, full_v = bench.build_inputs(wl, "gauss", torch.device("cpu"), 0, 28)
    for ws in (8, 3):
        for r in range(ws):
            h0, h1, _ = bench.head_range(28, ws, r)
            q, k, v = bench.build_inputs(wl, "gauss", torch.device("cpu"), h0, h1)
            assert torch.equal(q, full_q[:, h0:h1])
            nq, nkv = q.shape[1], k.shape[1]
            assert nq % nkv == 0
            for i in range(nq):   # the ABI maps local head i to local KV head i / (nq / nkv)
                g = (h0 + i) // 7
                assert torch.equal(k[:, i // (nq // nkv)], full_k[:, g])
                assert torch.equal(v[:, i // (nq // nkv)], full_v[:, g])


def test_e2e_groups_cover_all_kv_heads_with_small_ends():
    """The pipelined e2e step's KV-head groups partition the heads and start and end with a
    single head, so only one head's H2D and one head's D2H are exposed (bench.e2e_groups)."""
    import bench
    for n in range(1, 65):
        g = bench.e2e_groups(n)
        assert sum(g) == n and min(g) >= 1
        assert g[0] == 1 and g[-1] == 1
        assert max(g) <= 8
