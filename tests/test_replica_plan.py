"""CPU: the head ranges the fused all-gather (bench.SymmGather) hands to
vecattn_forward_replicated.  Over all ranks, the replica rows (head0 + q0 .. head0 + q1) of
every KV-head group tile [0, H) exactly once, uneven splits included (no padding), and each
group's query heads map onto whole local KV heads."""
import pytest

import bench


@pytest.mark.parametrize("H,Hkv,ws", [(24, 24, 1), (24, 24, 2), (24, 24, 8), (28, 4, 8), (28, 4, 3), (40, 40, 8),
                                      (24, 8, 5), (7, 7, 8)])
def test_replica_rows_tile_all_heads(H, Hkv, ws):
    covered = []
    for r in range(ws):
        h0, h1, _ = bench.head_range(H, ws, r)
        nkv, rep = bench.local_kv(H, Hkv, h0, h1)
        for (q0, q1, k0, k1) in bench.kv_groups(H, Hkv, ws, r):
            assert 0 <= q0 < q1 <= h1 - h0
            assert (q1 - q0) == (k1 - k0) * rep and 0 <= k0 < k1 <= nkv
            covered.extend(range(h0 + q0, h0 + q1))
    assert sorted(covered) == list(range(H))
