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


@pytest.mark.parametrize("H,N,ws", [(28, 131072, 8), (28, 65536, 3), (24, 131072, 8), (5, 1000, 4), (40, 75600, 7)])
def test_flat_windows_tile_all_items(H, N, ws):
    """The flattened partition's windows cover every (head, item) exactly once, and differ
    in size by at most one item (no 87.5% cap for 28/8)."""
    n_items = (N + 255) // 256
    seen, sizes = [], []
    for r in range(ws):
        h0, h1, (a, b) = bench.flat_window(H, N, ws, r)
        assert 0 <= a < b <= (h1 - h0) * n_items and 0 <= h0 < h1 <= H
        seen.extend(range(h0 * n_items + a, h0 * n_items + b))
        sizes.append(b - a)
    assert sorted(seen) == list(range(H * n_items))
    assert max(sizes) - min(sizes) <= 1
