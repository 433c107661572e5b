"""Multi-process (gloo, world_size 2) tests of the head-parallel host logic:
head partitioning, the group-wise overlapped all-gather of O (C1) and reassembly.
Per-head compute is the fp64 oracle (test infrastructure), so this runs on CPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def test_head_range_partition():
    for H in (1, 3, 24, 28, 40):
        for ws in (1, 2, 3, 4, 8):
            seen = []
            hmax = 0
            for r in range(ws):
                h0, h1, hm = bench.head_range(H, ws, r)
                assert 0 <= h0 <= h1 <= H
                seen += list(range(h0, h1))
                hmax = max(hmax, h1 - h0)
                assert hm == -(-H // ws)
            assert seen == list(range(H))
            assert hmax == -(-H // ws)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _head_inputs(h, kvh, N, D):
    from paper_2603_29494_b200 import synth
    q = synth.gauss_head(N, D, synth.seed_of(9, 0, h, 0)).double().numpy()
    k = synth.gauss_head(N, D, synth.seed_of(9, 0, kvh, 1)).double().numpy()
    v = synth.gauss_head(N, D, synth.seed_of(9, 0, kvh, 2)).double().numpy()
    return q, k, v


def _worker(rank, ws, port, H, Hkv, N, D, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from oracle import oracle as orc
    B = 1
    h0, h1, _ = bench.head_range(H, ws, rank)
    hg = bench.HeadGather(H, Hkv, B, N, D, ws, rank, torch.float64, "cpu", ngroups=2)
    rep = H // Hkv

    def compute(g, rng, o_out):  # per-group compute; the group's all-gather runs async meanwhile
        q0, q1, _, _ = rng
        for hl in range(q0, q1):
            h = h0 + hl
            q, k, v = _head_inputs(h, h // rep, N, D)
            o, _ = orc.dense_attn(q, k, v)
            o_out[0, hl - q0] = torch.from_numpy(o)

    hg.run(compute)
    full = hg.assemble()
    if rank == 0:
        torch.save(full, out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("H,Hkv", [(4, 4), (3, 3), (7, 1), (6, 2)])
def test_gloo_overlapped_allgather_matches_single_rank(tmp_path, H, Hkv):
    """Group-wise async all-gather (HeadGather) over 2 ranks: the assembled O is bit-identical
    to one rank's computation, including uneven (3 over 2) and GQA-cut (7/1, 6/2) splits."""
    N, D = 96, 16
    out = str(tmp_path / "o.pt")
    mp.spawn(_worker, args=(2, _free_port(), H, Hkv, N, D, out), nprocs=2, join=True)
    full = torch.load(out)
    from oracle import oracle as orc
    for h in range(H):
        q, k, v = _head_inputs(h, h // (H // Hkv), N, D)
        o, _ = orc.dense_attn(q, k, v)
        np.testing.assert_array_equal(full[0, h].numpy(), o)  # bit-identical to 1-rank


def test_kv_groups_cover_local_heads():
    for H, Hkv in ((24, 24), (28, 4), (40, 40), (28, 28)):
        for ws in (1, 2, 4, 8):
            for r in range(ws):
                h0, h1, _ = bench.head_range(H, ws, r)
                groups = bench.kv_groups(H, Hkv, ws, r)
                assert groups[0][0] == 0 and groups[-1][1] == h1 - h0
                for (a0, a1, b0, b1), (c0, _, d0, _) in zip(groups, groups[1:]):
                    assert a1 == c0 and b1 == d0 and a1 > a0
