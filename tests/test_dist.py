"""Multi-process (gloo, world_size 2) tests of the head-parallel host logic:
head partitioning, the padded all-gather of O (C1) and reassembly.
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


def _worker(rank, ws, port, H, N, D, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from oracle import oracle as orc
    from paper_2603_29494_b200 import synth
    B = 1
    h0, h1, hmax = bench.head_range(H, ws, rank)
    o_local = torch.empty(B, h1 - h0, N, D, dtype=torch.float64)
    for h in range(h0, h1):  # per-head seeded inputs: identical on any rank count
        q = synth.gauss_head(N, D, synth.seed_of(9, 0, h, 0)).double().numpy()
        k = synth.gauss_head(N, D, synth.seed_of(9, 0, h, 1)).double().numpy()
        v = synth.gauss_head(N, D, synth.seed_of(9, 0, h, 2)).double().numpy()
        o, _ = orc.dense_attn(q, k, v)
        o_local[0, h - h0] = torch.from_numpy(o)
    o_pad = torch.zeros(B * hmax * N * D, dtype=torch.float64)
    o_all = torch.empty(ws, B * hmax * N * D, dtype=torch.float64)
    bench.allgather_heads(o_local, o_pad, o_all)
    full = bench.assemble_heads(o_all, B, H, N, D, ws)
    if rank == 0:
        torch.save(full, out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("H", [4, 3])
def test_gloo_allgather_matches_single_rank(tmp_path, H):
    N, D = 96, 16
    out = str(tmp_path / "o.pt")
    mp.spawn(_worker, args=(2, _free_port(), H, N, D, out), nprocs=2, join=True)
    full = torch.load(out)
    from oracle import oracle as orc
    from paper_2603_29494_b200 import synth
    for h in range(H):
        q = synth.gauss_head(N, D, synth.seed_of(9, 0, h, 0)).double().numpy()
        k = synth.gauss_head(N, D, synth.seed_of(9, 0, h, 1)).double().numpy()
        v = synth.gauss_head(N, D, synth.seed_of(9, 0, h, 2)).double().numpy()
        o, _ = orc.dense_attn(q, k, v)
        np.testing.assert_array_equal(full[0, h].numpy(), o)  # bit-identical to 1-rank
