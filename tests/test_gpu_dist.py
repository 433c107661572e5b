"""C1 on the GPU: the group-wise overlapped NCCL all-gather of O that
bench.py runs at N > 1 (bench.HeadGather + vecattn_forward per KV-head group) assembles an
O that is bit-identical to one vecattn_forward over all heads.  World size = the visible
GPU count, capped at 2 (1 on the driver's box: NCCL with one rank still runs the
collective and the group/async plumbing)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
from paper_2603_29494_b200 import synth
import paper_2603_29494_b200.vecattn as va

CASES = [  # (H, Hkv, N, causal, gk, alpha)
    (6, 6, 4096 + 100, False, 8192, 1.0),
    (7, 1, 2048 + 64, True, 16, 1.0),
]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _wl(H, Hkv, N, causal, gk):
    return synth.Workload("t", 1, H, Hkv, N, 128, causal, gk, None, 77)


def _worker(rank, ws, port, case, out):
    H, Hkv, N, causal, gk, alpha = case
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=ws)
    dev = torch.device("cuda", rank)
    wl = _wl(H, Hkv, N, causal, gk)
    h0, h1, _ = bench.head_range(H, ws, rank)
    q, k, v = bench.build_inputs(wl, "video", dev, h0, h1)
    cfg = va.SelectConfig(mode="alg1", pq=64, gk=gk, alpha=alpha)
    hg = bench.HeadGather(H, Hkv, 1, N, 128, ws, rank, torch.bfloat16, dev, ngroups=3)

    def compute(g, rng, o_out):
        q0, q1, k0, k1 = rng
        o, _, _, _ = va.forward(q[:, q0:q1].contiguous(), k[:, k0:k1].contiguous(), v[:, k0:k1].contiguous(),
                                cfg, causal=causal)
        o_out.copy_(o)

    hg.run(compute)
    full = hg.assemble()
    torch.cuda.synchronize()
    if rank == 0:
        torch.save(full.cpu(), out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=["dit-6h", "vlm-gqa-7h"])
def test_nccl_overlapped_allgather_bit_identical(tmp_path, case):
    H, Hkv, N, causal, gk, alpha = case
    ws = max(1, min(2, torch.cuda.device_count()))
    out = str(tmp_path / "o.pt")
    if ws == 1:
        _worker(0, 1, _port(), case, out)
    else:
        mp.spawn(_worker, args=(ws, _port(), case, out), nprocs=ws, join=True)
    full = torch.load(out)
    dev = torch.device("cuda", 0)
    q, k, v = bench.build_inputs(_wl(H, Hkv, N, causal, gk), "video", dev, 0, H)
    cfg = va.SelectConfig(mode="alg1", pq=64, gk=gk, alpha=alpha)
    o, _, _, _ = va.forward(q, k, v, cfg, causal=causal)
    torch.cuda.synchronize()
    assert torch.equal(full, o.cpu())
