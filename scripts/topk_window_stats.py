"""How wide must the windowed-TOPK sample window be?  For every pooled row of a few heads, the
number of sampled keys (stride 8, the hashed offsets of select.cu's tk_sample_k_kernel) scoring
above the row's true k-th largest pooled score, against the sample-rank estimate ks = k * ns / n:
z = (count - ks) / sigma with sigma = sqrt(ns p (1 - p)) (the binomial rank spread select.cu's
window uses, d = c sigma + 8).  Prints the |z| distribution and the rows a window of c sigma + 8
would miss, per workload.  Scores: fp32 torch matmul of the bf16 pooled Q and K (statistics only).

usage: python scripts/topk_window_stats.py   (GPU)"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2603_29494_b200 import synth
import paper_2603_29494_b200.vecattn as va

STRIDE = 8
dev = torch.device("cuda")


def sample_pos(N):
    js = np.arange((N + STRIDE - 1) // STRIDE, dtype=np.uint64)
    h = (js * np.uint64(2654435761)) & np.uint64(0xFFFFFFFF)
    j = js * STRIDE + (h >> np.uint64(16)) % np.uint64(STRIDE)
    return torch.tensor(np.minimum(j, N - 1).astype(np.int64), device=dev)


def stats(wl_name, heads, keep, pq=64):
    wl = synth.WORKLOADS[wl_name]
    q, k, _ = bench.build_inputs(wl, "video", dev, 0, heads)
    qp = va.pool(q, pq).float()
    N, Np, rep = wl.N, (wl.N + pq - 1) // pq, wl.Hq // wl.Hkv
    pos = sample_pos(N)
    zs = []
    for h in range(heads):
        kf = k[0, h // rep].float()
        for r0 in range(0, Np, 256):
            s = qp[0, h, r0:r0 + 256] @ kf.T  # [rows, N]
            rows = torch.arange(r0, min(r0 + 256, Np), device=dev)
            vis = torch.minimum(torch.full_like(rows, N), (rows + 1) * pq) if wl.causal else torch.full_like(rows, N)
            cols = torch.arange(N, device=dev)
            s = torch.where(cols[None, :] < vis[:, None], s, torch.full_like(s, -float("inf")))
            ki = torch.clamp(torch.floor(keep * vis.double() + 0.5), min=1).long()
            srt = torch.sort(s, dim=1, descending=True).values
            theta = srt.gather(1, (ki - 1)[:, None])
            ss = s[:, pos]
            ns = ((vis + STRIDE - 1) // STRIDE).double()
            cnt = (ss > theta).sum(1).double()
            ks = ki.double() * ns / vis.double()
            p = torch.clamp(ki.double() / vis.double(), max=1.0)
            sig = torch.sqrt(ns * p * (1 - p)).clamp(min=1e-9)
            zs.append(((cnt - ks) / sig).cpu().numpy())
    z = np.abs(np.concatenate(zs))
    out = [f"{wl_name} ({heads} heads, {z.size} rows, keep {keep}): |z| median {np.median(z):.2f} "
           f"p99 {np.percentile(z, 99):.2f} p99.99 {np.percentile(z, 99.99):.2f} max {z.max():.2f}"]
    for c in (2.0, 3.0, 4.0, 5.0, 6.0):
        out.append(f"   c = {c}: rows outside c*sigma (before the +8 margin): {int((z > c).sum())}")
    return "\n".join(out)


if __name__ == "__main__":
    va.load()
    for wl_name, heads, keep in (("dit128k", 6, 0.215), ("dit128k", 6, 0.05), ("vlm128k", 8, 0.215), ("hy", 4, 0.3)):
        print(stats(wl_name, heads, keep), flush=True)
