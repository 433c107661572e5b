"""Fraction of the sparse plan's 8-entry groups (at 8-aligned positions of each 64-key chunk)
that are 8 consecutive keys -- the rows a single 8-row TMA tile load could fetch instead of
two tile::gather4s.  dit128k VIDEO selection, first H heads."""
import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2603_29494_b200 import synth
import paper_2603_29494_b200.vecattn as va
wl = synth.WORKLOADS["dit128k"]
H = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dev = torch.device("cuda")
q, k, v = bench.build_inputs(wl, "video", dev, 0, H)
cfg = va.SelectConfig(mode="alg1", pq=64, gk=wl.gk, alpha=1.0039)
off, idx = va.select(q, k, cfg)
pr = va.problem(q, k, False)
cap = idx.numel()
ws = torch.empty(va.sparse_workspace_bytes(pr, 64, cap), dtype=torch.uint8, device=dev)
o = torch.empty_like(q); lse = torch.empty(q.shape[:3], device=dev)
va.sparse_fwd_into(q, k, v, off, idx, 64, o, lse, ws, cap, False)
torch.cuda.synchronize()
wlv = ws[: cap * 4].view(torch.int32).cpu().numpy().astype(np.int64) & 0x0FFFFFFF
base_len = (cap * 4 + 255) // 256 * 256
n_it = (wl.N + 255) // 256
Np = wl.N // 64
lens = ws[base_len: base_len + H * n_it * 12].view(torch.int32).view(-1, 3).cpu().numpy().astype(np.int64)
offh = off.cpu().numpy()
groups = runs = 0
for x in range(H * n_it):
    bh, it = divmod(x, n_it)
    b = offh[bh * Np + 4 * it]
    pos = b
    for L in lens[x]:
        seg = wlv[pos:pos + L]
        pos += L
        nfull = (L // 64) * 64  # full chunks; tail chunk groups counted too
        for c0 in range(0, L, 64):
            ch = seg[c0:c0 + 64]
            ng = len(ch) // 8
            if ng == 0:
                continue
            g = ch[:ng * 8].reshape(ng, 8)
            groups += ng
            runs += int(((g[:, 7] - g[:, 0]) == 7).sum())
print(f"8-groups {groups}, consecutive runs {runs} ({runs / max(1, groups):.3f})")
