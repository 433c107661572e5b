"""Debug driver: run one sparse case step by step with syncs (used under `timeout`)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2603_29494_b200 import synth
import paper_2603_29494_b200.vecattn as va

def run(kind, B, Hq, Hkv, N, D, pq, causal, sel, skip_attn=False):
    q, k, v = synth.make_inputs(kind, B, Hq, Hkv, N, D, cfg_id=7, device="cpu")
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    cfg = va.SelectConfig(pq=pq, **sel)
    t = time.time()
    off, idx = va.select(qd, kd, cfg, causal=causal)
    torch.cuda.synchronize()
    oh = off.cpu().numpy(); cnt = np.diff(oh)
    Np = (N + pq - 1) // pq
    G = 128 // pq
    print(f"select ok {time.time()-t:.2f}s nnz={oh[-1]} cnt min/med/max={cnt.min()}/{int(np.median(cnt))}/{cnt.max()}", flush=True)
    # expected union lengths
    ih = idx.cpu().numpy()
    lens = []
    for r0 in range(0, B * Hq * Np, Np):
        for mt in range((N + 127) // 128):
            a = ih[oh[r0 + G*mt]:oh[r0 + G*mt + 1]]
            bset = ih[oh[r0 + G*mt + 1]:oh[r0 + G*mt + 2]] if (G == 2 and G*mt + 1 < Np) else []
            lens.append(len(set(a.tolist()) | set(list(bset))))
    print(f"union len max={max(lens)} total={sum(lens)}", flush=True)
    if skip_attn:
        return
    t = time.time()
    o, lse = va.sparse_fwd(qd, kd, vd, off, idx, pq=pq, causal=causal)
    torch.cuda.synchronize()
    print(f"sparse ok {time.time()-t:.2f}s finite={bool(torch.isfinite(o.float()).all())}", flush=True)

CASES = {
  "3": ("video", 1, 4, 2, 8192 + 100, 128, 64, True, dict(mode="alg1", alpha=1.0, gk=16)),
  "3b": ("video", 1, 1, 1, 8192 + 100, 128, 64, True, dict(mode="alg1", alpha=1.0, gk=16)),
  "3c": ("video", 1, 1, 1, 8192, 128, 64, True, dict(mode="alg1", alpha=1.0, gk=16)),
  "3d": ("video", 1, 1, 1, 8192, 128, 64, False, dict(mode="alg1", alpha=1.0, gk=16)),
  "3e": ("gauss", 1, 1, 1, 8192, 128, 64, False, dict(mode="exact", alpha=100.0)),
  "3f": ("gauss", 1, 1, 1, 8192, 128, 64, True, dict(mode="exact", alpha=100.0)),
  "4": ("video", 1, 2, 2, 5000, 128, 128, True, dict(mode="exact", alpha=1.2)),
  "5": ("video", 1, 2, 1, 6000, 64, 64, False, dict(mode="alg1", alpha=1.5, gk=8192)),
  "6": ("gauss", 2, 2, 2, 2000, 128, 64, True, dict(mode="topk", keep_frac=0.2)),
}
if __name__ == "__main__":
    c = CASES[sys.argv[1]]
    run(*c, skip_attn=len(sys.argv) > 2)
