"""Timeline of CTA 0 of the in-library dense attention kernel (attn.cu, GATHER=false) via the
VECATTN_TRACE hook (%globaltimer ns): per 128-key chunk, S ready / P done per tile, PV issue."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_29494_b200.vecattn as va
dev = torch.device("cuda")
H, N, D = 4, 32768, 128
g = torch.Generator(device="cpu").manual_seed(0)
q = torch.randn(1, H, N, D, generator=g).bfloat16().to(dev)
k = torch.randn(1, H, N, D, generator=g).bfloat16().to(dev)
v = torch.randn(1, H, N, D, generator=g).bfloat16().to(dev)
va.dense_fwd(q, k, v, causal=False)
tr = torch.zeros(32 * 4096, dtype=torch.int64, device=dev)
os.environ["VECATTN_TRACE"] = str(tr.data_ptr())
va.dense_fwd(q, k, v, causal=False)
torch.cuda.synchronize()
t = tr.view(32, 4096).cpu().numpy().astype(np.int64)
n = int((t[4] > 0).sum())
t0 = t[t > 0].min()
def st(x): return f"median {np.median(x):.0f} p10 {np.percentile(x, 10):.0f} p90 {np.percentile(x, 90):.0f} (n={len(x)})" if len(x) else "n/a"
def d(a, b): return np.array([t[b, c] - t[a, c] for c in range(4, n - 4) if t[a, c] > 0 and t[b, c] > 0])
print("chunks traced", n)
for a, b, lab in [(6, 7, "softmax tile 0"), (8, 9, "softmax tile 1"), (7, 4, "P0 done -> PV0 issued"), (9, 5, "P1 done -> PV1 issued"),
                  (2, 6, "K landed -> S0 ready"), (6, 10, "t0: SFULL -> S in regs"), (10, 11, "t0: row max"),
                  (11, 12, "t0: exps + P stores issued"), (12, 7, "t0: st wait -> P done"), (4, 5, "PV0 -> PV1 issued"), (6, 8, "S0 ready -> S1 ready")]:
    print(f"{lab:28s}", st(d(a, b)))
x = np.array([t[4, c] for c in range(n) if t[4, c] > 0])
print("period PV0 issue", st(np.diff(x)))
x = np.array([t[6, c] for c in range(n) if t[6, c] > 0])
print("period S0 ready", st(np.diff(x)))
for c in list(range(0, 6)) + list(range(100, 106)):
    print(c, [int(t[e, c] - t0) if t[e, c] > 0 else -1 for e in (2, 6, 7, 4, 8, 9, 5)])
