"""Windowed TOPK (select.cu: sampled passes -> window -> candidate pass -> exact select, radix
fallback for rows the window missed) against the radix-pass TOPK (VECATTN_TOPK_RADIX=1) and
against itself with every row forced onto the fallback: the CSR must be bit-identical (the
k-th largest and the lowest-index tie rule R12 are unique).  The oracle parity of TOPK is in
test_gpu_parity.py / test_gpu_fullsize.py."""
import numpy as np
import pytest
import torch

from paper_2603_29494_b200 import synth

pytestmark = pytest.mark.gpu

CASES = [
    # kind, Hq, Hkv, N, D, pq, causal, topk, keep_frac, tie_period
    ("video", 2, 1, 16384 + 100, 128, 64, False, 0, 0.215, 0),
    ("video", 2, 2, 12000, 128, 64, True, 0, 0.3, 0),
    ("gauss", 1, 1, 33000, 128, 64, False, 500, 0.0, 0),
    ("gauss", 2, 1, 5000, 64, 128, True, 0, 0.5, 0),
    ("gauss", 1, 1, 9000, 128, 64, False, 0, 0.25, 37),    # every score repeats: ties at the cut
    ("gauss", 1, 1, 9000, 128, 64, False, 0, 0.25, 13),    # > 512 in the cut's bin: exact radix path
    ("gauss", 1, 1, 9000, 128, 64, True, 0, 0.4, 7),       # > 1024 ties: radix fallback rows
    ("gauss", 1, 1, 300, 128, 64, True, 0, 0.9, 0),         # tiny rows, keep ~everything
    ("gauss", 1, 1, 4096, 128, 64, False, 0, 1.0, 0),       # keep all
]


def _run(monkeypatch, env, q, k, cfg, causal):
    import paper_2603_29494_b200.vecattn as va
    for key in ("VECATTN_TOPK_RADIX", "VECATTN_TOPK_FORCE_FALLBACK"):
        monkeypatch.delenv(key, raising=False)
    if env:
        monkeypatch.setenv(env, "1")
    off, idx = va.select(q, k, cfg, causal=causal)
    torch.cuda.synchronize()
    return off.cpu().numpy(), idx.cpu().numpy()


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}-N{c[3]}-{'c' if c[6] else 'nc'}-k{c[7]}-f{c[8]}-t{c[9]}" for c in CASES])
def test_windowed_topk_equals_radix(case, monkeypatch):
    import paper_2603_29494_b200.vecattn as va
    va.load()
    kind, Hq, Hkv, N, D, pq, causal, topk, keep_frac, tie = case
    q, k, v = synth.make_inputs(kind, 1, Hq, Hkv, N, D, cfg_id=13, device="cpu")
    if tie:
        k = k[:, :, torch.arange(N) % tie].contiguous()
    q, k = q.cuda(), k.cuda()
    cfg = va.SelectConfig(mode="topk", pq=pq, topk=topk, keep_frac=keep_frac)
    ow, iw = _run(monkeypatch, None, q, k, cfg, causal)
    orad, irad = _run(monkeypatch, "VECATTN_TOPK_RADIX", q, k, cfg, causal)
    off_, iff = _run(monkeypatch, "VECATTN_TOPK_FORCE_FALLBACK", q, k, cfg, causal)
    assert np.array_equal(ow, orad) and np.array_equal(iw, irad)
    assert np.array_equal(off_, orad) and np.array_equal(iff, irad)
