"""Scheduler / synchronisation switches of the attention kernels change timing only: the
per-die item counters (VECATTN_DIE_SPLIT=1/2) and the strict ODONE observation
(VECATTN_STRICT_SYNC=1) must give bit-identical O and LSE (every item's result is independent
of which CTA runs it and when)."""
import pytest
import torch

from paper_2603_29494_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("causal", [False, True])
def test_scheduler_knobs_bit_identical(causal, monkeypatch):
    import paper_2603_29494_b200.vecattn as va
    va.load()
    N, D = 9000, 128
    q, k, v = synth.make_inputs("video", 1, 4, 2, N, D, cfg_id=17, device="cpu")
    q, k, v = q.cuda(), k.cuda(), v.cuda()
    cfg = va.SelectConfig(mode="alg1", pq=64, gk=16 if causal else 8192, alpha=1.0)
    for key in ("VECATTN_DIE_SPLIT", "VECATTN_STRICT_SYNC"):
        monkeypatch.delenv(key, raising=False)
    o0, l0, off0, idx0 = va.forward(q, k, v, cfg, causal=causal)
    od, ld = va.dense_fwd(q, k, v, causal=causal)
    for key, val in (("VECATTN_DIE_SPLIT", "1"), ("VECATTN_DIE_SPLIT", "2"), ("VECATTN_STRICT_SYNC", "1")):
        monkeypatch.setenv(key, val)
        o1, l1, off1, idx1 = va.forward(q, k, v, cfg, causal=causal)
        od1, ld1 = va.dense_fwd(q, k, v, causal=causal)
        torch.cuda.synchronize()
        assert torch.equal(off0, off1) and torch.equal(idx0, idx1), key
        assert torch.equal(o0, o1) and torch.equal(l0, l1), (key, val)
        assert torch.equal(od, od1) and torch.equal(ld, ld1), (key, val)
        monkeypatch.delenv(key)
