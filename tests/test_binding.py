"""Host-side argument checks of the ctypes binding (no GPU): wrong dtypes, shapes, sizes or
devices are rejected before any pointer reaches the C ABI."""
import pytest
import torch

from paper_2603_29494_b200 import vecattn as va


def t(*shape, dtype=torch.bfloat16):
    return torch.zeros(*shape, dtype=dtype)


def test_accepts_consistent_arguments():
    q, k = t(1, 4, 130, 64), t(1, 2, 130, 64)
    va._check_io(q, k, k.clone(), t(1, 4, 130, 64), t(1, 4, 130, dtype=torch.float32),
                 offsets=t(4 * 3 + 1, dtype=torch.int64), indices=t(10, dtype=torch.int32),
                 d_nnz=t(1, dtype=torch.int64), pq=64, cfg=va.SelectConfig(alpha_per_head=[0.1] * 4))


@pytest.mark.parametrize("bad", [
    dict(q=t(1, 4, 130, 64, dtype=torch.float32)),            # fp32 q
    dict(k=t(1, 2, 129, 64)),                                  # k length != q length
    dict(k=t(1, 3, 130, 64)),                                  # Hq % Hkv != 0
    dict(v=t(1, 1, 130, 64)),                                  # v shape != k shape
    dict(o=t(1, 4, 130, 32)),                                  # o shape
    dict(lse=t(1, 4, 130)),                                    # lse not float32
    dict(offsets=t(13, dtype=torch.int32)),                    # offsets int32
    dict(offsets=t(5, dtype=torch.int64)),                     # offsets too short for B*Hq*Np+1
    dict(indices=t(10, dtype=torch.int64)),                    # indices int64
    dict(d_nnz=t(1, dtype=torch.int32)),                       # d_nnz int32
    dict(cfg=va.SelectConfig(alpha_per_head=[0.1] * 3)),       # alpha_per_head length != Hq
])
def test_rejects_inconsistent_arguments(bad):
    args = dict(q=t(1, 4, 130, 64), k=t(1, 2, 130, 64), v=t(1, 2, 130, 64), o=t(1, 4, 130, 64),
                lse=t(1, 4, 130, dtype=torch.float32), offsets=t(13, dtype=torch.int64),
                indices=t(10, dtype=torch.int32), d_nnz=t(1, dtype=torch.int64), pq=64, cfg=va.SelectConfig())
    args.update(bad)
    with pytest.raises(ValueError):
        va._check_io(args.pop("q"), args.pop("k"), args.pop("v"), args.pop("o"), args.pop("lse"), **args)
