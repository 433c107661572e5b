"""Seeded synthetic inputs shaped like the paper's workloads.

This module is SHARED by the product tests and the oracle tests.  It holds none
of the method's arithmetic (no pooling, scoring, filtering or attention): it
only draws random Q/K/V tensors with torch generators and returns bf16 tensors.

Recipes:

* GAUSS: Q, K, V i.i.d. N(0,1), rounded once to bf16.  Low-overlap worst case.
* VIDEO: vertical-vector structure ("adjacent tokens ... similar attention
  preferences").  Tokens t = (f, y, x) on an F x Hh x Ww latent grid
  (x fastest).  Per KV head: region directions c_r ~ N(0, I_D) for 8x8-token
  patches, per-frame drift c_{r,f} = normalize(c_r + 0.3 xi), keys
  k_t = 6 c_{r(t),f(t)} + eps', queries q_t = 6 c_{r(t),f(t)} + eps (eps, eps' ~
  N(0, I)), 4 sink keys k_{0..3} = 12 normalize(mean_r c_r) + eps', V ~ N(0,1).
  Query heads of one GQA group share their KV head's directions but draw their
  own noise.

Seeds: seed(cfg_id, b, h) = 0x7EC0 + 1_000_003*cfg_id + 10_007*b + 101*h, drawn
per (batch, head) in a fixed order, so a head's tensors do not depend on how
many heads / GPUs the job has.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch


def seed_of(cfg_id: int, b: int, h: int, salt: int = 0) -> int:
    return 0x7EC0 + 1_000_003 * cfg_id + 10_007 * b + 101 * h + 7 * salt


@dataclass(frozen=True)
class Workload:
    """A named configuration (BASELINE.json configs)."""
    name: str
    B: int
    Hq: int
    Hkv: int
    N: int
    D: int
    causal: bool
    gk: int
    grid: tuple | None  # (F, Hh, Ww) latent grid for VIDEO inputs
    cfg_id: int


WORKLOADS = {
    "toy": Workload("toy", 1, 1, 1, 1024, 64, False, 16, (1, 32, 32), 0),
    "vlm64k": Workload("vlm64k", 1, 28, 4, 65536, 128, True, 16, (64, 32, 32), 1),
    "hy": Workload("hy", 1, 24, 24, 118800, 128, False, 8192, (33, 45, 80), 2),
    "wan": Workload("wan", 1, 40, 40, 75600, 128, False, 8192, (21, 45, 80), 3),
    "dit128k": Workload("dit128k", 1, 24, 24, 131072, 128, False, 8192, (32, 64, 64), 4),
    "vlm128k": Workload("vlm128k", 1, 28, 4, 131072, 128, True, 16, (32, 64, 64), 5),
}
# SURVEY.md 8(d) sweep: F x 64 x 64 VIDEO grids, N = 16K..256K, DiT-like and VLM-like
for _f in (4, 8, 16, 32, 64):
    _n = _f * 64 * 64
    WORKLOADS[f"dit{_n // 1024}k"] = WORKLOADS.get(f"dit{_n // 1024}k") or Workload(
        f"dit{_n // 1024}k", 1, 24, 24, _n, 128, False, 8192, (_f, 64, 64), 10 + _f)
    WORKLOADS[f"vlm{_n // 1024}k"] = WORKLOADS.get(f"vlm{_n // 1024}k") or Workload(
        f"vlm{_n // 1024}k", 1, 28, 4, _n, 128, True, 16, (_f, 64, 64), 100 + _f)


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def gauss_head(N: int, D: int, seed: int, device="cpu") -> torch.Tensor:
    g = _gen(seed, device)
    return torch.randn(N, D, generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)


def gauss(B: int, Hq: int, Hkv: int, N: int, D: int, cfg_id: int = 0, device="cpu"):
    """GAUSS inputs: returns (q [B,Hq,N,D], k [B,Hkv,N,D], v [B,Hkv,N,D]) bf16."""
    q = torch.empty(B, Hq, N, D, dtype=torch.bfloat16, device=device)
    k = torch.empty(B, Hkv, N, D, dtype=torch.bfloat16, device=device)
    v = torch.empty(B, Hkv, N, D, dtype=torch.bfloat16, device=device)
    for b in range(B):
        for h in range(Hq):
            q[b, h] = gauss_head(N, D, seed_of(cfg_id, b, h, 0), device)
        for h in range(Hkv):
            k[b, h] = gauss_head(N, D, seed_of(cfg_id, b, h, 1), device)
            v[b, h] = gauss_head(N, D, seed_of(cfg_id, b, h, 2), device)
    return q, k, v


def _grid_for(N: int, grid):
    if grid is not None and math.prod(grid) == N:
        return grid
    # fall back to a 1 x 1 x N "line" of tokens with 64-wide rows
    ww = 64
    return (1, (N + ww - 1) // ww, ww)


def _normalize(x: torch.Tensor) -> torch.Tensor:
    return x / x.norm(dim=-1, keepdim=True).clamp_min(1e-6)


def video_kv_head(N: int, D: int, grid, seed: int, device="cpu"):
    """Directions + K, V of one KV head. Returns (dirs [N,D] fp32, k bf16, v bf16)."""
    F, Hh, Ww = _grid_for(N, grid)
    g = _gen(seed, device)
    ry, rx = (Hh + 7) // 8, (Ww + 7) // 8
    c = torch.randn(ry * rx, D, generator=g, device=device)                 # c_r
    xi = torch.randn(F, ry * rx, D, generator=g, device=device)             # per-frame drift
    cf = _normalize(c.unsqueeze(0) + 0.3 * xi)                              # c_{r,f}
    t = torch.arange(F * Hh * Ww, device=device)[:N]
    f = t // (Hh * Ww)
    y = (t // Ww) % Hh
    x = t % Ww
    r = (y // 8) * rx + (x // 8)
    dirs = cf[f, r]                                                          # [N, D]
    k = 6.0 * dirs + torch.randn(N, D, generator=g, device=device)
    sink = 12.0 * _normalize(c.mean(0, keepdim=True))
    ns = min(4, N)
    k[:ns] = sink + torch.randn(ns, D, generator=g, device=device)
    v = torch.randn(N, D, generator=g, device=device)
    return dirs, k.to(torch.bfloat16), v.to(torch.bfloat16)


def video(B: int, Hq: int, Hkv: int, N: int, D: int, grid=None, cfg_id: int = 0, device="cpu"):
    """VIDEO inputs: returns (q [B,Hq,N,D], k [B,Hkv,N,D], v [B,Hkv,N,D]) bf16."""
    assert Hq % Hkv == 0
    rep = Hq // Hkv
    q = torch.empty(B, Hq, N, D, dtype=torch.bfloat16, device=device)
    k = torch.empty(B, Hkv, N, D, dtype=torch.bfloat16, device=device)
    v = torch.empty(B, Hkv, N, D, dtype=torch.bfloat16, device=device)
    for b in range(B):
        for hk in range(Hkv):
            dirs, kk, vv = video_kv_head(N, D, grid, seed_of(cfg_id, b, hk, 1), device)
            k[b, hk] = kk
            v[b, hk] = vv
            for hq in range(hk * rep, (hk + 1) * rep):
                g = _gen(seed_of(cfg_id, b, hq, 0), device)
                q[b, hq] = (6.0 * dirs + torch.randn(N, D, generator=g, device=device)).to(torch.bfloat16)
            del dirs
    return q, k, v


def make_inputs(kind: str, B: int, Hq: int, Hkv: int, N: int, D: int, grid=None, cfg_id: int = 0,
                device="cpu"):
    if kind == "gauss":
        return gauss(B, Hq, Hkv, N, D, cfg_id, device)
    if kind == "video":
        return video(B, Hq, Hkv, N, D, grid, cfg_id, device)
    raise ValueError(kind)


def bf16_bits(t: torch.Tensor):
    """uint16 numpy view of a bf16 tensor's bit patterns (host copy)."""
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view("uint16")
