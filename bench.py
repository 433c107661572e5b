#!/usr/bin/env python
"""VecAttention hot-path benchmark (select + vector-sparse attention) on B200.

Contract (see README/DESIGN.md): `python bench.py --gpus N --steps K --warmup W`
prints ONE JSON line on rank 0.  A step = one pass of the whole hot path over the
workload: query pooling + TilingSelect/minS selection + CSR emission (vecattn_select)
then vector-sparse attention (vecattn_sparse_fwd), plus the head-parallel output
all-gather (NCCL) when N > 1.  Workload (BASELINE.json metric, quoted at 128K
tokens): `dit128k` = HunyuanVideo-like DiT layer, B=1, H=24, N=131072 (32x64x64
latent grid), D=128, bf16, non-causal, P_q=64, B_K=16, G_K=8192, MINS_ALG1 with one
global alpha calibrated to the paper's average sparsity rho=0.785 (Table 1),
synthetic VIDEO inputs.

value = effective (dense-equivalent) TFLOP/s of the whole job: 4*N^2*D*H flops of
the full attention the step replaces, divided by the step time (max over ranks).
The in-library dense kernel (vecattn_dense_fwd) is timed beside it; speed-up =
dense_ms / step_ms.  `--impl reference` times the fp64 CPU oracle instead
(bounded samples, extrapolated), as the reference arm.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import platform
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# alpha for rho=0.785 from the ours-arm calibration on the box (used only by the
# reference arm, which must not call our kernels); the ours arm re-calibrates.
ALPHA_TABLE = {("dit128k", "video", "alg1", 0.785): 1.0039}

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    d = dict(PEAKS_FALLBACK)
    d["source"] = "fallback (B200_PROFILING.md)"
    return d


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="dit128k")
    ap.add_argument("--kind", default="video", choices=["video", "gauss"])
    ap.add_argument("--mode", default="alg1", choices=["alg1", "exact", "topk"])
    ap.add_argument("--rho", type=float, default=0.785)
    ap.add_argument("--alpha", type=float, default=None, help="skip calibration")
    ap.add_argument("--pq", type=int, default=64, help="query-block (vector) size P_q (64 or 128)")
    ap.add_argument("--bk", type=int, default=16, help="Alg. 1 semantic K-tile size B_K")
    ap.add_argument("--gk", type=int, default=0, help="Alg. 1 tiles per group G_K (0 = the workload's)")
    ap.add_argument("--dense-reps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-blocks", type=int, default=192)
    ap.add_argument("--cpu-sample-rows", type=int, default=64)
    ap.add_argument("--quick", action="store_true", help="small debug run (no e2e/dense/cpu)")
    ap.add_argument("--no-context", action="store_true", help="skip the torch SDPA / flash-attn dense timings")
    ap.add_argument("--no-causal-extra", action="store_true", help="skip the causal vlm128k extra line")
    ap.add_argument("--flat-partition", action="store_true",
                    help="N > 1: split the flattened (head, 256-row item) work evenly over ranks (work windows of "
                         "vecattn_forward_replicated) instead of whole heads; per-rank selection statistics then "
                         "count a head shared by two ranks on both")
    ap.add_argument("--nccl-gather", action="store_true",
                    help="N > 1: all-gather O with NCCL after each KV-head group instead of the fused "
                         "symmetric-memory stores of the attention epilogue")
    return ap.parse_args()


# ----------------------------------------------------------------------------- dist
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def head_range(H, ws, rank):
    """Contiguous Q-head range of a rank (head-parallel)."""
    base, rem = divmod(H, ws)
    h0 = rank * base + min(rank, rem)
    return h0, h0 + base + (1 if rank < rem else 0), base + (1 if rem else 0)



def flat_window(H, N, ws, rank):
    """Flattened (head, 256-row item) partition of SURVEY 8(e) (B = 1): rank r owns items
    [r T / ws, (r+1) T / ws) of the T = H * ceil(N/256) items.  Returns the query heads
    [h0, h1) those items touch and the window relative to head h0's first item (the
    item_begin / item_end of vecattn_replica_t)."""
    n_items = (N + 255) // 256
    lo, hi = rank * H * n_items // ws, (rank + 1) * H * n_items // ws
    h0, h1 = lo // n_items, -(-hi // n_items)
    return h0, h1, (lo - h0 * n_items, hi - h0 * n_items)


def local_kv(H, Hkv, h0, h1):
    """(local KV heads, query heads per local KV head) of a rank owning query heads [h0, h1),
    as build_inputs lays them out: whole GQA groups share their KV head; a range that cuts a
    group gets one KV copy per local query head."""
    rep = H // Hkv
    kv0, kv1 = h0 // rep, (h1 - 1) // rep + 1
    if rep > 1 and (h0 % rep != 0 or (h1 - h0) % rep != 0):
        return h1 - h0, 1
    return kv1 - kv0, rep


def kv_groups(H, Hkv, ws, rank, ngroups=4):
    """A rank's local heads as up to `ngroups` KV-head groups: [(q0, q1, k0, k1)] local ranges
    (deterministic, so every rank knows every rank's plan)."""
    h0, h1, _ = head_range(H, ws, rank)
    if h1 <= h0:
        return []
    nkv, rep = local_kv(H, Hkv, h0, h1)
    g = max(1, min(ngroups, nkv))
    base, rem = divmod(nkv, g)
    out, k0 = [], 0
    for i in range(g):
        k1 = k0 + base + (1 if i < rem else 0)
        out.append((k0 * rep, k1 * rep, k0, k1))
        k0 = k1
    return out


class HeadGather:
    """C1: head-parallel output all-gather, overlapped with compute.  Each
    rank's local heads run as KV-head groups; group g's O is computed straight into a send
    buffer and its all-gather is issued asynchronously (NCCL: on the communicator's stream,
    which waits for the compute stream at issue time) while group g+1 computes.  Send
    buffers of group g are padded to the largest group g over ranks (no padding when H
    divides evenly).  `assemble` returns the full O [B, H, N, D] (bit-identical to one rank:
    kernels are deterministic and inputs are seeded per head)."""

    def __init__(self, H, Hkv, B, N, D, ws, rank, dtype, device, ngroups=4, group=None):
        import torch
        self.H, self.Hkv, self.B, self.N, self.D, self.ws, self.rank = H, Hkv, B, N, D, ws, rank
        self.group = group
        self.plans = [kv_groups(H, Hkv, ws, r, ngroups) for r in range(ws)]
        self.G = max(len(p) for p in self.plans)
        unit = B * N * D
        self.sizes = [unit * max((p[g][1] - p[g][0]) if g < len(p) else 0 for p in self.plans)
                      for g in range(self.G)]
        self.send = [torch.zeros(sz, dtype=dtype, device=device) for sz in self.sizes]
        self.recv = [torch.empty(ws, sz, dtype=dtype, device=device) for sz in self.sizes]

    def out_view(self, g):
        """This rank's O slice of group g ([B, q1-q0, N, D]) inside the send buffer."""
        q0, q1, _, _ = self.plans[self.rank][g]
        return self.send[g][:self.B * (q1 - q0) * self.N * self.D].view(self.B, q1 - q0, self.N, self.D)

    def run(self, compute):
        """compute(g, (q0, q1, k0, k1), out) writes the group's O into `out`; returns after
        every all-gather is complete (on the caller's stream, for NCCL)."""
        import torch.distributed as dist
        works = []
        mine = self.plans[self.rank]
        for g in range(self.G):
            if g < len(mine):
                compute(g, mine[g], self.out_view(g))
            works.append(dist.all_gather_into_tensor(self.recv[g].view(-1), self.send[g], group=self.group,
                                                    async_op=True))
        for w in works:
            w.wait()

    def bytes_received(self):
        return sum(self.recv[g].numel() * self.recv[g].element_size() * (self.ws - 1) // self.ws
                   for g in range(self.G))

    def assemble(self):
        import torch
        out = torch.empty(self.B, self.H, self.N, self.D, dtype=self.send[0].dtype, device=self.send[0].device)
        for r in range(self.ws):
            h0, _, _ = head_range(self.H, self.ws, r)
            for g, (q0, q1, _, _) in enumerate(self.plans[r]):
                n = self.B * (q1 - q0) * self.N * self.D
                out[:, h0 + q0:h0 + q1] = self.recv[g][r, :n].view(self.B, q1 - q0, self.N, self.D)
        return out

class SymmGather:
    """C1 fused into the attention: the full O
    [B, H, N, D] lives in torch symmetric memory on every rank, and each rank's attention
    epilogue stores its heads' rows straight into every rank's buffer
    (vecattn_forward_replicated: P2P stores over NVLink into the peers' mappings, or one NVLS
    multicast store per row with VECATTN_NVLS=1 when the box exposes a multicast address).
    No all-gather runs after the kernels, and uneven head splits need no padding.  A
    symmetric-memory barrier before a step (every rank is done with the previous O) and after
    it (every rank's stores have landed) orders the buffers.  `ok` is False (and `why` says
    why) when symmetric memory is unavailable; the bench then uses HeadGather (NCCL)."""

    def __init__(self, H, Hkv, B, N, D, ws, rank, dtype, device, ngroups=4, group=None, h_range=None, window=None):
        self.H, self.B, self.N, self.D, self.ws, self.rank = H, B, N, D, ws, rank
        # one call over all local heads: there is no all-gather to overlap with later groups,
        # and one call gives the attention's item scheduler the whole rank's items to balance.
        # h_range/window: the rank's heads and item window of the flattened partition.
        self.window = window
        if h_range is not None and window is not None:
            h0, h1 = h_range
            self.h0 = h0
            self.plans = [None] * ws
            self.plans[rank] = [(0, h1 - h0, 0, local_kv(H, Hkv, h0, h1)[0])]
        else:
            self.plans = [kv_groups(H, Hkv, ws, r, 1) for r in range(ws)]
            self.h0 = head_range(H, ws, rank)[0]
        self.ok, self.why, self.mc, self.mode = False, "", 0, "p2p"
        try:
            import torch.distributed as dist
            import torch.distributed._symmetric_memory as symm_mem
            self.buf = symm_mem.empty(B * H * N * D, dtype=dtype, device=device)
            self.handle = symm_mem.rendezvous(self.buf, (group or dist.group.WORLD).group_name)
            self.peers = [int(x) for x in self.handle.buffer_ptrs]
            if os.environ.get("VECATTN_NVLS") == "1" and int(self.handle.multicast_ptr or 0):
                self.mc, self.mode = int(self.handle.multicast_ptr), "nvls"
            self.ok = len(self.peers) == ws and ws <= 8
            if not self.ok:
                self.why = f"{len(self.peers)} peer buffers for world size {ws}"
        except Exception as e:  # no symmetric memory on this build / box
            self.why = repr(e)

    def run(self, compute):
        """compute(g, (q0, q1, k0, k1), rep) runs the group's forward with replica `rep`."""
        import paper_2603_29494_b200.vecattn as va
        self.handle.barrier(channel=0)
        for g, rng in enumerate(self.plans[self.rank]):
            w = self.window or (0, 0)
            rep = va.replica([] if self.mc else self.peers, self.mc, self.h0 + rng[0], self.H, w[0], w[1])
            compute(g, rng, rep)
        self.handle.barrier(channel=0)

    def bytes_received(self):
        return self.buf.numel() * self.buf.element_size() * (self.ws - 1) // self.ws

    def assemble(self):
        return self.buf.view(self.B, self.H, self.N, self.D)

# ------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.idx = gpu_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{gpu_index}.csv")

    def start(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.fh,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, mx, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
                power.append(float(parts[3]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        load = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(power) if power else None}


# ------------------------------------------------------------------------ helpers
def dense_flops(H, N, D, causal):
    return (2.0 if causal else 4.0) * N * N * D * H


def sparse_algo_flops(offsets_np, N, pq, D, causal, indices_np=None, Np=None):
    """4*D*sum_r |J_r| (useful flops of Eq. 5): C_i*h_i per block (non-causal)."""
    import numpy as np
    counts = np.diff(offsets_np).astype(np.float64)
    Np = Np or counts.size
    i = np.arange(counts.size) % Np
    h = np.minimum(N, (i + 1) * pq) - i * pq
    if not causal:
        return 4.0 * D * float((counts * h).sum())
    # causal: count visible (row, key) pairs per block
    assert indices_np is not None
    tot = 0.0
    for r in range(counts.size):
        ib = r % Np
        keys = indices_np[offsets_np[r]:offsets_np[r + 1]]
        rows0 = ib * pq
        rows = min(N, rows0 + pq) - rows0
        # row rows0+t sees keys <= rows0+t
        tot += float(np.clip(rows0 + rows - keys, 0, rows).sum())
    return 4.0 * D * tot


def sparsity(offsets_np, N, pq, Np, causal, indices_np=None, D=128):
    f = sparse_algo_flops(offsets_np, N, pq, D, causal, indices_np, Np) / (4.0 * D)
    H = (offsets_np.size - 1) // Np
    tot = H * (N * N if not causal else N * (N + 1) / 2)
    return 1.0 - f / tot



def build_inputs(wl, kind, dev, h0, h1):
    """Seeded synthetic Q/K/V for query heads [h0, h1) and the KV heads they read,
    generated per head on `dev` (a head's tensors do not depend on the GPU count)."""
    import torch
    from paper_2603_29494_b200 import synth
    B, H, Hkv, N, D = wl.B, wl.Hq, wl.Hkv, wl.N, wl.D
    rep = H // Hkv
    kv0, kv1 = h0 // rep, (h1 - 1) // rep + 1
    q = torch.empty(B, h1 - h0, N, D, dtype=torch.bfloat16, device=dev)
    k = torch.empty(B, kv1 - kv0, N, D, dtype=torch.bfloat16, device=dev)
    v = torch.empty(B, kv1 - kv0, N, D, dtype=torch.bfloat16, device=dev)
    for b in range(B):
        for hk in range(kv0, kv1):
            if kind == "video":
                dirs, kk, vv = synth.video_kv_head(N, D, wl.grid, synth.seed_of(wl.cfg_id, b, hk, 1), dev)
            else:
                dirs = None
                kk = synth.gauss_head(N, D, synth.seed_of(wl.cfg_id, b, hk, 1), dev)
                vv = synth.gauss_head(N, D, synth.seed_of(wl.cfg_id, b, hk, 2), dev)
            k[b, hk - kv0], v[b, hk - kv0] = kk, vv
            for hq in range(max(h0, hk * rep), min(h1, (hk + 1) * rep)):
                g = torch.Generator(device=dev)
                g.manual_seed(synth.seed_of(wl.cfg_id, b, hq, 0))
                if kind == "video":
                    q[b, hq - h0] = (6.0 * dirs + torch.randn(N, D, generator=g, device=dev)).to(torch.bfloat16)
                else:
                    q[b, hq - h0] = torch.randn(N, D, generator=g, device=dev).to(torch.bfloat16)
            del dirs
    if rep > 1 and (h0 % rep != 0 or (h1 - h0) % rep != 0):
        # head range not aligned with KV groups (e.g. 28 heads over 8 ranks): give every
        # local query head its own copy of its KV head so the ABI's GQA mapping (local head
        # h reads KV head h / (Hq/Hkv)) stays exact
        sel = torch.tensor([hq // rep - kv0 for hq in range(h0, h1)], device=dev)
        k, v = k.index_select(1, sel).contiguous(), v.index_select(1, sel).contiguous()
    return q, k, v

# ---------------------------------------------------------------------------- ours
def e2e_groups(n):
    """KV-head group sizes for the pipelined end-to-end step: 1, 2, 4, 7, ... (x1.6, at most 8)
    then a 2, 1 tail.  The first group's H2D and the last group's D2H are the only copies not
    overlapped with compute; the growth keeps each group's H2D close to the previous group's
    compute time (about 1.8 ms of PCIe per 3.3 ms of compute per head at dit128k)."""
    if n <= 3:
        return [1] * n
    tail = [2, 1] if n >= 8 else [1]
    body = n - sum(tail)
    sizes, step = [], 1
    while body > 0:
        t = min(step, body)
        sizes.append(t)
        body -= t
        step = min(int(step * 1.6) + 1, 8)
    return sizes + tail


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2603_29494_b200 import synth
    import paper_2603_29494_b200.vecattn as va

    ws, rank, local = dist_env()
    if args.gpus > 1 or ws > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    va.load()

    wl = synth.WORKLOADS[args.workload]
    B, H, Hkv, N, D, causal = wl.B, wl.Hq, wl.Hkv, wl.N, wl.D, wl.causal
    pq, bk, gk = args.pq, args.bk, (args.gk or wl.gk)
    h0, h1, hmax = head_range(H, ws, rank)
    window = None
    if args.flat_partition and ws > 1:
        # flattened (head, 256-row item) partition: rank r computes items
        # [r T / ws, (r+1) T / ws) of the B*H*ceil(N/256) items, with the heads they touch
        # (a head cut between two ranks is selected on both; each computes its own rows)
        assert B == 1, "--flat-partition: B = 1"
        h0, h1, window = flat_window(H, N, ws, rank)
    Hl = h1 - h0

    q, k, v = build_inputs(wl, args.kind, dev, h0, h1)
    torch.cuda.synchronize()
    Np = (N + pq - 1) // pq
    R = B * Hl * Np

    # ---- alpha calibration: bisection on counts-only selects (global alpha, all ranks agree)
    cfg = va.SelectConfig(mode=args.mode, pq=pq, bk=bk, gk=gk)
    pr = va.problem(q, k, causal)
    ws_sel = torch.empty(va.select_workspace_bytes(pr, cfg), dtype=torch.uint8, device=dev)
    offsets = torch.empty(R + 1, dtype=torch.int64, device=dev)
    d_nnz = torch.empty(1, dtype=torch.int64, device=dev)

    def rho_of(alpha):
        cfg.alpha = alpha
        va.select_into(q, k, cfg, offsets, None, 0, d_nnz, ws_sel, causal)
        oh = offsets.cpu().numpy()
        if causal:  # exact visible-pair count needs indices; approximate with C_i*h_i for calibration
            counts = np.diff(oh).astype(np.float64)
            i = np.arange(counts.size) % Np
            h = np.minimum(N, (i + 1) * pq) - i * pq
            sel = float((counts * h).sum())
            tot = Hl * N * (N + 1) / 2.0
        else:
            sel = float(sparse_algo_flops(oh, N, pq, D, False, Np=Np) / (4.0 * D))
            tot = Hl * N * N
        t = torch.tensor([sel, tot], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(t)
        return 1.0 - float(t[0] / t[1])

    if args.mode == "topk":
        cfg.keep_frac = 1.0 - args.rho
        alpha = None
    elif args.alpha is not None:
        alpha = args.alpha
        cfg.alpha = alpha
    else:
        lo, hi = 0.0, 1.0
        while rho_of(hi) > args.rho and hi < 1e4:
            lo, hi = hi, hi * 2.0
        for _ in range(40):
            mid = 0.5 * (lo + hi)
            r = rho_of(mid)
            if abs(r - args.rho) < 0.0025:
                lo = hi = mid
                break
            if r > args.rho:
                lo = mid
            else:
                hi = mid
        alpha = 0.5 * (lo + hi)
        cfg.alpha = alpha

    # ---- buffers sized once (outside the timed region)
    va.select_into(q, k, cfg, offsets, None, 0, d_nnz, ws_sel, causal)
    nnz = int(d_nnz.item())
    cap = int(nnz * 1.02) + 1024
    indices = torch.empty(cap, dtype=torch.int32, device=dev)
    ws_fwd = torch.empty(va.forward_workspace_bytes(pr, cfg, cap), dtype=torch.uint8, device=dev)
    o = torch.empty_like(q)
    lse = torch.empty(B, Hl, N, dtype=torch.float32, device=dev)
    hg = HeadGather(H, Hkv, B, N, D, ws, rank, torch.bfloat16, dev) if ws > 1 else None
    sg = (SymmGather(H, Hkv, B, N, D, ws, rank, torch.bfloat16, dev, h_range=(h0, h1), window=window)
          if ws > 1 and not args.nccl_gather else None)
    if sg is not None:
        okt = torch.tensor([1 if sg.ok else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)  # every rank takes the same all-gather path
        if not int(okt.item()):
            if window is not None:
                raise SystemExit(f"--flat-partition needs symmetric memory ({sg.why or 'on another rank'})")
            print(f"[bench] symmetric memory unavailable ({sg.why or 'on another rank'}); NCCL all-gather instead",
                  file=sys.stderr)
            sg = None
    assert ws == 1 or B == 1, "head-group slices of [B,H,N,D] are contiguous only for B = 1"
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def fwd_group(g, rng, out):
        q0, q1, k0, k1 = rng
        va.forward_into(q[:, q0:q1], k[:, k0:k1], v[:, k0:k1], cfg, offsets, indices, cap, d_nnz, cap, out,
                        lse[:, q0:q1], ws_fwd, causal)

    def fwd_group_rep(g, rng, rep):
        q0, q1, k0, k1 = rng
        va.forward_replicated_into(q[:, q0:q1], k[:, k0:k1], v[:, k0:k1], cfg, offsets, indices, cap, d_nnz, cap,
                                   None, lse[:, q0:q1], rep, ws_fwd, causal)

    def step(timers=None):
        """One hot-path pass: vecattn_forward (pool + select + CSR/plan + sparse attention);
        with N > 1 GPUs per KV-head group, each group's O all-gathered (NCCL, async) while the
        next group computes."""
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)] if timers is not None else None
        if ev:
            ev[0].record(stream)
        if ws == 1:
            va.forward_into(q, k, v, cfg, offsets, indices, cap, d_nnz, cap, o, lse, ws_fwd, causal)
            if ev:
                ev[1].record(stream)
        elif sg is not None:
            sg.run(fwd_group_rep)
            if ev:
                ev[1].record(stream)
        else:
            hg.run(fwd_group)
            if ev:
                ev[1].record(stream)
        if ev:
            ev[2].record(stream)
            timers.append(ev)

    for _ in range(max(3, args.warmup)):
        step()
    # selection statistics of all local heads (one untimed call over every local head)
    va.forward_into(q, k, v, cfg, offsets, indices, cap, d_nnz, cap, o, lse, ws_fwd, causal)
    torch.cuda.synchronize()
    oh = offsets.cpu().numpy()
    ih = indices[:int(oh[-1])].cpu().numpy() if causal else None
    rho_local = sparsity(oh, N, pq, Np, causal, ih, D)
    sp_flops = sparse_algo_flops(oh, N, pq, D, causal, ih, Np)

    clk = ClockSampler(local)
    timers = []
    stage = []  # library-recorded (select, emit+plan, attention) ms per timed step
    va.kernel_timing(True)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk.start()
    time.sleep(0.3)
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between timed steps (outside the events)
        step(timers)
        stage.append(va.kernel_timing_last())
    torch.cuda.synchronize()
    va.kernel_timing(False)
    if ws > 1:
        dist.barrier()
    clocks = clk.stop()
    fwd_ms = [t[0].elapsed_time(t[1]) for t in timers]
    ag_ms = [t[1].elapsed_time(t[2]) for t in timers]
    tot_ms = [t[0].elapsed_time(t[2]) for t in timers]
    tt = torch.tensor([sum(tot_ms), sum(fwd_ms), sum(ag_ms)], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    step_ms = float(tt[0]) / args.steps

    # ---- warm-L2 step time (no flush between steps; SURVEY 8(d) reports both)
    torch.cuda.synchronize()
    ew0, ew1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ew0.record(stream)
    for _ in range(args.steps):
        step()
    ew1.record(stream)
    torch.cuda.synchronize()
    warm_ms = ew0.elapsed_time(ew1) / args.steps

    # ---- stage breakdown via the two-call C ABI path (vecattn_select + vecattn_sparse_fwd)
    ws_sp = torch.empty(va.sparse_workspace_bytes(pr, pq, cap), dtype=torch.uint8, device=dev)
    brk = []
    for _ in range(2):
        flush.zero_()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(stream)
        va.select_into(q, k, cfg, offsets, indices, cap, d_nnz, ws_sel, causal)
        e[1].record(stream)
        va.sparse_fwd_into(q, k, v, offsets, indices, pq, o, lse, ws_sp, cap, causal)
        e[2].record(stream)
        torch.cuda.synchronize()
        brk.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])))
    sel_ms_avg = min(b[0] for b in brk)
    sparse_ms_avg = min(b[1] for b in brk)
    del ws_sp

    # ---- dense reference (in-library denominator), timed on the same heads
    dense_ms = None
    if not args.quick and args.dense_reps > 0:
        ws_d = torch.empty(256, dtype=torch.uint8, device=dev)
        od = torch.empty_like(q)
        va.dense_fwd_into(q, k, v, od, None, ws_d, causal)
        torch.cuda.synchronize()
        times = []
        for _ in range(args.dense_reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            va.dense_fwd_into(q, k, v, od, None, ws_d, causal)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        dt = torch.tensor([statistics.median(times)], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        dense_ms = float(dt[0])
        del od

    # ---- end-to-end through the C ABI with host buffers (pinned H2D in, O D2H out)
    e2e = None
    if not args.no_e2e and not args.quick and window is None:  # (e2e groups are whole heads)
        qh = torch.empty(q.shape, dtype=q.dtype, pin_memory=True)
        kh = torch.empty(k.shape, dtype=k.dtype, pin_memory=True)
        vh = torch.empty(v.shape, dtype=v.dtype, pin_memory=True)
        n_out = sum(r.numel() for r in hg.recv) if ws > 1 else o.numel()
        oh_host = torch.empty(n_out, dtype=o.dtype, pin_memory=True)
        qh.copy_(q)
        kh.copy_(k)
        vh.copy_(v)
        qd, kd, vd = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)

        # Host copies overlap the compute: the local heads run as KV-head groups; group g's
        # H2D (copy stream) runs while group g-1 computes, and (one rank) group g-1's output
        # D2H (second copy stream) while group g computes.  Group sizes ramp up from one KV
        # head and back down (e2e_groups), so only one head's H2D and one head's D2H are not
        # hidden behind compute.
        nkv, nq = k.shape[1], q.shape[1]
        rep_l = nq // nkv
        sizes = e2e_groups(nkv) if B == 1 else [nkv]
        if os.environ.get("BENCH_E2E_GROUPS") and B == 1:  # A/B of the group ramp (sizes summing to nkv)
            sizes = [int(x) for x in os.environ["BENCH_E2E_GROUPS"].split(",")]
            assert sum(sizes) == nkv, sizes
        cb = [0]
        for g in sizes:
            cb.append(cb[-1] + g)
        chunks = [(cb[i] * rep_l, cb[i + 1] * rep_l, cb[i], cb[i + 1]) for i in range(len(sizes))]
        s_h2d, s_d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        # Consecutive groups alternate between two compute streams with their own selection
        # and plan buffers, so one group's attention tail overlaps the next group's start.
        stream2 = torch.cuda.Stream(device=dev)
        sets = [(stream, offsets, indices, d_nnz, ws_fwd),
                (stream2, torch.empty_like(offsets), torch.empty_like(indices), torch.empty_like(d_nnz),
                 torch.empty_like(ws_fwd))]

        def e2e_step():
            s_h2d.wait_stream(stream)
            stream2.wait_stream(stream)
            for gi, (q0, q1, k0, k1) in enumerate(chunks):
                st_c, off_c, idx_c, nnz_c, ws_c = sets[gi % 2]
                with torch.cuda.stream(s_h2d):
                    qd[:, q0:q1].copy_(qh[:, q0:q1], non_blocking=True)
                    kd[:, k0:k1].copy_(kh[:, k0:k1], non_blocking=True)
                    vd[:, k0:k1].copy_(vh[:, k0:k1], non_blocking=True)
                    ev_in = torch.cuda.Event()
                    ev_in.record(s_h2d)
                st_c.wait_event(ev_in)
                with torch.cuda.stream(st_c):
                    va.forward_into(qd[:, q0:q1], kd[:, k0:k1], vd[:, k0:k1], cfg, off_c, idx_c, cap, nnz_c, cap,
                                    o[:, q0:q1], lse[:, q0:q1], ws_c, causal)
                ev_out = torch.cuda.Event()
                ev_out.record(st_c)
                if ws == 1:
                    with torch.cuda.stream(s_d2h):
                        s_d2h.wait_event(ev_out)
                        oh_host.view(o.shape)[:, q0:q1].copy_(o[:, q0:q1], non_blocking=True)
            stream.wait_stream(stream2)
            if ws > 1:
                hg.run(lambda g, rng, out: out.copy_(o[:, rng[0]:rng[1]]))
                off_h = 0
                for r in hg.recv:
                    oh_host[off_h:off_h + r.numel()].copy_(r.view(-1), non_blocking=True)
                    off_h += r.numel()
            else:
                stream.wait_stream(s_d2h)

        e2e_step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n_e2e = max(1, min(args.steps, 3))
        e0.record(stream)
        for _ in range(n_e2e):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        et = torch.tensor([e0.elapsed_time(e1) / n_e2e], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e_ms = float(et[0])
        h2d = (q.numel() + k.numel() + v.numel()) * 2 * ws
        d2h = n_out * 2
        e2e = {"value": dense_flops(B * H, N, D, causal) / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
               "ms_per_step": e2e_ms, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}
        del qh, kh, vh, oh_host, qd, kd, vd

    # ---- library kernel launches per step, counted (CUPTI via torch.profiler) over one step
    launches, launch_names = count_launches(step)

    # ---- external dense context (not the denominator): torch SDPA backends / flash-attn on
    # the same heads, same protocol (L2 flush, CUDA events)
    dense_context = None
    if not args.quick and not args.no_context and ws == 1:
        dense_context = time_dense_context(q, k, v, causal, flush, stream, total_dense=dense_flops(B * H, N, D, causal),
                                           ours_ms=dense_ms)

    # ---- aggregate results
    sp_tot = torch.tensor([sp_flops, float(int(oh[-1]))], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(sp_tot)
    total_dense = dense_flops(B * H, N, D, causal)
    value = total_dense / (step_ms * 1e-3) / 1e12
    peaks = load_peaks()
    attn_ms = statistics.mean(x[2] for x in stage)  # the attention kernel alone, CUDA events on its stream
    sel_stage_ms = statistics.mean(x[0] for x in stage)
    plan_stage_ms = statistics.mean(x[1] for x in stage)
    achieved = sp_flops / (attn_ms * 1e-3) / 1e12
    tt2 = torch.tensor([attn_ms, sel_stage_ms, plan_stage_ms], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(tt2, op=dist.ReduceOp.MAX)
    attn_ms, sel_stage_ms, plan_stage_ms = (float(x) for x in tt2)
    # selection stage (pool + pooled-score GEMM/filter + offsets scan): algorithmic HBM bytes,
    # Q read (pool), Q_p write + read, K read once per KV head, bitmask write,
    # counts + offsets
    Npq = (N + pq - 1) // pq
    sel_bytes = B * Hl * (2 * N * D + 4 * Npq * D + Npq * ((N + 255) // 256) * 32 + 16 * Npq) + \
        B * max(1, Hkv * Hl // H) * 2 * N * D
    sel_bytes_all = torch.tensor([float(sel_bytes)], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(sel_bytes_all)
    peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    # selection GEMM work: 2*D flops per (pooled row, visible key), all local heads
    vis_keys = Npq * N if not causal else sum(min(N, (i + 1) * pq) for i in range(Npq))  # R5: keys <= L_i
    sel_flops = 2.0 * D * B * Hl * vis_keys
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp) and args.workload == "dit128k" and ws == 1:
        traffic = json.load(open(tp)).get("dram_bytes_per_launch")
    line = {
        "metric": "select+sparse attention at 128K tokens (DiT H=24, rho=0.785): effective dense-equivalent "
                  "TFLOP/s (ms_per_step, speedup vs in-library dense in extra keys)",
        "value": round(value, 3),
        "unit": "TFLOP/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": max(3, args.warmup),
        "ms_per_step": round(step_ms, 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": f"synthetic {args.kind.upper()} (seeded per head; DESIGN.md input recipe)",
        "config": {"workload": args.workload, "B": B, "H": H, "Hkv": Hkv, "N": N, "D": D, "causal": causal,
                   "pq": pq, "bk": bk, "gk": gk, "mode": args.mode, "alpha": alpha, "rho_target": args.rho,
                   "rho_achieved": round(1.0 - float(sp_tot[0]) / (4.0 * D) /
                                         (H * B * (N * N if not causal else N * (N + 1) / 2)), 5),
                   "nnz": int(sp_tot[1]), "parallelism": ("flattened (head, item)" if window else "head") + f"-parallel x{ws}" + (
                       "" if ws == 1 else (f" + O all-gather fused into the attention epilogue ({sg.mode} stores into symmetric memory)"
                                           if sg is not None else " + NCCL all-gather(O) per KV-head group, overlapped")),
                   "l2": "256 MB L2 flush between timed steps; inputs (2.4 GB) >> L2"},
        "forward_ms": round(float(tt[1]) / args.steps, 4),
        "step_ms_warm_l2": round(warm_ms, 4),
        "allgather_bytes_received_per_rank": (sg or hg).bytes_received() if ws > 1 else 0,
        "breakdown_two_call": {"select_ms": round(sel_ms_avg, 4), "sparse_fwd_ms": round(sparse_ms_avg, 4),
                               "note": "vecattn_select + vecattn_sparse_fwd (CSR round trip), L2-flushed"},
        "dense_ms": round(dense_ms, 3) if dense_ms else None,
        "speedup_vs_dense": round(dense_ms / step_ms, 3) if dense_ms else None,
        "dense_tflops": round(total_dense / (dense_ms * 1e-3) / 1e12, 2) if dense_ms else None,
        "sparse_achieved_tflops": round(achieved, 2),
        "stage_ms": {"select": round(sel_stage_ms, 4), "emit_plan": round(plan_stage_ms, 4),
                     "attention": round(attn_ms, 4),
                     "note": "CUDA events recorded by the library on the launching stream (vecattn_kernel_timing)"},
        "select_roofline": {"bound": "tensor", "achieved": round(sel_flops / (sel_stage_ms * 1e-3) / 1e12, 2),
                            "peak": peak, "unit": "TFLOP/s",
                            "frac": round(sel_flops / (sel_stage_ms * 1e-3) / 1e12 / peak, 4),
                            "algorithmic_flops": int(sel_flops),
                            "hbm": {"achieved": round(float(sel_bytes_all[0]) / ws / (sel_stage_ms * 1e-3) / 1e9, 1),
                                    "peak": peaks["hbm_gbs"], "unit": "GB/s",
                                    "frac": round(float(sel_bytes_all[0]) / ws / (sel_stage_ms * 1e-3) / 1e9 / peaks["hbm_gbs"], 4),
                                    "algorithmic_bytes": int(sel_bytes_all[0] / ws)},
                            "note": "pool + pooled-score GEMM (2*D per pooled row x visible key, tcgen05) + Alg.1 "
                                    "filter epilogue + scan; tensor/issue-bound (SURVEY 8(d)), HBM fraction beside it"},
        "roofline": {"bound": "tensor", "kernel": ("attn_kernel<128,gather>" if causal else "attn_db_kernel<128,gather>") +
                     " (attention kernel alone, vecattn_forward)",
                     "achieved": round(achieved, 2), "peak": peak, "unit": "TFLOP/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "traffic_note": "dram read+write bytes per launch from profiles/traffic.json (ncu --set full)",
                     "peak_source": peaks["source"] + " bf16 sustained",
                     "algorithmic": "4*D*sum_r |J_r| flops per launch (DESIGN.md 'Rooflines')"},
        "clocks": clocks,
        "e2e": e2e,
        "gpu_launches": launches * args.steps,
        "gpu_launches_note": f"{launches} library kernels per step counted with torch.profiler (CUPTI) over one "
                             f"step: {launch_names}",
    }
    if dense_ms:
        line["dense_roofline"] = {"achieved": line["dense_tflops"], "peak": peak,
                                  "frac": round(line["dense_tflops"] / peak, 4)}
    if dense_context is not None:
        line["dense_context"] = dense_context

    # ---- CPU baseline: the oracle on a bounded sample of the same workload (rank 0, N=1)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and not args.quick:
        line["cpu_baseline"] = cpu_baseline(args, q, k, v, oh, indices, wl, alpha, cfg)
    # ---- the causal VLM headline beside it (rank 0, N=1; frees the DiT buffers first)
    if rank == 0 and ws == 1 and not args.quick and not args.no_causal_extra and args.workload == "dit128k":
        del q, k, v, o, lse, ws_fwd, indices, ws_sel, flush
        torch.cuda.empty_cache()
        line["causal_vlm128k"] = causal_extra(args, dev, peak)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def count_launches(step):
    """Kernels of this library launched by one call of `step` (names in namespace va::),
    from a CUPTI trace (torch.profiler): (count, sorted distinct names)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type.name == "CUDA" and "va::" in e.name]
    short = sorted({n.split("(")[0].replace("void ", "") for n in names})
    return len(names), short


def time_dense_context(q, k, v, causal, flush, stream, total_dense, ours_ms, reps=2):
    """Dense attention outside this library on the same [B, H, N, D] bf16 tensors, as context
    for the in-library denominator: torch SDPA with the cuDNN and the
    flash backends, and flash_attn (FlashAttention-2, the paper's dense baseline) if it
    runs on this GPU.  Same protocol as the in-library dense timing."""
    import torch
    import torch.nn.functional as F
    out = {}
    Hq, Hkv = q.shape[1], k.shape[1]

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    try:
        from torch.nn.attention import SDPBackend, sdpa_kernel
        for name, be in (("torch_sdpa_cudnn", SDPBackend.CUDNN_ATTENTION), ("torch_sdpa_flash", SDPBackend.FLASH_ATTENTION)):
            try:
                with sdpa_kernel([be]):
                    ms = timed(lambda: F.scaled_dot_product_attention(q, k, v, is_causal=causal, enable_gqa=Hq != Hkv))
                out[name] = {"ms": round(ms, 3), "tflops": round(total_dense / (ms * 1e-3) / 1e12, 1)}
            except Exception as e:  # backend not available for this shape / GPU
                out[name] = {"error": f"{type(e).__name__}: {str(e).splitlines()[0][:160]}"}
    except Exception as e:
        out["torch_sdpa"] = {"error": f"{type(e).__name__}: {str(e)[:160]}"}
    try:
        from flash_attn import flash_attn_func
        qt, kt, vt = (x.transpose(1, 2).contiguous() for x in (q, k, v))  # [B, N, H, D]
        ms = timed(lambda: flash_attn_func(qt, kt, vt, causal=causal))
        out["flash_attn2"] = {"ms": round(ms, 3), "tflops": round(total_dense / (ms * 1e-3) / 1e12, 1),
                              "note": "layout transpose outside the timed region"}
        del qt, kt, vt
    except Exception as e:
        out["flash_attn2"] = {"error": f"{type(e).__name__}: {str(e).splitlines()[0][:160] if str(e) else ''}"}
    best = min((x["ms"] for x in out.values() if "ms" in x), default=None)
    out["note"] = ("context only: the speed-up denominator is the in-library dense kernel (dense_ms); "
                   "best external / in-library = " + (f"{best / ours_ms:.3f}" if best and ours_ms else "n/a"))
    return out


def causal_extra(args, dev, peak):
    """The causal VLM headline beside the DiT one (SURVEY 8(d) 'report both'): vlm128k
    (H = 28, GQA 4 KV heads, N = 131072, causal), ALG1 at rho = 0.785, fused forward vs the
    in-library dense kernel, same timing protocol (L2 flush, CUDA events, median)."""
    import numpy as np
    import torch
    from paper_2603_29494_b200 import synth
    import paper_2603_29494_b200.vecattn as va

    wl = synth.WORKLOADS["vlm128k"]
    B, H, Hkv, N, D = wl.B, wl.Hq, wl.Hkv, wl.N, wl.D
    pq = 64
    q, k, v = build_inputs(wl, "video", dev, 0, H)
    cfg = va.SelectConfig(mode="alg1", pq=pq, bk=16, gk=wl.gk)
    pr = va.problem(q, k, True)
    Np = (N + pq - 1) // pq
    R = B * H * Np
    ws_sel = torch.empty(va.select_workspace_bytes(pr, cfg), dtype=torch.uint8, device=dev)
    offsets = torch.empty(R + 1, dtype=torch.int64, device=dev)
    d_nnz = torch.empty(1, dtype=torch.int64, device=dev)
    tot = H * N * (N + 1) / 2.0

    def rho_of(alpha):  # visible-pair sparsity needs indices; calibrate on C_i * h_i (as the main run)
        cfg.alpha = alpha
        va.select_into(q, k, cfg, offsets, None, 0, d_nnz, ws_sel, True)
        counts = np.diff(offsets.cpu().numpy()).astype(np.float64)
        i = np.arange(counts.size) % Np
        h = np.minimum(N, (i + 1) * pq) - i * pq
        return 1.0 - float((counts * h).sum()) / tot

    lo, hi = 0.0, 1.0
    while rho_of(hi) > args.rho and hi < 1e4:
        lo, hi = hi, hi * 2.0
    for _ in range(30):
        mid = 0.5 * (lo + hi)
        r = rho_of(mid)
        if abs(r - args.rho) < 0.0025:
            lo = hi = mid
            break
        lo, hi = (mid, hi) if r > args.rho else (lo, mid)
    cfg.alpha = 0.5 * (lo + hi)
    va.select_into(q, k, cfg, offsets, None, 0, d_nnz, ws_sel, True)
    cap = int(int(d_nnz.item()) * 1.02) + 1024
    indices = torch.empty(cap, dtype=torch.int32, device=dev)
    ws_fwd = torch.empty(va.forward_workspace_bytes(pr, cfg, cap), dtype=torch.uint8, device=dev)
    o = torch.empty_like(q)
    lse = torch.empty(B, H, N, dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def fwd():
        va.forward_into(q, k, v, cfg, offsets, indices, cap, d_nnz, cap, o, lse, ws_fwd, True)

    for _ in range(3):
        fwd()
    torch.cuda.synchronize()
    oh = offsets.cpu().numpy()
    ih = indices[:int(oh[-1])].cpu().numpy()
    rho = sparsity(oh, N, pq, Np, True, ih, D)
    sp_flops = sparse_algo_flops(oh, N, pq, D, True, ih, Np)
    ts, stages = [], []
    va.kernel_timing(True)
    for _ in range(max(3, args.steps)):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fwd()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        stages.append(va.kernel_timing_last())
    va.kernel_timing(False)
    ws_d = torch.empty(256, dtype=torch.uint8, device=dev)
    od = torch.empty_like(q)
    dts = []
    for _ in range(2):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        va.dense_fwd_into(q, k, v, od, None, ws_d, True)
        e1.record(stream)
        torch.cuda.synchronize()
        dts.append(e0.elapsed_time(e1))
    ms, dms = statistics.median(ts), statistics.median(dts)
    attn_ms = statistics.median(x[2] for x in stages)
    total = dense_flops(B * H, N, D, True)
    return {"workload": "vlm128k", "B": B, "H": H, "Hkv": Hkv, "N": N, "D": D, "causal": True, "pq": pq,
            "mode": "alg1", "gk": wl.gk, "alpha": round(cfg.alpha, 5), "rho_achieved": round(float(rho), 5),
            "ms_per_step": round(ms, 4), "value": round(total / (ms * 1e-3) / 1e12, 3), "unit": "TFLOP/s",
            "dense_ms": round(dms, 3), "speedup_vs_dense": round(dms / ms, 3),
            "stage_ms": {"select": round(statistics.median(x[0] for x in stages), 4),
                         "emit_plan": round(statistics.median(x[1] for x in stages), 4), "attention": round(attn_ms, 4)},
            "roofline": {"bound": "tensor", "kernel": "attn_kernel<128,gather>", "achieved": round(sp_flops / (attn_ms * 1e-3) / 1e12, 2),
                         "peak": peak, "unit": "TFLOP/s", "frac": round(sp_flops / (attn_ms * 1e-3) / 1e12 / peak, 4)},
            "note": "same process, after the headline; visible-pair sparsity (reading R15)"}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def cpu_baseline(args, q, k, v, oh, indices, wl, alpha, cfg, t_budget=None):
    """Time the fp64 oracle on head 0: selection of a few pooled rows + Eq. 5 on a few
    blocks; extrapolate linearly (rows/blocks are independent) to the full workload."""
    import numpy as np
    from oracle import oracle as orc

    N, D, pq, H = wl.N, wl.D, 64, wl.Hq
    Np = (N + pq - 1) // pq
    q0 = q[0, 0].double().cpu().numpy()
    k0 = k[0, 0].double().cpu().numpy()
    v0 = v[0, 0].double().cpu().numpy()
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(Np, args.cpu_sample_rows, replace=False))
    blocks = np.sort(rng.choice(Np, args.cpu_sample_blocks, replace=False))
    ho = oh[:Np + 1] - oh[0]
    hi = indices[:int(oh[Np])].cpu().numpy()
    t0 = time.perf_counter()
    qp = orc.pool(q0, pq)
    t1 = time.perf_counter()
    mode = {"alg1": orc.SEL_MINS_ALG1, "exact": orc.SEL_MINS_EXACT, "topk": orc.SEL_TOPK}[args.mode]
    orc.select(qp, k0, pq, causal=wl.causal, mode=mode, bk=16, gk=wl.gk, alpha=alpha or 0.0,
               keep_frac=cfg.keep_frac, rows=rows)
    t2 = time.perf_counter()
    orc.sparse_attn(q0, k0, v0, ho, hi, pq, causal=wl.causal, blocks=blocks)
    t3 = time.perf_counter()
    full_s = H * ((t1 - t0) + (t2 - t1) * Np / rows.size + (t3 - t2) * Np / blocks.size)
    value = dense_flops(H, N, D, wl.causal) / full_s / 1e12
    return {"value": value, "unit": "TFLOP/s", "cores": orc.num_threads(), "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"head 0 of {H}: pool all rows, select {rows.size}/{Np} pooled rows, Eq.5 on "
                      f"{blocks.size}/{Np} blocks (GPU index sets); measured {t3 - t0:.1f} s, "
                      f"extrapolated x{H} heads, linear in rows/blocks -> {full_s:.0f} s per step",
            "measured_s": round(t3 - t0, 2)}


# ---------------------------------------------------------------------- reference
def run_reference(args):
    """Reference arm: the fp64 CPU oracle on bounded samples of the same workload."""
    import numpy as np

    ws, rank, local = dist_env()
    if rank != 0:
        return
    from oracle import oracle as orc
    from paper_2603_29494_b200 import synth

    wl = synth.WORKLOADS[args.workload]
    N, D, pq, H = wl.N, wl.D, 64, wl.Hq
    Np = (N + pq - 1) // pq
    if args.kind == "video":
        dirs, kk, vv = synth.video_kv_head(N, D, wl.grid, synth.seed_of(wl.cfg_id, 0, 0, 1), "cpu")
        g = synth._gen(synth.seed_of(wl.cfg_id, 0, 0, 0), "cpu")
        qq = (6.0 * dirs + torch_randn(N, D, g)).to(__import__("torch").bfloat16)
    else:
        qq = synth.gauss_head(N, D, synth.seed_of(wl.cfg_id, 0, 0, 0))
        kk = synth.gauss_head(N, D, synth.seed_of(wl.cfg_id, 0, 0, 1))
        vv = synth.gauss_head(N, D, synth.seed_of(wl.cfg_id, 0, 0, 2))
    q0, k0, v0 = (t.double().numpy() for t in (qq, kk, vv))
    alpha = args.alpha if args.alpha is not None else (ALPHA_TABLE.get((args.workload, args.kind, args.mode,
                                                                        args.rho)) or 1.0)
    mode = {"alg1": orc.SEL_MINS_ALG1, "exact": orc.SEL_MINS_EXACT, "topk": orc.SEL_TOPK}[args.mode]
    qp = orc.pool(q0, pq)
    rng = np.random.default_rng(0)
    nb = max(1, args.cpu_sample_blocks // 6)

    def one_step():
        blocks = np.sort(rng.choice(Np, nb, replace=False))
        t0 = time.perf_counter()
        off, idx = orc.select(qp, k0, pq, causal=wl.causal, mode=mode, bk=16, gk=wl.gk, alpha=alpha,
                              keep_frac=1.0 - args.rho, rows=blocks)
        t1 = time.perf_counter()
        full_off = np.zeros(Np + 1, np.int64)
        cnt = np.zeros(Np, np.int64)
        cnt[blocks] = np.diff(off)
        full_off[1:] = np.cumsum(cnt)
        full_idx = np.zeros(full_off[-1], np.int32)
        for t, b in enumerate(blocks):
            full_idx[full_off[b]:full_off[b + 1]] = idx[off[t]:off[t + 1]]
        orc.sparse_attn(q0, k0, v0, full_off, full_idx, pq, causal=wl.causal, blocks=blocks)
        t2 = time.perf_counter()
        return H * Np / nb * (t2 - t0)  # extrapolated seconds per full step

    for _ in range(args.warmup):
        one_step()
    est = [one_step() for _ in range(args.steps)]
    step_s = statistics.mean(est)
    value = dense_flops(H, N, D, wl.causal) / step_s / 1e12
    line = {
        "impl": "reference",
        "metric": "select+sparse attention at 128K tokens (DiT H=24, rho=0.785): effective dense-equivalent "
                  "TFLOP/s (ms_per_step, speedup vs in-library dense in extra keys)",
        "value": value, "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": f"synthetic {args.kind.upper()}",
        "config": {"workload": args.workload, "N": N, "D": D, "H": H, "alpha": alpha, "mode": args.mode},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": orc.num_threads(), "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": f"per step: select + Eq.5 for {nb}/{Np} random blocks of head 0, "
                                   f"extrapolated x{Np // nb} blocks x{H} heads"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def torch_randn(N, D, g):
    import torch
    return torch.randn(N, D, generator=g)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
