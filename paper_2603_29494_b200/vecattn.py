"""Thin ctypes binding of include/vecattn.h (argument marshalling only).

Every step of the hot path runs in libvecattn.so's sm_100a kernels; torch is
used for device memory and streams.  There is no CPU or eager fallback: if the
library is missing or the device is not sm_100, these functions raise.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libvecattn.so")

SEL_MINS_ALG1 = 0
SEL_MINS_EXACT = 1
SEL_TOPK = 2
MODES = {"alg1": SEL_MINS_ALG1, "exact": SEL_MINS_EXACT, "topk": SEL_TOPK}

STATUS = {0: "ok", 1: "invalid argument", 2: "shape", 3: "unsupported", 4: "workspace", 5: "cuda"}


class VecAttnError(RuntimeError):
    def __init__(self, fn, code):
        super().__init__(f"{fn} failed: {STATUS.get(code, code)} ({code})")
        self.code = code


class Problem(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int64), ("Hq", ctypes.c_int64), ("Hkv", ctypes.c_int64), ("N", ctypes.c_int64),
                ("D", ctypes.c_int64), ("causal", ctypes.c_int32), ("scale", ctypes.c_float)]


class SelectParams(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("pq", ctypes.c_int32), ("bk", ctypes.c_int32), ("gk", ctypes.c_int32),
                ("alpha", ctypes.c_float), ("alpha_per_head", ctypes.POINTER(ctypes.c_float)),
                ("topk", ctypes.c_int64), ("keep_frac", ctypes.c_float)]


class Replica(ctypes.Structure):
    """vecattn_replica_t (include/vecattn.h): where the fused attention -> all-gather stores O."""
    _fields_ = [("n_peers", ctypes.c_int32), ("peer_o", ctypes.c_void_p * 8), ("o_multicast", ctypes.c_void_p),
                ("head0", ctypes.c_int64), ("heads_total", ctypes.c_int64), ("item_begin", ctypes.c_int64),
                ("item_end", ctypes.c_int64)]


_lib = None


def load(path: str = LIB_PATH):
    """Load libvecattn.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    P, vp = ctypes.POINTER, ctypes.c_void_p
    i32, i64, sz = ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    prob, sel = P(Problem), P(SelectParams)
    sig = {
        "vecattn_pool": (i32, [prob, i32, vp, vp, vp]),
        "vecattn_select_workspace_bytes": (sz, [prob, sel]),
        "vecattn_select": (i32, [prob, sel, vp, vp, vp, vp, i64, vp, vp, sz, vp]),
        "vecattn_sparse_workspace_bytes": (sz, [prob, i32, i64]),
        "vecattn_sparse_fwd": (i32, [prob, i32, vp, vp, vp, vp, vp, i64, vp, vp, vp, sz, vp]),
        "vecattn_dense_workspace_bytes": (sz, [prob]),
        "vecattn_dense_fwd": (i32, [prob, vp, vp, vp, vp, vp, vp, sz, vp]),
        "vecattn_forward_workspace_bytes": (sz, [prob, sel, i64]),
        "vecattn_forward": (i32, [prob, sel, vp, vp, vp, vp, vp, i64, vp, i64, vp, vp, vp, sz, vp]),
        "vecattn_forward_replicated": (i32, [prob, sel, vp, vp, vp, vp, vp, i64, vp, i64, vp, vp, P(Replica), vp, sz,
                                             vp]),
        "vecattn_validate_selection": (i32, [prob, i32, vp, vp, vp, vp]),
        "vecattn_debug_scores": (i32, [prob, i32, vp, vp, vp, vp, sz, vp]),
        "vecattn_status_string": (ctypes.c_char_p, [i32]),
        "vecattn_last_cuda_error": (ctypes.c_char_p, []),
        "vecattn_abi_version": (i32, []),
        "vecattn_kernel_timing": (i32, [i32]),
        "vecattn_alpha_dp": (i32, [i32, i32, P(ctypes.c_float), P(ctypes.c_float), ctypes.c_float, i32, P(i32),
                                   P(ctypes.c_double)]),
        "vecattn_select_naive_workspace_bytes": (sz, [prob, i32, i32]),
        "vecattn_select_naive": (i32, [prob, i32, i32, ctypes.c_float, ctypes.c_float, vp, vp, vp, vp, i64, vp, vp,
                                       sz, vp]),
        "vecattn_kernel_timing_last": (i32, [P(ctypes.c_float), P(ctypes.c_float), P(ctypes.c_float)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


EXPORTED = ["vecattn_pool", "vecattn_select_workspace_bytes", "vecattn_select", "vecattn_sparse_workspace_bytes",
            "vecattn_sparse_fwd", "vecattn_dense_workspace_bytes", "vecattn_dense_fwd",
            "vecattn_forward_workspace_bytes", "vecattn_forward", "vecattn_forward_replicated",
            "vecattn_validate_selection", "vecattn_debug_scores", "vecattn_status_string", "vecattn_last_cuda_error",
            "vecattn_abi_version", "vecattn_kernel_timing", "vecattn_kernel_timing_last",
            "vecattn_select_naive_workspace_bytes", "vecattn_select_naive", "vecattn_alpha_dp"]


def alpha_dp(sp, perf, rho_target: float, grid: int = 1000):
    """Eq. 4 per-head filter-ratio search (host-only C ABI call, vecattn_alpha_dp).
    sp, perf: array-likes [H, n_cand].  Returns (choice int32 [H], best total perf); raises
    VecAttnError if no assignment reaches rho_target."""
    import numpy as np
    sp = np.ascontiguousarray(sp, np.float32)
    perf = np.ascontiguousarray(perf, np.float32)
    H, C = sp.shape
    choice = np.zeros(H, np.int32)
    best = ctypes.c_double()
    rc = load().vecattn_alpha_dp(H, C, sp.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                 perf.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), float(rho_target), int(grid),
                                 choice.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), ctypes.byref(best))
    _check("vecattn_alpha_dp", rc)
    return choice, best.value

NAIVE_MINS = 0
NAIVE_TOPP = 1
NAIVE_MODES = {"mins": NAIVE_MINS, "topp": NAIVE_TOPP}


def select_naive_workspace_bytes(pr: Problem, pq: int, mode: str) -> int:
    return int(load().vecattn_select_naive_workspace_bytes(ctypes.byref(pr), pq, NAIVE_MODES[mode]))


def select_naive_into(q, k, mode: str, offsets, indices, cap: int, d_nnz, ws: torch.Tensor, *, pq: int = 64,
                      alpha: float = 0.0, top_p: float = 0.9, causal: bool = False, scale=None, stream=None):
    """Raw vecattn_select_naive call (materialise-then-filter baseline) into caller buffers."""
    lib = load()
    _dev_check(q, k, offsets, indices, d_nnz)
    _check_io(q, k, offsets=offsets, indices=indices, d_nnz=d_nnz, pq=pq)
    pr = problem(q, k, causal, scale)
    rc = lib.vecattn_select_naive(ctypes.byref(pr), int(pq), NAIVE_MODES[mode], float(alpha), float(top_p), _ptr(q),
                                  _ptr(k), _ptr(offsets), _ptr(indices), int(cap), _ptr(d_nnz), _ptr(ws), ws.numel(),
                                  _stream(stream))
    _check("vecattn_select_naive", rc)


def select_naive(q, k, mode: str, *, pq: int = 64, alpha: float = 0.0, top_p: float = 0.9, causal: bool = False,
                 scale=None, ws: "Workspace | None" = None, stream=None):
    """Naive selection baseline with the capacity protocol: returns (offsets int64, indices int32)."""
    B, H, N, D = q.shape
    Np = (N + pq - 1) // pq
    pr = problem(q, k, causal, scale)
    ws = ws or Workspace(q.device)
    wbuf = ws.get(select_naive_workspace_bytes(pr, pq, mode))
    offsets = torch.empty(B * H * Np + 1, dtype=torch.int64, device=q.device)
    d_nnz = torch.empty(1, dtype=torch.int64, device=q.device)
    select_naive_into(q, k, mode, offsets, None, 0, d_nnz, wbuf, pq=pq, alpha=alpha, top_p=top_p, causal=causal,
                      scale=scale, stream=stream)
    cap = int(d_nnz.item())
    indices = torch.empty(max(cap, 1), dtype=torch.int32, device=q.device)
    select_naive_into(q, k, mode, offsets, indices, cap, d_nnz, wbuf, pq=pq, alpha=alpha, top_p=top_p,
                      causal=causal, scale=scale, stream=stream)
    return offsets, indices[:cap]


def kernel_timing(enable: bool) -> None:
    """Enable/disable the library's per-stage CUDA-event timing (vecattn_kernel_timing)."""
    _check("vecattn_kernel_timing", load().vecattn_kernel_timing(1 if enable else 0))


def kernel_timing_last() -> tuple[float, float, float]:
    """(select_ms, plan_ms, attn_ms) of the most recent timed call; -1 for stages it did not run."""
    a, b_, c = ctypes.c_float(), ctypes.c_float(), ctypes.c_float()
    _check("vecattn_kernel_timing_last", load().vecattn_kernel_timing_last(ctypes.byref(a), ctypes.byref(b_),
                                                                             ctypes.byref(c)))
    return a.value, b_.value, c.value


def _ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _check(fn, rc):
    if rc != 0:
        err = VecAttnError(fn, rc)
        if rc == 5:
            err.args = (f"{err.args[0]}: {load().vecattn_last_cuda_error().decode()}",)
        raise err


def _dev_check(*ts):
    for t in ts:
        if t is None:
            continue
        if not t.is_cuda:
            raise ValueError("vecattn: tensors must be CUDA device tensors (no CPU fallback)")
        if not t.is_contiguous():
            raise ValueError("vecattn: tensors must be contiguous")


def _check_io(q, k=None, v=None, o=None, lse=None, offsets=None, indices=None, d_nnz=None, pq=None,
              cfg=None):
    """Argument checks the C ABI cannot do on raw pointers: dtypes, shapes,
    devices and sizes.  A mismatch would otherwise read or write out of bounds on the device."""
    if q.dim() != 4 or q.dtype != torch.bfloat16:
        raise ValueError(f"vecattn: q must be bf16 [B,Hq,N,D], got {q.dtype} {tuple(q.shape)}")
    B, Hq, N, D = q.shape
    for name, t in (("k", k), ("v", v)):
        if t is None:
            continue
        if t.dtype != torch.bfloat16 or t.dim() != 4 or t.shape[0] != B or t.shape[2] != N or t.shape[3] != D:
            raise ValueError(f"vecattn: {name} must be bf16 [B,Hkv,N,D] matching q {tuple(q.shape)}, "
                             f"got {t.dtype} {tuple(t.shape)}")
        if Hq % t.shape[1] != 0:
            raise ValueError(f"vecattn: Hq={Hq} is not a multiple of Hkv={t.shape[1]}")
    if k is not None and v is not None and k.shape != v.shape:
        raise ValueError(f"vecattn: k {tuple(k.shape)} and v {tuple(v.shape)} differ")
    if o is not None and (o.dtype != torch.bfloat16 or o.shape != q.shape):
        raise ValueError(f"vecattn: o must be bf16 {tuple(q.shape)}, got {o.dtype} {tuple(o.shape)}")
    if lse is not None and (lse.dtype != torch.float32 or tuple(lse.shape) != (B, Hq, N)):
        raise ValueError(f"vecattn: lse must be float32 {(B, Hq, N)}, got {lse.dtype} {tuple(lse.shape)}")
    if offsets is not None:
        if offsets.dtype != torch.int64:
            raise ValueError("vecattn: offsets must be int64")
        if pq is not None and offsets.numel() < B * Hq * ((N + pq - 1) // pq) + 1:
            raise ValueError(f"vecattn: offsets needs B*Hq*N_p+1 = {B * Hq * ((N + pq - 1) // pq) + 1} entries")
    if indices is not None and indices.dtype != torch.int32:
        raise ValueError("vecattn: indices must be int32")
    if d_nnz is not None and (d_nnz.dtype != torch.int64 or d_nnz.numel() < 1):
        raise ValueError("vecattn: d_nnz must be an int64 device scalar")
    if cfg is not None and cfg.alpha_per_head is not None and len(cfg.alpha_per_head) != Hq:
        raise ValueError(f"vecattn: alpha_per_head needs Hq={Hq} entries, got {len(cfg.alpha_per_head)}")
    for t in (k, v, o, lse, offsets, indices, d_nnz):
        if t is not None and t.device != q.device:
            raise ValueError(f"vecattn: every tensor must be on {q.device}, got one on {t.device}")


def problem(q: torch.Tensor, k: torch.Tensor, causal: bool, scale: float | None = None) -> Problem:
    B, Hq, N, D = q.shape
    Hkv = k.shape[1]
    return Problem(B, Hq, Hkv, N, D, int(bool(causal)), 0.0 if scale is None else float(scale))


@dataclass
class SelectConfig:
    mode: str = "alg1"
    pq: int = 64
    bk: int = 16
    gk: int = 16
    alpha: float = 0.0
    alpha_per_head: list | None = None
    topk: int = 0
    keep_frac: float = 0.0

    def params(self) -> SelectParams:
        sp = SelectParams()
        sp.mode, sp.pq, sp.bk, sp.gk = MODES[self.mode], self.pq, self.bk, self.gk
        sp.alpha = float(self.alpha)
        if self.alpha_per_head is not None:
            arr = (ctypes.c_float * len(self.alpha_per_head))(*[float(a) for a in self.alpha_per_head])
            sp.alpha_per_head = ctypes.cast(arr, ctypes.POINTER(ctypes.c_float))
            sp._keep = arr  # keep alive
        sp.topk = int(self.topk)
        sp.keep_frac = float(self.keep_frac)
        return sp


class Workspace:
    """Caller-owned device workspace, grown on demand (allocation happens outside the hot loop)."""

    def __init__(self, device="cuda"):
        self.device = device
        self.buf = None

    def get(self, nbytes: int) -> torch.Tensor:
        nbytes = max(int(nbytes), 256)
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        return self.buf


def pool(q: torch.Tensor, pq: int = 64, stream=None) -> torch.Tensor:
    lib = load()
    _dev_check(q)
    _check_io(q)
    B, H, N, D = q.shape
    Np = (N + pq - 1) // pq
    qp = torch.empty(B, H, Np, D, dtype=torch.bfloat16, device=q.device)
    pr = problem(q, q, False)
    _check("vecattn_pool", lib.vecattn_pool(ctypes.byref(pr), pq, _ptr(q), _ptr(qp), _stream(stream)))
    return qp


def select_workspace_bytes(pr: Problem, cfg: SelectConfig) -> int:
    return int(load().vecattn_select_workspace_bytes(ctypes.byref(pr), ctypes.byref(cfg.params())))


def select_into(q, k, cfg: SelectConfig, offsets, indices, cap: int, d_nnz, ws: torch.Tensor, causal: bool,
                scale=None, stream=None):
    """Raw vecattn_select call into caller buffers (no host sync)."""
    lib = load()
    _dev_check(q, k, offsets, indices, d_nnz)
    _check_io(q, k, offsets=offsets, indices=indices, d_nnz=d_nnz, pq=cfg.pq, cfg=cfg)
    pr = problem(q, k, causal, scale)
    sp = cfg.params()
    rc = lib.vecattn_select(ctypes.byref(pr), ctypes.byref(sp), _ptr(q), _ptr(k), _ptr(offsets), _ptr(indices),
                            int(cap), _ptr(d_nnz), _ptr(ws), ws.numel(), _stream(stream))
    _check("vecattn_select", rc)


def select(q, k, cfg: SelectConfig, causal: bool = False, scale=None, ws: Workspace | None = None,
           cap: int | None = None, stream=None):
    """Selection with the capacity protocol: returns (offsets int64, indices int32)."""
    B, H, N, D = q.shape
    Np = (N + cfg.pq - 1) // cfg.pq
    pr = problem(q, k, causal, scale)
    ws = ws or Workspace(q.device)
    wbuf = ws.get(select_workspace_bytes(pr, cfg))
    offsets = torch.empty(B * H * Np + 1, dtype=torch.int64, device=q.device)
    d_nnz = torch.empty(1, dtype=torch.int64, device=q.device)
    if cap is None:
        select_into(q, k, cfg, offsets, None, 0, d_nnz, wbuf, causal, scale, stream)
        cap = int(d_nnz.item())
    indices = torch.empty(max(cap, 1), dtype=torch.int32, device=q.device)
    select_into(q, k, cfg, offsets, indices, max(cap, 1), d_nnz, wbuf, causal, scale, stream)
    nnz = int(d_nnz.item())
    if nnz > cap:
        return select(q, k, cfg, causal, scale, ws, nnz, stream)
    return offsets, indices[:nnz]


def debug_scores(q, k, pq: int = 64, ws: Workspace | None = None, stream=None) -> torch.Tensor:
    lib = load()
    _dev_check(q, k)
    _check_io(q, k)
    B, H, N, D = q.shape
    Np = (N + pq - 1) // pq
    pr = problem(q, k, False)
    cfg = SelectConfig(pq=pq)
    ws = ws or Workspace(q.device)
    wbuf = ws.get(select_workspace_bytes(pr, cfg))
    out = torch.full((B * H * Np, N), float("nan"), dtype=torch.float32, device=q.device)
    _check("vecattn_debug_scores", lib.vecattn_debug_scores(ctypes.byref(pr), pq, _ptr(q), _ptr(k), _ptr(out),
                                                              _ptr(wbuf), wbuf.numel(), _stream(stream)))
    return out


def sparse_workspace_bytes(pr: Problem, pq: int, nnz_cap: int) -> int:
    return int(load().vecattn_sparse_workspace_bytes(ctypes.byref(pr), pq, int(nnz_cap)))


def sparse_fwd_into(q, k, v, offsets, indices, pq, o, lse, ws: torch.Tensor, nnz_cap: int, causal: bool,
                    scale=None, stream=None):
    lib = load()
    _dev_check(q, k, v, offsets, indices, o, lse)
    _check_io(q, k, v, o, lse, offsets=offsets, indices=indices, pq=pq)
    if indices is not None and indices.numel() < nnz_cap:
        raise ValueError(f"vecattn: indices has {indices.numel()} entries < nnz_cap={nnz_cap}")
    pr = problem(q, k, causal, scale)
    rc = lib.vecattn_sparse_fwd(ctypes.byref(pr), pq, _ptr(q), _ptr(k), _ptr(v), _ptr(offsets), _ptr(indices),
                                int(nnz_cap), _ptr(o), _ptr(lse), _ptr(ws), ws.numel(), _stream(stream))
    _check("vecattn_sparse_fwd", rc)


def sparse_fwd(q, k, v, offsets, indices, pq: int = 64, causal: bool = False, scale=None,
               ws: Workspace | None = None, with_lse: bool = True, stream=None):
    B, H, N, D = q.shape
    pr = problem(q, k, causal, scale)
    nnz_cap = max(int(indices.numel()), 1)
    ws = ws or Workspace(q.device)
    wbuf = ws.get(sparse_workspace_bytes(pr, pq, nnz_cap))
    o = torch.empty_like(q)
    lse = torch.empty(B, H, N, dtype=torch.float32, device=q.device) if with_lse else None
    sparse_fwd_into(q, k, v, offsets, indices, pq, o, lse, wbuf, nnz_cap, causal, scale, stream)
    return o, lse


def dense_fwd_into(q, k, v, o, lse, ws: torch.Tensor, causal: bool, scale=None, stream=None):
    lib = load()
    _dev_check(q, k, v, o, lse)
    _check_io(q, k, v, o, lse)
    pr = problem(q, k, causal, scale)
    rc = lib.vecattn_dense_fwd(ctypes.byref(pr), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), _ptr(ws),
                               ws.numel(), _stream(stream))
    _check("vecattn_dense_fwd", rc)


def dense_fwd(q, k, v, causal: bool = False, scale=None, with_lse: bool = True, stream=None):
    B, H, N, D = q.shape
    o = torch.empty_like(q)
    lse = torch.empty(B, H, N, dtype=torch.float32, device=q.device) if with_lse else None
    ws = torch.empty(256, dtype=torch.uint8, device=q.device)
    dense_fwd_into(q, k, v, o, lse, ws, causal, scale, stream)
    return o, lse


def forward_workspace_bytes(pr: Problem, cfg: SelectConfig, nnz_cap: int) -> int:
    return int(load().vecattn_forward_workspace_bytes(ctypes.byref(pr), ctypes.byref(cfg.params()), int(nnz_cap)))


def forward_into(q, k, v, cfg: SelectConfig, offsets, indices, cap: int, d_nnz, nnz_cap: int, o, lse,
                 ws: torch.Tensor, causal: bool, scale=None, stream=None):
    """Raw vecattn_forward (fused selection + sparse attention) into caller buffers."""
    lib = load()
    _dev_check(q, k, v, offsets, indices, d_nnz, o, lse)
    _check_io(q, k, v, o, lse, offsets=offsets, indices=indices, d_nnz=d_nnz, pq=cfg.pq, cfg=cfg)
    if indices is not None and indices.numel() < cap:
        raise ValueError(f"vecattn: indices has {indices.numel()} entries < cap={cap}")
    pr = problem(q, k, causal, scale)
    sp = cfg.params()
    rc = lib.vecattn_forward(ctypes.byref(pr), ctypes.byref(sp), _ptr(q), _ptr(k), _ptr(v), _ptr(offsets),
                             _ptr(indices), int(cap), _ptr(d_nnz), int(nnz_cap), _ptr(o), _ptr(lse), _ptr(ws),
                             ws.numel(), _stream(stream))
    _check("vecattn_forward", rc)


def replica(peer_ptrs=(), multicast_ptr: int = 0, head0: int = 0, heads_total: int = 0, item_begin: int = 0,
            item_end: int = 0) -> Replica:
    """vecattn_replica_t from raw device addresses (e.g. a torch symmetric-memory handle's
    buffer_ptrs / multicast_ptr) of every rank's full O [B, heads_total, N, D] bf16, and an
    optional work window [item_begin, item_end) over the call's flattened 256-row items."""
    peer_ptrs = [int(x) for x in peer_ptrs]
    if len(peer_ptrs) > 8:
        raise ValueError("vecattn: at most 8 replicas")
    r = Replica()
    r.n_peers = len(peer_ptrs)
    for i, x in enumerate(peer_ptrs):
        r.peer_o[i] = x
    r.o_multicast = int(multicast_ptr) or None
    r.head0 = int(head0)
    r.heads_total = int(heads_total)
    r.item_begin = int(item_begin)
    r.item_end = int(item_end)
    return r


def forward_replicated_into(q, k, v, cfg: SelectConfig, offsets, indices, cap: int, d_nnz, nnz_cap: int, o, lse,
                            rep: Replica, ws: torch.Tensor, causal: bool, scale=None, stream=None):
    """Raw vecattn_forward_replicated: vecattn_forward whose attention epilogue also stores
    every O row into each replica buffer (the fused output all-gather).  o may be None."""
    lib = load()
    _dev_check(q, k, v, offsets, indices, d_nnz, o, lse)
    _check_io(q, k, v, o, lse, offsets=offsets, indices=indices, d_nnz=d_nnz, pq=cfg.pq, cfg=cfg)
    if indices is not None and indices.numel() < cap:
        raise ValueError(f"vecattn: indices has {indices.numel()} entries < cap={cap}")
    pr = problem(q, k, causal, scale)
    sp = cfg.params()
    rc = lib.vecattn_forward_replicated(ctypes.byref(pr), ctypes.byref(sp), _ptr(q), _ptr(k), _ptr(v), _ptr(offsets),
                                        _ptr(indices), int(cap), _ptr(d_nnz), int(nnz_cap), _ptr(o), _ptr(lse),
                                        ctypes.byref(rep), _ptr(ws), ws.numel(), _stream(stream))
    _check("vecattn_forward_replicated", rc)


def forward(q, k, v, cfg: SelectConfig, causal: bool = False, scale=None, nnz_cap: int | None = None,
            want_indices: bool = True, stream=None):
    """Fused VecAttention forward: returns (o, lse, offsets, indices-or-None)."""
    B, H, N, D = q.shape
    Np = (N + cfg.pq - 1) // cfg.pq
    pr = problem(q, k, causal, scale)
    offsets = torch.empty(B * H * Np + 1, dtype=torch.int64, device=q.device)
    d_nnz = torch.empty(1, dtype=torch.int64, device=q.device)
    o = torch.empty_like(q)
    lse = torch.empty(B, H, N, dtype=torch.float32, device=q.device)
    if nnz_cap is None:  # counts-only selection to size the plan (one host sync)
        wsel = torch.empty(select_workspace_bytes(pr, cfg), dtype=torch.uint8, device=q.device)
        select_into(q, k, cfg, offsets, None, 0, d_nnz, wsel, causal, scale, stream)
        nnz_cap = max(1, int(d_nnz.item()))
    ws = torch.empty(forward_workspace_bytes(pr, cfg, nnz_cap), dtype=torch.uint8, device=q.device)
    indices = torch.empty(nnz_cap, dtype=torch.int32, device=q.device) if want_indices else None
    forward_into(q, k, v, cfg, offsets, indices, nnz_cap if want_indices else 0, d_nnz, nnz_cap, o, lse, ws,
                 causal, scale, stream)
    nnz = int(d_nnz.item())
    if nnz > nnz_cap:
        return forward(q, k, v, cfg, causal, scale, nnz, want_indices, stream)
    return o, lse, offsets, (indices[:nnz] if want_indices else None)


def validate_selection(offsets, indices, q_shape, pq: int, causal: bool, stream=None) -> int:
    lib = load()
    B, H, N, D = q_shape
    pr = Problem(B, H, H, N, D, int(causal), 0.0)
    bad = torch.zeros(1, dtype=torch.int32, device=offsets.device)
    _check("vecattn_validate_selection", lib.vecattn_validate_selection(
        ctypes.byref(pr), pq, _ptr(offsets), _ptr(indices), _ptr(bad), _stream(stream)))
    return int(bad.item())


def default_scale(D: int) -> float:
    return 1.0 / math.sqrt(D)
