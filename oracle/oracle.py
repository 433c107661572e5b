"""fp64 CPU ORACLE for VecAttention (arXiv 2603.29494) -- ctypes front-end.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product package ``paper_2603_29494_b200`` never imports it, and
it never imports the product package: the two share no code.

All arithmetic lives in ``vecattn_oracle.cpp`` (plain fp64 loops, one function
per paper definition, each citing PAPER.md).  This file only marshals numpy
arrays and loops over (batch, head).  Inputs arrive as exact bf16 bit patterns
(uint16) or float64; bf16 -> float64 is exact (bits << 16 reinterpreted as
float32, then widened).

Functions and the passages they follow:
  pool          Eq. 2, P:187-194 (ragged last block: its true height)
  select        Alg. 1 P:755-850 (MINS_ALG1), Eq. 3 P:224-228 (MINS_EXACT),
                topK P:213-214 (TOPK)
  sparse_attn   Eq. 5 P:320-341 / Alg. 2 P:857-955 (plain softmax form)
  dense_attn    Eq. 1
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "vecattn_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

SEL_MINS_ALG1 = 0
SEL_MINS_EXACT = 1
SEL_TOPK = 2

_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ (-O2 -fopenmp, strict IEEE: no -ffast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["g++", "-std=c++17", "-O2", "-fopenmp", "-fPIC", "-shared",
               "-fno-fast-math", "-ffp-contract=off", _SRC, "-o", _LIB]
        subprocess.check_call(cmd)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.POINTER
        d, i32, i64 = ctypes.c_double, ctypes.c_int32, ctypes.c_int64
        pd, pi32, pi64 = P(d), P(i32), P(i64)
        lib.oracle_pool.argtypes = [pd, i64, i64, i32, i32, pd]
        lib.oracle_round_bf16.argtypes = [pd, i64, pd]
        lib.oracle_scores_row.argtypes = [pd, pd, i64, i64, d, i64, pd]
        lib.oracle_select_rows.argtypes = [pd, pd, i64, i64, i32, i32, d, i32, i32, i32, d, i64, d,
                                           pi64, i64, pi64, pi32, i64, pd, pi64]
        lib.oracle_topp_rows.argtypes = [pd, pd, i64, i64, i32, i32, d, d, pi64, i64, pi64, ctypes.POINTER(ctypes.c_int32),
                                         i64, pd]
        lib.oracle_attn_blocks.argtypes = [pd, pd, pd, i64, i64, i32, i32, d, pi64, i64, pi64,
                                           pi32, pd, pd]
        lib.oracle_dense_rows.argtypes = [pd, pd, pd, i64, i64, i32, d, pi64, i64, pd, pd]
        lib.oracle_set_num_threads.argtypes = [ctypes.c_int]
        _lib = lib
    return _lib


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def set_num_threads(n: int) -> None:
    _load().oracle_set_num_threads(int(n))


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def bf16_bits_to_f64(bits) -> np.ndarray:
    """Exact up-conversion of bf16 bit patterns (uint16/int16 array) to float64."""
    b = np.ascontiguousarray(bits).view(np.uint16).astype(np.uint32) << 16
    return b.view(np.float32).astype(np.float64)


def round_bf16(x) -> np.ndarray:
    """RNE-round float64 values to bf16 values (returned as float64)."""
    x = _f64(x)
    out = np.empty_like(x)
    _load().oracle_round_bf16(_p(x, ctypes.c_double), x.size, _p(out, ctypes.c_double))
    return out


def f64_to_bf16_bits(x) -> np.ndarray:
    """bf16 bit patterns of already-bf16-representable float64 values."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    f = x.astype(np.float32)
    assert np.array_equal(f.astype(np.float64), x), "values are not bf16-representable"
    u = f.view(np.uint32)
    assert not np.any(u & 0xFFFF), "values are not bf16-representable"
    return (u >> 16).astype(np.uint16)


def default_scale(D: int) -> float:
    return 1.0 / np.sqrt(np.float64(D))


# ----------------------------------------------------------------------------- pool
def pool(q, pq: int, round_to_bf16: bool = True) -> np.ndarray:
    """Eq. 2 for one head: q [N,D] float64 -> Q_p [ceil(N/pq), D] float64."""
    q = _f64(q)
    N, D = q.shape
    Np = (N + pq - 1) // pq
    out = np.empty((Np, D), np.float64)
    rc = _load().oracle_pool(_p(q, ctypes.c_double), N, D, pq, int(round_to_bf16),
                             _p(out, ctypes.c_double))
    if rc:
        raise ValueError(f"oracle_pool: bad arguments (rc={rc})")
    return out


def scores_row(qp, k, i: int, scale: float | None = None) -> np.ndarray:
    qp, k = _f64(qp), _f64(k)
    N, D = k.shape
    scale = default_scale(D) if scale is None else float(scale)
    out = np.empty(N, np.float64)
    _load().oracle_scores_row(_p(qp, ctypes.c_double), _p(k, ctypes.c_double), N, D, scale, i,
                              _p(out, ctypes.c_double))
    return out


# --------------------------------------------------------------------------- select
def select(qp, k, pq: int, *, causal: bool = False, mode: int = SEL_MINS_ALG1, bk: int = 16,
           gk: int = 16, alpha: float = 0.0, topk: int = 0, keep_frac: float = 0.0,
           scale: float | None = None, rows=None, detail: bool = False):
    """Important-vector selection for one head.

    qp: [Np, D] pooled queries (float64), k: [N, D].  Returns (offsets int64
    [R+1], indices int32 [nnz]) as CSR over the requested pooled rows (default:
    all).  With detail=True also returns (thr [R, n_tiles], jstar [R, n_tiles]).
    """
    qp, k = _f64(qp), _f64(k)
    N, D = k.shape
    Np = qp.shape[0]
    scale = default_scale(D) if scale is None else float(scale)
    rows = np.arange(Np, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, np.int64)
    R = rows.size
    counts = np.zeros(R, np.int64)
    idx = np.empty((R, N), np.int32)
    n_tiles = (N + bk - 1) // bk
    thr = np.empty((R, n_tiles), np.float64) if detail else None
    js = np.empty((R, n_tiles), np.int64) if detail else None
    rc = _load().oracle_select_rows(
        _p(qp, ctypes.c_double), _p(k, ctypes.c_double), N, D, pq, int(causal), scale, int(mode),
        bk, gk, float(alpha), int(topk), float(keep_frac), _p(rows, ctypes.c_int64), R,
        _p(counts, ctypes.c_int64), _p(idx, ctypes.c_int32), N,
        _p(thr, ctypes.c_double) if detail else None, _p(js, ctypes.c_int64) if detail else None)
    if rc:
        raise ValueError(f"oracle_select_rows: bad arguments (rc={rc})")
    offsets = np.zeros(R + 1, np.int64)
    np.cumsum(counts, out=offsets[1:])
    indices = np.concatenate([idx[r, :counts[r]] for r in range(R)]) if R else np.zeros(0, np.int32)
    indices = indices.astype(np.int32)
    if detail:
        return offsets, indices, thr, js
    return offsets, indices


def select_topp(qp, k, pq: int, p: float, *, causal: bool = False, scale: float | None = None, rows=None,
                detail: bool = False):
    """topP selection of the naive approach for one head: per pooled
    row, the smallest set of keys in descending softmax(s) order whose mass is >= p.
    Returns CSR (offsets, indices) over the requested pooled rows; detail=True also returns
    the selected mass per row."""
    qp, k = _f64(qp), _f64(k)
    N, D = k.shape
    Np = qp.shape[0]
    scale = default_scale(D) if scale is None else float(scale)
    rows = np.arange(Np, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, np.int64)
    R = rows.size
    counts = np.zeros(R, np.int64)
    idx = np.empty((R, N), np.int32)
    mass = np.empty(R, np.float64)
    rc = _load().oracle_topp_rows(_p(qp, ctypes.c_double), _p(k, ctypes.c_double), N, D, pq, int(causal), scale,
                                  float(p), _p(rows, ctypes.c_int64), R, _p(counts, ctypes.c_int64),
                                  _p(idx, ctypes.c_int32), N, _p(mass, ctypes.c_double))
    if rc:
        raise ValueError(f"oracle_topp_rows: bad arguments (rc={rc})")
    offsets = np.zeros(R + 1, np.int64)
    np.cumsum(counts, out=offsets[1:])
    indices = (np.concatenate([idx[r, :counts[r]] for r in range(R)]) if R else np.zeros(0)).astype(np.int32)
    return (offsets, indices, mass) if detail else (offsets, indices)


# ---------------------------------------------------------------------- attention
def sparse_attn(q, k, v, offsets, indices, pq: int, *, causal: bool = False,
                scale: float | None = None, blocks=None):
    """Eq. 5 for one head.  offsets/indices: CSR over ALL query blocks of the head
    (row i = block i).  blocks: subset of block ids to compute (default all).
    Returns (O [len(blocks)*pq, D], LSE [len(blocks)*pq]); rows past N are 0/NaN."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    N, D = q.shape
    Np = (N + pq - 1) // pq
    scale = default_scale(D) if scale is None else float(scale)
    offsets = np.asarray(offsets, np.int64)
    indices = np.asarray(indices, np.int32)
    blocks = np.arange(Np, dtype=np.int64) if blocks is None else np.ascontiguousarray(blocks, np.int64)
    nb = blocks.size
    sub_off = np.zeros(nb + 1, np.int64)
    parts = []
    for t, b in enumerate(blocks):
        seg = indices[offsets[b]:offsets[b + 1]]
        parts.append(seg)
        sub_off[t + 1] = sub_off[t] + seg.size
    sub_idx = np.ascontiguousarray(np.concatenate(parts) if parts else np.zeros(0), np.int32)
    if sub_idx.size == 0:
        sub_idx = np.zeros(1, np.int32)
    o = np.empty((nb * pq, D), np.float64)
    lse = np.empty(nb * pq, np.float64)
    rc = _load().oracle_attn_blocks(
        _p(q, ctypes.c_double), _p(k, ctypes.c_double), _p(v, ctypes.c_double), N, D, pq,
        int(causal), scale, _p(blocks, ctypes.c_int64), nb, _p(sub_off, ctypes.c_int64),
        _p(sub_idx, ctypes.c_int32), _p(o, ctypes.c_double), _p(lse, ctypes.c_double))
    if rc:
        raise ValueError(f"oracle_attn_blocks: bad arguments (rc={rc})")
    return o, lse


def dense_attn(q, k, v, *, causal: bool = False, scale: float | None = None, rows=None):
    """Eq. 1 for one head; returns (O [len(rows), D], LSE [len(rows)])."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    N, D = q.shape
    scale = default_scale(D) if scale is None else float(scale)
    rows = np.arange(N, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, np.int64)
    o = np.empty((rows.size, D), np.float64)
    lse = np.empty(rows.size, np.float64)
    rc = _load().oracle_dense_rows(_p(q, ctypes.c_double), _p(k, ctypes.c_double),
                                   _p(v, ctypes.c_double), N, D, int(causal), scale,
                                   _p(rows, ctypes.c_int64), rows.size, _p(o, ctypes.c_double),
                                   _p(lse, ctypes.c_double))
    if rc:
        raise ValueError(f"oracle_dense_rows: bad arguments (rc={rc})")
    return o, lse


def sparsity(offsets, indices, N: int, pq: int, causal: bool) -> float:
    """rho = 1 - sum_r |J_r| / S_tot ("how many entries are dropped"), DESIGN.md
    reading R15, for ONE head's CSR: J_r is the row's visible selected keys, Idx(i) for
    non-causal and {j in Idx(i) : j <= r} for causal (Eq. 5's mask); S_tot = N^2 or
    N(N+1)/2 (the visible entries of the dense map).  Plain loops over blocks and rows."""
    offsets = np.asarray(offsets, np.int64)
    indices = np.asarray(indices, np.int64)
    Np = offsets.size - 1
    kept = 0
    for i in range(Np):
        idx = indices[offsets[i]:offsets[i + 1]]
        for r in range(i * pq, min(N, (i + 1) * pq)):
            kept += int(np.count_nonzero(idx <= r)) if causal else idx.size
    tot = N * N if not causal else N * (N + 1) // 2
    return 1.0 - kept / tot
