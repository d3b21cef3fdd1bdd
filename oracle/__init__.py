"""fp64 CPU oracle for the Ulysses sequence-parallel exact-attention hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with the CUDA path (``paper_2405_15780_b200``) and
never imports it; the product never imports this package.

Contents
  * ``attn_fwd``, ``attn_fwd_rows``, ``attn_bwd``, ``attn_bwd_dq_rows``,
    ``attn_bwd_kv_rows`` — ctypes wrappers over ``oracle.c`` (plain fp64 loops +
    OpenMP; definitions and citations there).  ``delta`` — Delta = rowsum(dO*O).
  * ``ulysses`` — the paper's sequence-parallel data movement (§2.5):
    sequence shards, the all-to-all, head shards, and the
    composition seq-shard -> a2a -> per-head attention -> a2a back.
  * ``lss`` — contiguous key-segment attention and the exact log-sum-exp merge
    of partial results ("LSS chunking" in BASELINE.json), and the
    LSS sequence-parallel strategy (per-rank forward, partial dK/dV, reduce).
  * ``layer`` — the attention layer around it: bias-free Q/K/V and output
    projections and their gradients.

Parity status: every function is pinned by ``tests/test_oracle.py`` (numpy
brute force on materialised N x N, central finite differences, closed forms
from S:46-52 / S:178-186, invariants).  No function is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc + OpenMP (generic x86-64, -O3).  The flags
    keep IEEE fp64 semantics: no -ffast-math, no FMA contraction."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O3", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
               "-std=c11", _SRC, "-o", _LIB + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            d = ctypes.POINTER(ctypes.c_double)
            i64 = ctypes.c_int64
            lib.oracle_attn_fwd.argtypes = [d, d, d, i64, i64, i64, i64, i64, d, d, d]
            lib.oracle_attn_fwd_rows.argtypes = [d, ctypes.POINTER(i64), i64, d, d,
                                                 i64, i64, i64, i64, d, d]
            lib.oracle_attn_bwd.argtypes = [d, d, d, d, i64, i64, i64, i64, d, d, d, d, d, d]
            lib.oracle_attn_bwd_dq_rows.argtypes = [d, d, ctypes.POINTER(i64), i64, d, d, i64, i64, i64, i64, d]
            lib.oracle_attn_bwd_kv_rows.argtypes = [d, d, d, d, i64, i64, ctypes.POINTER(i64), i64, d, d]
            lib.oracle_num_threads.restype = ctypes.c_int
            lib.oracle_set_num_threads.argtypes = [ctypes.c_int]
            _lib = lib
    return _lib


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def set_num_threads(n: int) -> None:
    """OpenMP thread count of the oracle's loops (no effect on its arithmetic)."""
    _load().oracle_set_num_threads(int(n))


def attn_fwd(q, k, v, with_abs: bool = False):
    """Dense exact attention.  q [B][Nq][H][D], k/v [B][Nk][H][D] (fp64, any
    values; callers pass bf16-rounded inputs widened exactly).  Returns
    (out [B][Nq][H][D], lse [B][H][Nq]) in fp64; with_abs=True appends
    absv = sum_j P_ij |v_jd| (error-scale helper for the tests)."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    B, Nq, H, D = q.shape
    Nk = k.shape[1]
    assert k.shape == (B, Nk, H, D) and v.shape == k.shape
    out = np.empty_like(q)
    lse = np.empty((B, H, Nq), dtype=np.float64)
    absv = np.empty_like(q) if with_abs else None
    _load().oracle_attn_fwd(_ptr(q), _ptr(k), _ptr(v), B, Nq, Nk, H, D, _ptr(out), _ptr(lse),
                            _ptr(absv) if with_abs else None)
    return (out, lse, absv) if with_abs else (out, lse)


def attn_fwd_rows(qrows, bh, k, v):
    """Exact forward for R explicit query rows: qrows [R][D], bh [R][2] =
    (batch, head) of each row.  Returns (out_rows [R][D], lse_rows [R])."""
    qrows, k, v = _f64(qrows), _f64(k), _f64(v)
    bh = np.ascontiguousarray(np.asarray(bh, dtype=np.int64))
    R, D = qrows.shape
    B, Nk, H, D2 = k.shape
    assert D == D2 and bh.shape == (R, 2)
    out = np.empty((R, D), dtype=np.float64)
    lse = np.empty((R,), dtype=np.float64)
    _load().oracle_attn_fwd_rows(_ptr(qrows), bh.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), R,
                                 _ptr(k), _ptr(v), B, Nk, H, D, _ptr(out), _ptr(lse))
    return out, lse


def attn_bwd_dq_rows(qrows, dorows, bh, k, v):
    """Exact dQ for R explicit query rows (qrows, dorows [R][D]; bh [R][2]) of
    self-attention over k, v [B][N][H][D].  Returns dq_rows [R][D]."""
    qrows, dorows, k, v = _f64(qrows), _f64(dorows), _f64(k), _f64(v)
    bh = np.ascontiguousarray(np.asarray(bh, dtype=np.int64))
    R, D = qrows.shape
    B, Nk, H, D2 = k.shape
    assert D == D2 and dorows.shape == (R, D) and bh.shape == (R, 2)
    out = np.empty((R, D), dtype=np.float64)
    _load().oracle_attn_bwd_dq_rows(_ptr(qrows), _ptr(dorows), bh.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), R,
                                    _ptr(k), _ptr(v), B, Nk, H, D, _ptr(out))
    return out


def attn_bwd_kv_rows(qh, kh, vh, doh, keys):
    """Exact (dK_j, dV_j) for the listed key rows of ONE head of self-attention:
    qh, kh, vh, doh [N][D] (that head's rows).  Recomputes lse_i and Delta_i for
    every query with the oracle's own fp64 forward.  Returns (dk_rows, dv_rows)
    [R][D].  Cost O(N^2 D) per call (the forward pass over the head)."""
    qh, kh, vh, doh = _f64(qh), _f64(kh), _f64(vh), _f64(doh)
    keys = np.ascontiguousarray(np.asarray(keys, dtype=np.int64))
    N, D = qh.shape
    assert kh.shape == (N, D) and vh.shape == (N, D) and doh.shape == (N, D)
    assert keys.ndim == 1 and (keys >= 0).all() and (keys < N).all()
    R = keys.shape[0]
    dk = np.empty((R, D), dtype=np.float64)
    dv = np.empty((R, D), dtype=np.float64)
    _load().oracle_attn_bwd_kv_rows(_ptr(qh), _ptr(kh), _ptr(vh), _ptr(doh), N, D,
                                    keys.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), R, _ptr(dk), _ptr(dv))
    return dk, dv


def delta(dout, out):
    """Delta_i = dO_i . O_i per (b, token, head) (the row term of
    dS = P (dP - Delta)), fp64, [B][N][H][D] -> [B][N][H]."""
    dout, out = _f64(dout), _f64(out)
    assert dout.shape == out.shape
    return (dout * out).sum(axis=-1)


def attn_bwd(q, k, v, dout, with_abs: bool = False):
    """Dense exact backward (self-attention).  Returns (dq, dk, dv, out, lse);
    with_abs=True appends (dq_abs, dk_abs, dv_abs), the error-scale sums of
    oracle.c (|dS|.|K|, |dS|^T.|Q| scaled, P^T.|dO|) used for tolerances."""
    q, k, v, dout = _f64(q), _f64(k), _f64(v), _f64(dout)
    B, N, H, D = q.shape
    assert k.shape == q.shape and v.shape == q.shape and dout.shape == q.shape
    dq, dk, dv, out = (np.empty_like(q) for _ in range(4))
    lse = np.empty((B, H, N), dtype=np.float64)
    gabs = np.empty((3,) + q.shape, dtype=np.float64) if with_abs else None
    _load().oracle_attn_bwd(_ptr(q), _ptr(k), _ptr(v), _ptr(dout), B, N, H, D,
                            _ptr(dq), _ptr(dk), _ptr(dv), _ptr(out), _ptr(lse),
                            _ptr(gabs) if with_abs else None)
    if with_abs:
        return dq, dk, dv, out, lse, (gabs[0], gabs[1], gabs[2])
    return dq, dk, dv, out, lse


from . import layer, lss, ulysses  # noqa: E402,F401
