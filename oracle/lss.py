"""Oracle for contiguous key-segment ("LSS chunking") attention and the exact
merge of partial results.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md P:72 (§1): LSS distributes "long sequences across GPUs as contiguous
segments" and aggregates "partial self-attention scores"; P:166 (§2.5): "each
GPU computing a partial self-attention for its segment".  BASELINE.json
north_star: "online softmax and Long-Sequence-Segmentation chunking so the NxN
matrix is never materialised".

Reading (R11): a key range [0, N) is split into contiguous segments
s; each gives (O_s, lse_s) = exact attention of the queries over that segment
only.  With lse = ln sum_s exp(lse_s) the full result is
    O = sum_s exp(lse_s - lse) O_s
because exp(lse_s - lse) is the softmax mass segment s holds.  This module
writes that out literally (logaddexp is numpy's, a library primitive).
"""
from __future__ import annotations

import numpy as np


def segment_fwd(q, k, v, j0: int, j1: int):
    """Attention of all queries over keys [j0, j1) only.  Returns (O_s, lse_s)
    with O_s [B][Nq][H][D], lse_s [B][H][Nq]."""
    from . import attn_fwd
    return attn_fwd(q, np.ascontiguousarray(k[:, j0:j1]), np.ascontiguousarray(v[:, j0:j1]))


def merge(parts):
    """parts = [(O_s [B][N][H][D], lse_s [B][H][N]), ...] -> (O, lse)."""
    lse = parts[0][1]
    for _, l in parts[1:]:
        lse = np.logaddexp(lse, l)
    out = np.zeros_like(parts[0][0], dtype=np.float64)
    for o, l in parts:
        w = np.exp(l - lse)                      # [B][H][N]
        out += np.transpose(w, (0, 2, 1))[..., None] * o
    return out, lse


def chunked_fwd(q, k, v, bounds):
    """Split keys at ``bounds`` = [0, b1, ..., N] and merge the segments."""
    parts = [segment_fwd(q, k, v, bounds[s], bounds[s + 1]) for s in range(len(bounds) - 1)]
    return merge(parts)


# --------------------------------------------------------------- LSS sequence parallelism
# PAPER.md P:166 (§2.5): "sequences are divided into segments, with each GPU
# computing a partial self-attention for its segment"; P:72 (§1): contiguous
# segments, partial results aggregated.  Reading (R14): rank r owns
# query/key/value rows [r*Nl, (r+1)*Nl) of every head; K and V are gathered,
# so rank r's output rows are exact attention of its queries over all keys.
# In the backward, rank r's queries contribute a PARTIAL sum to every dK_j,
# dV_j; the sums over ranks are scattered back to the key owners.


def sp_fwd(q, k, v, P: int):
    """Per-rank forward.  Returns ([out_r [B][Nl][H][D]], [lse_r [B][H][Nl]])."""
    from . import attn_fwd
    N = q.shape[1]
    Nl = N // P
    outs, lses = [], []
    for r in range(P):
        kg = np.concatenate([k[:, s * Nl:(s + 1) * Nl] for s in range(P)], axis=1)   # the all-gather
        vg = np.concatenate([v[:, s * Nl:(s + 1) * Nl] for s in range(P)], axis=1)
        o, lse = attn_fwd(q[:, r * Nl:(r + 1) * Nl], kg, vg)
        outs.append(o)
        lses.append(lse)
    return outs, lses


def sp_bwd_partial(q_r, do_r, o_r, lse_r, k, v):
    """Rank r's backward (S:181-183 restricted to its query rows i):
        P_ij  = exp(s_ij - lse_i),  s_ij = q_i.k_j / sqrt(D)
        Delta_i = dO_i.o_i,   dS_ij = P_ij (dO_i.v_j - Delta_i)
        dQ_i = scale sum_j dS_ij k_j          (complete: all keys are local)
        dK_j^(r) = scale sum_{i in r} dS_ij q_i,  dV_j^(r) = sum_{i in r} P_ij dO_i   (partial)
    q_r, do_r, o_r [B][Nl][H][D]; lse_r [B][H][Nl]; k, v [B][N][H][D] (gathered)."""
    B, Nl, H, D = q_r.shape
    scale = 1.0 / np.sqrt(D)
    dq = np.zeros_like(q_r)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    for b in range(B):
        for h in range(H):
            qi, di, oi = q_r[b, :, h], do_r[b, :, h], o_r[b, :, h]       # [Nl][D]
            kj, vj = k[b, :, h], v[b, :, h]                              # [N][D]
            p = np.exp(scale * (qi @ kj.T) - lse_r[b, h][:, None])       # [Nl][N]
            delta = np.sum(di * oi, axis=1)                              # [Nl]
            ds = p * (di @ vj.T - delta[:, None])
            dq[b, :, h] = scale * (ds @ kj)
            dk[b, :, h] = scale * (ds.T @ qi)
            dv[b, :, h] = p.T @ di
    return dq, dk, dv


def sp_bwd(q, k, v, dout, P: int):
    """Per-rank backward of the LSS strategy: every rank's partial (dK, dV)
    over all keys, then the reduce-scatter (sum over ranks, rows of rank r to
    rank r).  Returns ([dq_r], [dk_r], [dv_r]), each [B][Nl][H][D]."""
    N = q.shape[1]
    Nl = N // P
    outs, lses = sp_fwd(q, k, v, P)
    parts = [sp_bwd_partial(q[:, r * Nl:(r + 1) * Nl], dout[:, r * Nl:(r + 1) * Nl], outs[r], lses[r], k, v)
             for r in range(P)]
    dqs = [p[0] for p in parts]
    dk_sum = sum(p[1] for p in parts)                                    # the reduce ...
    dv_sum = sum(p[2] for p in parts)
    dks = [dk_sum[:, r * Nl:(r + 1) * Nl] for r in range(P)]             # ... and the scatter
    dvs = [dv_sum[:, r * Nl:(r + 1) * Nl] for r in range(P)]
    return dqs, dks, dvs
