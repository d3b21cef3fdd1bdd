"""Oracle for contiguous key-segment ("LSS chunking") attention and the exact
merge of partial results.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md P:72 (§1): LSS distributes "long sequences across GPUs as contiguous
segments" and aggregates "partial self-attention scores"; P:166 (§2.5): "each
GPU computing a partial self-attention for its segment".  BASELINE.json
north_star: "online softmax and Long-Sequence-Segmentation chunking so the NxN
matrix is never materialised".

Reading (Q15): a key range [0, N) is split into contiguous segments
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
