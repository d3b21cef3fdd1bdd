"""Oracle for the attention layer around the Ulysses attention.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md P:346 (§5.4) and P:425 (§6.1): per layer, DeepSpeed-Ulysses issues
"two all-to-all calls in the forward pass and two all-to-all calls + all
reduce in the backward pass"; the all-reduce sums the SP group's weight
gradients.  Reading (R16): bias-free projections y = x W^T with
W_qkv = [Wq; Wk; Wv] ([3E][E]) and Wo ([E][E]), E = H * D, head h = columns
h*D .. h*D+D-1 of q, k, v, o.  Because every rank holds the same weights and
the attention is exact, the sequence-parallel layer computes the same y, dx
as the unsharded layer, and the all-reduced weight gradients equal the
unsharded ones (sums over all tokens).  This module writes the unsharded
layer out in fp64: matmuls (numpy, library primitive) and the dense attention
of oracle.c.
"""
from __future__ import annotations

import numpy as np


def _split(t, H):
    B, N, E = t.shape
    return t.reshape(B, N, H, E // H)


def layer_fwd(x, w_qkv, w_o, H: int):
    """x [B][N][E], w_qkv [3E][E], w_o [E][E] -> (y [B][N][E], (q, k, v, o, lse))."""
    from . import attn_fwd
    x, w_qkv, w_o = (np.asarray(t, np.float64) for t in (x, w_qkv, w_o))
    E = x.shape[-1]
    q, k, v = (x @ w_qkv[i * E:(i + 1) * E].T for i in range(3))      # x W^T
    o, lse = attn_fwd(_split(q, H), _split(k, H), _split(v, H))
    o = o.reshape(x.shape)
    y = o @ w_o.T
    return y, (q, k, v, o, lse)


def layer_bwd(x, w_qkv, w_o, dy, H: int):
    """Returns (dx, dw_qkv, dw_o) of the loss <y, dy>.
        do = dy Wo, dWo = dy^T o; (dq, dk, dv) = attention backward;
        dx = dq Wq + dk Wk + dv Wv; dW_i = dqkv_i^T x (summed over all tokens)."""
    from . import attn_bwd
    x, w_qkv, w_o, dy = (np.asarray(t, np.float64) for t in (x, w_qkv, w_o, dy))
    E = x.shape[-1]
    _, (q, k, v, o, _) = layer_fwd(x, w_qkv, w_o, H)
    do = dy @ w_o
    dw_o = np.einsum("bnj,bni->ji", dy, o)                                  # dy^T o
    dq, dk, dv, _, _ = attn_bwd(_split(q, H), _split(k, H), _split(v, H), _split(do, H))
    g = [t.reshape(x.shape) for t in (dq, dk, dv)]
    dx = sum(g[i] @ w_qkv[i * E:(i + 1) * E] for i in range(3))
    dw_qkv = np.concatenate([np.einsum("bnj,bni->ji", g[i], x) for i in range(3)], axis=0)
    return dx, dw_qkv, dw_o
