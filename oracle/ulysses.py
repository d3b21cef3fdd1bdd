"""Oracle for DeepSpeed-Ulysses sequence parallelism (data movement only).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md P:165 (§2.5): "DeepSpeed-Ulysses partitions the input data along the
sequence dimension ... employs an all-to-all collective communication to ensure
that each GPU receives a complete sequence, but only for a non-overlapping
subset of the attention heads".  P:425 (§6.1): "two all-to-all calls in the
forward pass and two all-to-all calls + all reduce in the backward pass".
SPEC.md S:122: all_to_all — "output[j] on rank i equals input[i] on rank j";
S:234: sequence shards are contiguous token ranges in rank order; S:244:
P must divide H and N and P <= H (errors otherwise).

Readings: rank r owns tokens [r*N/P, (r+1)*N/P) and,
after the all-to-all, heads [r*H/P, (r+1)*H/P) (contiguous head blocks, Q3).
The all-reduce in the backward is the weight-gradient sync of the model's
projections; the attention op has no weights, so it has none (Q9).

Everything here is index bookkeeping on numpy arrays; the only arithmetic is
the dense attention of the parent module, run per rank on its head shard.
"""
from __future__ import annotations

import numpy as np


class HeadDivisibilityError(ValueError):
    """P does not divide H, or P > H."""


class SeqDivisibilityError(ValueError):
    """P does not divide N."""


def check(N: int, H: int, P: int) -> None:
    if P > H or H % P != 0:
        raise HeadDivisibilityError(f"P={P} must divide H={H} and be <= H")
    if N % P != 0:
        raise SeqDivisibilityError(f"P={P} must divide N={N}")


def shard_seq(x: np.ndarray, P: int) -> list[np.ndarray]:
    """[B][N][H][D] -> P contiguous token ranges [B][N/P][H][D]."""
    B, N, H, D = x.shape
    n = N // P
    return [x[:, r * n:(r + 1) * n] for r in range(P)]


def gather_seq(shards: list[np.ndarray]) -> np.ndarray:
    return np.concatenate(shards, axis=1)


def all_to_all(sends: list[list[np.ndarray]]) -> list[list[np.ndarray]]:
    """sends[i][j] = chunk rank i sends to rank j.  Returns recv with
    recv[j][i] = sends[i][j] (output[j] on rank i == input[i] on rank j)."""
    P = len(sends)
    assert all(len(s) == P for s in sends)
    return [[sends[i][j] for i in range(P)] for j in range(P)]


def seq_to_head(x_shards: list[np.ndarray], P: int) -> list[np.ndarray]:
    """Forward all-to-all: rank i holds [B][N/P][H][D]; sends head block j to
    rank j; rank j concatenates what it receives in source-rank order along the
    sequence -> [B][N][H/P][D] (full sequence, its head subset)."""
    H = x_shards[0].shape[2]
    hl = H // P
    sends = [[x[:, :, j * hl:(j + 1) * hl] for j in range(P)] for x in x_shards]
    recv = all_to_all(sends)
    return [np.concatenate(recv[j], axis=1) for j in range(P)]


def head_to_seq(y_heads: list[np.ndarray], P: int) -> list[np.ndarray]:
    """Return all-to-all: rank j holds [B][N][H/P][D]; sends token range i to
    rank i; rank i concatenates received head blocks in source-rank order
    along heads -> [B][N/P][H][D]."""
    N = y_heads[0].shape[1]
    n = N // P
    sends = [[y[:, i * n:(i + 1) * n] for i in range(P)] for y in y_heads]
    recv = all_to_all(sends)
    return [np.concatenate(recv[i], axis=2) for i in range(P)]


def ulysses_fwd(q_shards, k_shards, v_shards, P: int):
    """Ulysses forward on P simulated ranks.  Inputs: per-rank [B][N/P][H][D].
    Returns (out_shards per rank [B][N/P][H][D], lse per rank [B][H/P][N])."""
    from . import attn_fwd
    B, n, H, D = q_shards[0].shape
    check(n * P, H, P)
    qh, kh, vh = (seq_to_head(x, P) for x in (q_shards, k_shards, v_shards))  # a2a #1 (fused)
    outs, lses = [], []
    for j in range(P):
        o, lse = attn_fwd(qh[j], kh[j], vh[j])
        outs.append(o)
        lses.append(lse)
    return head_to_seq(outs, P), lses                                        # a2a #2


def ulysses_bwd(q_shards, k_shards, v_shards, do_shards, P: int):
    """Ulysses backward on P simulated ranks.  Returns per-rank (dq, dk, dv)
    shards [B][N/P][H][D]."""
    from . import attn_bwd
    B, n, H, D = q_shards[0].shape
    check(n * P, H, P)
    qh, kh, vh, doh = (seq_to_head(x, P) for x in (q_shards, k_shards, v_shards, do_shards))  # a2a #3
    dqs, dks, dvs = [], [], []
    for j in range(P):
        dq, dk, dv, _, _ = attn_bwd(qh[j], kh[j], vh[j], doh[j])
        dqs.append(dq)
        dks.append(dk)
        dvs.append(dv)
    return head_to_seq(dqs, P), head_to_seq(dks, P), head_to_seq(dvs, P)     # a2a #4
