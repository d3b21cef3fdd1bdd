"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: it only draws random
numbers and rounds them to bf16.  Both the tests/bench (GPU side) and the
oracle side take their inputs from here; the oracle never receives a value
computed by the CUDA path.

Recipe:
  * Q, K, V, dO ~ N(0, sigma^2) i.i.d. (sigma = 1 for the performance runs and
    gate A; sigma_qk = 2 for Q and K in the sharpness gate B), drawn as
    float32 and rounded to bf16 (round-to-nearest-even, torch's conversion).
  * Counter-based by construction: the values of tokens [1024 k, 1024 k + 1024)
    of (tensor, batch b, head h) come from their own numpy PCG64 stream keyed
    by (seed, tensor id, b, h, k).  Any rank can draw exactly its sequence
    shard, and the oracle can redraw any head, without materialising the
    global tensor (c5 is 4.3e9 values per tensor); the data are identical for
    every P.
  * Seeds: BASE_SEED = 1234 (offset by the test's seed); tensor ids q=0, k=1,
    v=2, dO=3; the attention layer's x=4, dy=5 (N(0,1), [B][N][E]) and weights
    w_qkv=6, w_o=7 (N(0, 1/E), so the projected q, k, v have unit scale).
  * Shapes follow BASELINE.json configs (c1..c5); the paper's 188,416-token
    workload is 92 channels x 2,048 patches.
"""
from __future__ import annotations

import numpy as np
import torch

TENSOR_IDS = {"q": 0, "k": 1, "v": 2, "do": 3, "x": 4, "dy": 5, "w_qkv": 6, "w_o": 7}
BASE_SEED = 1234
BLOCK = 1024

# BASELINE.json "configs"; c3 and c4 list several P values, c5 is P=8.
CONFIGS = {
    "c1": dict(B=1, N=256, H=4, D=32, P=(1,)),
    "c2": dict(B=1, N=8192, H=16, D=64, P=(1,)),
    "c3": dict(B=1, N=65536, H=16, D=128, P=(2, 4, 8)),
    "c4": dict(B=1, N=188416, H=32, D=64, P=(1, 2, 4, 8)),
    "c5": dict(B=1, N=1048576, H=32, D=128, P=(8,)),
}


def _block(seed: int, name: str, b: int, h: int, k: int, D: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64([int(seed), TENSOR_IDS[name], int(b), int(h), int(k)]))
    return rng.standard_normal(size=(BLOCK, D), dtype=np.float32)


def normal_f32(B, N, H, D, seed: int, name: str, sigma: float = 1.0, n0: int = 0, n1: int | None = None,
               heads=None) -> np.ndarray:
    """float32 draws of tokens [n0, n1) and the listed heads (default all) of
    the global [B][N][H][D] tensor ``name``: shape [B][n1-n0][len(heads)][D]."""
    n1 = N if n1 is None else n1
    heads = list(range(H)) if heads is None else list(heads)
    out = np.empty((B, n1 - n0, len(heads), D), dtype=np.float32)

    def fill(job):
        b, hi, h = job
        for k in range(n0 // BLOCK, (n1 + BLOCK - 1) // BLOCK):
            lo, hi_ = max(n0, k * BLOCK), min(n1, (k + 1) * BLOCK)
            out[b, lo - n0:hi_ - n0, hi, :] = _block(seed, name, b, h, k, D)[lo - k * BLOCK:hi_ - k * BLOCK]

    jobs = [(b, hi, h) for b in range(B) for hi, h in enumerate(heads)]
    if len(jobs) > 1 and (n1 - n0) * D >= (1 << 20):
        from concurrent.futures import ThreadPoolExecutor  # numpy's generator releases the GIL
        with ThreadPoolExecutor(max_workers=min(16, len(jobs))) as ex:
            list(ex.map(fill, jobs))
    else:
        for job in jobs:
            fill(job)
    if sigma != 1.0:
        out *= np.float32(sigma)
    return out


def normal_bf16(B, N, H, D, seed: int, name: str, sigma: float = 1.0, **kw) -> torch.Tensor:
    """bf16-rounded CPU tensor of the draws above."""
    return torch.from_numpy(normal_f32(B, N, H, D, seed, name, sigma, **kw)).to(torch.bfloat16)


def qkv(B, N, H, D, seed: int = BASE_SEED, sigma_qk: float = 1.0, with_do: bool = False, n0: int = 0,
        n1: int | None = None, heads=None):
    """bf16 CPU tensors (q, k, v[, dout]) of tokens [n0, n1) (default: the
    whole sequence) and the listed heads of the global [B][N][H][D] tensors."""
    kw = dict(n0=n0, n1=n1, heads=heads)
    out = [normal_bf16(B, N, H, D, seed, "q", sigma_qk, **kw),
           normal_bf16(B, N, H, D, seed, "k", sigma_qk, **kw),
           normal_bf16(B, N, H, D, seed, "v", **kw)]
    if with_do:
        out.append(normal_bf16(B, N, H, D, seed, "do", **kw))
    return tuple(out)


def to_f64(x: torch.Tensor) -> np.ndarray:
    """Exact widening of bf16 values to float64 numpy (for the oracle)."""
    return x.to(torch.float64).numpy()


def layer_inputs(B, N, H, D, seed: int = BASE_SEED, n0: int = 0, n1: int | None = None):
    """Attention-layer inputs (bf16 CPU): x, dy [B][n1-n0][E] (tokens [n0, n1)
    of the global sequence), w_qkv [3E][E], w_o [E][E]; E = H * D."""
    E = H * D
    n1 = N if n1 is None else n1
    x = normal_bf16(B, N, 1, E, seed, "x", n0=n0, n1=n1).reshape(B, n1 - n0, E)
    dy = normal_bf16(B, N, 1, E, seed, "dy", n0=n0, n1=n1).reshape(B, n1 - n0, E)
    w_qkv = normal_bf16(1, 3 * E, 1, E, seed, "w_qkv", sigma=E ** -0.5).reshape(3 * E, E)
    w_o = normal_bf16(1, E, 1, E, seed, "w_o", sigma=E ** -0.5).reshape(E, E)
    return x, dy, w_qkv, w_o
