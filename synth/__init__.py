"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: it only draws random
numbers and rounds them to bf16.  Both the tests/bench (GPU side) and the
oracle side take their inputs from here; the oracle never receives a value
computed by the CUDA path.

Recipe:
  * Q, K, V, dO ~ N(0, sigma^2) i.i.d. (sigma = 1 for the performance runs and
    gate A; sigma_qk = 2 for Q and K in the sharpness gate B), drawn as float32
    with numpy's PCG64 generator keyed by (seed, tensor id), then rounded to
    bf16 (round-to-nearest-even, torch's conversion).
  * The whole GLOBAL tensor [B][N][H][D] is drawn in one order and sequence
    shards are slices of it, so the data are identical for every P.
  * Seeds: q=1234, k=1235, v=1236, dO=1237 (offset by the test's seed).
  * Shapes follow BASELINE.json configs (c1..c5); the paper's 188,416-token
    workload is 92 channels x 2,048 patches.
"""
from __future__ import annotations

import numpy as np
import torch

TENSOR_IDS = {"q": 0, "k": 1, "v": 2, "do": 3}
BASE_SEED = 1234

# BASELINE.json "configs"; c3 and c4 list several P values, c5 is P=8.
CONFIGS = {
    "c1": dict(B=1, N=256, H=4, D=32, P=(1,)),
    "c2": dict(B=1, N=8192, H=16, D=64, P=(1,)),
    "c3": dict(B=1, N=65536, H=16, D=128, P=(2, 4, 8)),
    "c4": dict(B=1, N=188416, H=32, D=64, P=(1, 2, 4, 8)),
    "c5": dict(B=1, N=1048576, H=32, D=128, P=(8,)),
}


def normal_f32(shape, seed: int, name: str, sigma: float = 1.0) -> np.ndarray:
    """float32 N(0, sigma^2) draws for tensor ``name`` (q/k/v/do)."""
    rng = np.random.Generator(np.random.PCG64([int(seed), TENSOR_IDS[name]]))
    x = rng.standard_normal(size=int(np.prod(shape)), dtype=np.float32).reshape(shape)
    if sigma != 1.0:
        x *= np.float32(sigma)
    return x


def normal_bf16(shape, seed: int, name: str, sigma: float = 1.0) -> torch.Tensor:
    """bf16-rounded CPU tensor of the draws above."""
    return torch.from_numpy(normal_f32(shape, seed, name, sigma)).to(torch.bfloat16)


def qkv(B, N, H, D, seed: int = BASE_SEED, sigma_qk: float = 1.0, with_do: bool = False):
    """Global bf16 CPU tensors (q, k, v[, dout]) of shape [B][N][H][D]."""
    shape = (B, N, H, D)
    out = [normal_bf16(shape, seed, "q", sigma_qk),
           normal_bf16(shape, seed, "k", sigma_qk),
           normal_bf16(shape, seed, "v")]
    if with_do:
        out.append(normal_bf16(shape, seed, "do"))
    return tuple(out)


def to_f64(x: torch.Tensor) -> np.ndarray:
    """Exact widening of bf16 values to float64 numpy (for the oracle)."""
    return x.to(torch.float64).numpy()
