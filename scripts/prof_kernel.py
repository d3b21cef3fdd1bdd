"""Small driver for ncu captures of the attention kernels:
    python scripts/prof_kernel.py --N 32768 --H 32 --D 64 [--iters 2]
Runs Ulysses fwd + bwd at P=1 on synthetic N(0,1) bf16 inputs."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_15780_b200 as ua  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=32768)
ap.add_argument("--H", type=int, default=32)
ap.add_argument("--D", type=int, default=64)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--fwd-only", action="store_true")
ap.add_argument("--det", action="store_true", help="deterministic backward")
a = ap.parse_args()
torch.manual_seed(0)
q, k, v, do = (torch.randn(1, a.N, a.H, a.D, device="cuda").bfloat16() for _ in range(4))
ctx = ua.Context(P=1)
ctx.set_deterministic(a.det)
for _ in range(a.iters):
    r = ua.ulysses_attn_fwd(ctx, q, k, v)
    if not a.fwd_only:
        ua.ulysses_attn_bwd(ctx, q, k, v, r.out, r.lse, do)
torch.cuda.synchronize()
ctx.enable_timing(True)
r = ua.ulysses_attn_fwd(ctx, q, k, v)
if not a.fwd_only:
    ua.ulysses_attn_bwd(ctx, q, k, v, r.out, r.lse, do)
t = ctx.phase_times()
f = 4.0 * a.N * a.N * a.H * a.D
for name, (ms, n) in t.items():
    if n:
        fl = f if name == "attn_fwd" else (2.5 * f if name == "attn_bwd" else 0)
        print(f"{name:12s} {ms:9.3f} ms" + (f"  {fl / ms / 1e9:7.1f} TFLOP/s" if fl else ""))
print("PROF_OK")
