"""Throughput of the projection GEMM (ua_gemm_bf16) at the c4 layer's shapes
(P = 1: M = 188,416 tokens, E = 2,048), CUDA events, best of 5 after warm-up.
Prints TFLOP/s per GEMM kind (tuning / DESIGN aid, not a test)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_15780_b200 as ua  # noqa: E402

M, E = int(os.environ.get("GEMM_M", 188416)), int(os.environ.get("GEMM_E", 2048))
x = torch.randn(M, E, device="cuda").bfloat16()
w = [torch.randn(E, E, device="cuda").bfloat16() for _ in range(3)]
g = [torch.randn(M, E, device="cuda").bfloat16() for _ in range(3)]
cases = {
    "y = x W^T      (M x E x E)": (lambda: ua.gemm([x], [w[0]], False, False), 2.0 * M * E * E),
    "dx = sum g_i W_i (3 segments)": (lambda: ua.gemm(g, w, False, True), 6.0 * M * E * E),
    "dW = g^T x     (E x E x M, fp32 out)": (lambda: ua.gemm([g[0]], [x], True, True, out_f32=True), 2.0 * M * E * E),
}
for name, (fn, flop) in cases.items():
    for _ in range(2):
        fn()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"{name:40s} {best:8.3f} ms  {flop / best / 1e9:7.1f} TFLOP/s")
