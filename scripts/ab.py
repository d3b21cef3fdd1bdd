"""Interleaved A/B timing of library variants (tuning aid, not a test).

    python scripts/ab.py --libs paper_2405_15780_b200/libulysses_attn.so variants/libX.so \
        --N 32768 --H 32 --D 64 --what fwd|bwd|both --rounds 6

Each round times every library once (fwd and/or bwd at P=1 through the C ABI,
CUDA events), so power-cap / clock drift hits all variants alike.  Prints the
median TFLOP/s per library."""
import argparse
import ctypes
import statistics

import torch

ap = argparse.ArgumentParser()
ap.add_argument("--libs", nargs="+", required=True)
ap.add_argument("--N", type=int, default=32768)
ap.add_argument("--H", type=int, default=32)
ap.add_argument("--D", type=int, default=64)
ap.add_argument("--what", default="both")
ap.add_argument("--rounds", type=int, default=6)
ap.add_argument("--det", action="store_true", help="deterministic backward (ua_ctx_set_deterministic)")
a = ap.parse_args()

vp, i64, i32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
torch.manual_seed(0)
B, N, H, D = 1, a.N, a.H, a.D
q, k, v, do = (torch.randn(B, N, H, D, device="cuda").bfloat16() for _ in range(4))
out = torch.empty_like(q)
lse = torch.empty(B, H, N, device="cuda")
dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
libs = []
for path in a.libs:
    L = ctypes.CDLL(path)
    L.ua_ctx_create.argtypes = [ctypes.c_char_p, i32, i32, i32, ctypes.POINTER(vp)]
    L.ua_workspace_size.argtypes = [i64, i64, i32, i32, i32, ctypes.POINTER(sz), ctypes.POINTER(sz)]
    L.ua_ulysses_attn_fwd.argtypes = [vp, vp, vp, vp, vp, vp, i64, i64, i32, i32, i32, vp, sz, vp]
    L.ua_ulysses_attn_bwd.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, i32, i32, i32, vp, sz, vp]
    h = vp(0)
    assert L.ua_ctx_create(None, 1, 0, torch.cuda.current_device(), ctypes.byref(h)) == 0
    if a.det:
        L.ua_ctx_set_deterministic.argtypes = [vp, i32]
        assert L.ua_ctx_set_deterministic(h, 1) == 0
    fb, bb = sz(0), sz(0)
    L.ua_workspace_size(B, N, H, D, 1, ctypes.byref(fb), ctypes.byref(bb))
    ws = torch.empty(max(fb.value, bb.value, 256), dtype=torch.uint8, device="cuda")
    libs.append((path, L, h, ws))

P = lambda t: vp(t.data_ptr())  # noqa: E731
stream = vp(torch.cuda.current_stream().cuda_stream)


def run(L, h, ws, what):
    if what in ("fwd", "both"):
        assert L.ua_ulysses_attn_fwd(h, P(q), P(k), P(v), P(out), P(lse), B, N, H, D, 1, P(ws), ws.numel(), stream) == 0
    if what in ("bwd", "both"):
        assert L.ua_ulysses_attn_bwd(h, P(q), P(k), P(v), P(out), P(lse), P(do), P(dq), P(dk), P(dv), B, N, H, D, 1,
                                     P(ws), ws.numel(), stream) == 0


flops = {"fwd": 4.0, "bwd": 10.0, "both": 14.0}[a.what] * B * N * N * H * D
for path, L, h, ws in libs:  # warm-up (and lse for the bwd)
    run(L, h, ws, "both")
torch.cuda.synchronize()
res = {path: [] for path, *_ in libs}
for r in range(a.rounds):
    for path, L, h, ws in (libs if r % 2 == 0 else libs[::-1]):
        if a.what == "bwd":
            run(L, h, ws, "fwd")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(L, h, ws, a.what)
        e1.record()
        torch.cuda.synchronize()
        res[path].append(flops / (e0.elapsed_time(e1) * 1e-3) / 1e12)
for path, vals in res.items():
    print(f"{statistics.median(vals):8.1f} TFLOP/s  (min {min(vals):.1f} max {max(vals):.1f})  {a.what} N={N} H={H} D={D}  {path}")
