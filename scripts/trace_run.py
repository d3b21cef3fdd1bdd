"""Run one fwd (+bwd) through a UA_TRACE=1 variant library and summarise the
per-CTA event timeline (tuning aid).  Usage:
    UA_TRACE_FILE=/tmp/t.txt python scripts/trace_run.py variants/libtrace.so --N 32768
"""
import argparse
import collections
import ctypes
import os
import statistics

import torch

ap = argparse.ArgumentParser()
ap.add_argument("lib")
ap.add_argument("--N", type=int, default=32768)
ap.add_argument("--H", type=int, default=32)
ap.add_argument("--D", type=int, default=64)
ap.add_argument("--bwd", action="store_true")
a = ap.parse_args()
path = os.environ.setdefault("UA_TRACE_FILE", "/tmp/ua_trace.txt")
if os.path.exists(path):
    os.remove(path)
vp, i64, i32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
L = ctypes.CDLL(a.lib)
L.ua_ctx_create.argtypes = [ctypes.c_char_p, i32, i32, i32, ctypes.POINTER(vp)]
L.ua_workspace_size.argtypes = [i64, i64, i32, i32, i32, ctypes.POINTER(sz), ctypes.POINTER(sz)]
L.ua_ulysses_attn_fwd.argtypes = [vp, vp, vp, vp, vp, vp, i64, i64, i32, i32, i32, vp, sz, vp]
L.ua_ulysses_attn_bwd.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, i32, i32, i32, vp, sz, vp]
B, N, H, D = 1, a.N, a.H, a.D
q, k, v, do = (torch.randn(B, N, H, D, device="cuda").bfloat16() for _ in range(4))
out, lse = torch.empty_like(q), torch.empty(B, H, N, device="cuda")
dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
h = vp(0)
L.ua_ctx_create(None, 1, 0, 0, ctypes.byref(h))
fb, bb = sz(0), sz(0)
L.ua_workspace_size(B, N, H, D, 1, ctypes.byref(fb), ctypes.byref(bb))
ws = torch.empty(max(fb.value, bb.value, 256), dtype=torch.uint8, device="cuda")
P = lambda t: vp(t.data_ptr())  # noqa: E731
for _ in range(2):
    os.path.exists(path) and os.remove(path)
    assert L.ua_ulysses_attn_fwd(h, P(q), P(k), P(v), P(out), P(lse), B, N, H, D, 1, P(ws), ws.numel(), None) == 0
    if a.bwd:
        assert L.ua_ulysses_attn_bwd(h, P(q), P(k), P(v), P(out), P(lse), P(do), P(dq), P(dk), P(dv), B, N, H, D, 1,
                                     P(ws), ws.numel(), None) == 0
    torch.cuda.synchronize()

ev = collections.defaultdict(dict)   # (tag, role, tile) -> {ev: clock}
for line in open(path):
    tag, clk, role, tile, e = line.split()
    ev[(tag, int(role), int(tile))][int(e)] = int(clk)
for tag in sorted({k[0] for k in ev}):
    roles = sorted({k[1] for k in ev if k[0] == tag})
    t0 = min(c for k, d in ev.items() if k[0] == tag for c in d.values())
    print(f"== {tag}: roles {roles}")
    for role in roles:
        tiles = sorted(k[2] for k in ev if k[0] == tag and k[1] == role)
        evs = sorted({e for t in tiles for e in ev[(tag, role, t)]})
        # durations between consecutive event ids, median over tiles (skip first 2 tiles)
        mid = tiles[2:-1] if len(tiles) > 4 else tiles
        parts = []
        for e0, e1 in zip(evs, evs[1:]):
            d = [ev[(tag, role, t)][e1] - ev[(tag, role, t)][e0] for t in mid
                 if e0 in ev[(tag, role, t)] and e1 in ev[(tag, role, t)]]
            if d:
                parts.append(f"{e0}->{e1}: {statistics.median(d):.0f}")
        starts = [min(ev[(tag, role, t)].values()) for t in mid]
        period = statistics.median([b - a for a, b in zip(starts, starts[1:])]) if len(starts) > 2 else 0
        print(f"  role {role}: {len(tiles)} tiles, period {period:.0f} clk | " + "  ".join(parts))
