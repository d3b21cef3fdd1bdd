"""Small forward + backward calls for compute-sanitizer (memcheck, racecheck,
synccheck): c1 (N=256, H=4, D=32) and ragged shapes at D = 64, 72, 128, in the
default and the deterministic backward mode, plus the rank-local layout steps
at P = 2 (simulated on one GPU).

    compute-sanitizer --tool memcheck python scripts/sanitize_run.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_15780_b200 as ua  # noqa: E402
import synth  # noqa: E402

CASES = [(1, 256, 4, 32), (1, 129, 2, 64), (1, 300, 2, 72), (1, 1000, 2, 128), (2, 384, 2, 64)]
for det in (False, True):
    ctx = ua.Context(P=1)
    ctx.set_deterministic(det)
    for B, N, H, D in CASES:
        q, k, v, do = (t.cuda() for t in synth.qkv(B, N, H, D, seed=1, with_do=True))
        r = ua.ulysses_attn_fwd(ctx, q, k, v)
        ua.ulysses_attn_bwd(ctx, q, k, v, r.out, r.lse, do)
        torch.cuda.synchronize()
    ctx.close()
# rank-local steps at P = 2: pack (+Delta), head attention fwd / bwd, unpack, peer push
B, N, H, D, P = 1, 512, 4, 64, 2
q, k, v, do = (t.cuda() for t in synth.qkv(B, N, H, D, seed=2, with_do=True))
sh = [[t[:, r * (N // P):(r + 1) * (N // P)].contiguous() for r in range(P)] for t in (q, k, v, do)]
sends = [ua.pack_seq_to_head([sh[w][r] for w in range(4)], P, dout=sh[3][r], out=sh[2][r]) for r in range(P)]
recv = [[torch.cat([sends[i][0][w][j] for i in range(P)]) for j in range(P)] for w in range(4)]
dl = [torch.cat([sends[i][1][j] for i in range(P)]) for j in range(P)]
for j in range(P):
    o, lse = ua.head_attn_fwd(recv[0][j], recv[1][j], recv[2][j], P, j)
    ua.head_attn_bwd(recv[0][j], recv[1][j], recv[2][j], recv[3][j], lse, dl[j], P, j)
    ua.unpack_head_to_seq([o.view(P, N // P, B, H // P, D)], P)
bufs = [torch.zeros(4 * B * N * (H // P) * D * 2 + B * N * (H // P) * 4, dtype=torch.uint8, device="cuda")
        for _ in range(P)]
for r in range(P):
    ua.push_seq_to_head([sh[w][r] for w in range(4)], bufs, P, r, dout=sh[3][r], out=sh[2][r])
torch.cuda.synchronize()
print("SANITIZE_RUN_OK")
