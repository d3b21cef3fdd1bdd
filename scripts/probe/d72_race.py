"""Probe: is the D=72 backward deterministic (dk bitwise across runs)?  (debug aid)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle  # noqa: E402
import paper_2405_15780_b200 as ua  # noqa: E402
import synth  # noqa: E402

ctx = ua.Context(P=1)
for N, H, sigma, D in [(300, 2, 2.0, 72), (300, 1, 2.0, 72), (1000, 3, 2.0, 72), (1000, 3, 2.0, 64)]:
    q, k, v, do = synth.qkv(1, N, H, D, seed=100 + N, sigma_qk=sigma, with_do=True)
    qc, kc, vc, dc = (t.cuda() for t in (q, k, v, do))
    r = ua.ulysses_attn_fwd(ctx, qc, kc, vc)
    runs = []
    for _ in range(4):
        g = ua.ulysses_attn_bwd(ctx, qc, kc, vc, r.out, r.lse, dc)
        torch.cuda.synchronize()
        runs.append([t.float().cpu().numpy() for t in g])
    same_dk = all(np.array_equal(runs[0][1], x[1]) for x in runs[1:])
    same_dv = all(np.array_equal(runs[0][2], x[2]) for x in runs[1:])
    ref = oracle.attn_bwd(*(synth.to_f64(t) for t in (q, k, v, do)))
    rl = [[float(np.linalg.norm(x[i] - ref[i]) / np.linalg.norm(ref[i])) for i in range(3)] for x in runs]
    print(N, H, sigma, D, "dk same", same_dk, "dv same", same_dv, "relL2 per run", np.round(rl, 4).tolist(), flush=True)
