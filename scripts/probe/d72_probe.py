"""Probe: D=72 backward errors per gradient over a few shapes (debug aid)."""
import itertools
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle  # noqa: E402
import paper_2405_15780_b200 as ua  # noqa: E402
import synth  # noqa: E402

ctx = ua.Context(P=1)
for N, H, sigma, D in [(300, 2, 1.0, 72), (300, 3, 1.0, 72), (300, 2, 2.0, 72), (1000, 2, 1.0, 72), (1000, 3, 1.0, 72),
                       (1000, 3, 2.0, 72), (1000, 3, 2.0, 64), (256, 1, 1.0, 72), (512, 1, 1.0, 72)]:
    q, k, v, do = synth.qkv(1, N, H, D, seed=100 + N, sigma_qk=sigma, with_do=True)
    qc, kc, vc, dc = (t.cuda() for t in (q, k, v, do))
    r = ua.ulysses_attn_fwd(ctx, qc, kc, vc)
    g = ua.ulysses_attn_bwd(ctx, qc, kc, vc, r.out, r.lse, dc)
    torch.cuda.synchronize()
    ref = oracle.attn_bwd(*(synth.to_f64(t) for t in (q, k, v, do)))
    msg = []
    for name, x, y in zip(("dq", "dk", "dv"), g, ref[:3]):
        x = x.float().cpu().numpy()
        e = np.abs(x - y)
        rl = np.linalg.norm(x - y) / np.linalg.norm(y)
        bad = np.argwhere(e > 0.05 + 0.05 * np.abs(y))
        rows = sorted(set(int(b[1]) for b in bad))
        cols = sorted(set(int(b[3]) for b in bad))
        heads = sorted(set(int(b[2]) for b in bad))
        msg.append(f"{name} relL2={rl:.2e} nbad={len(bad)} rows[{rows[:3]}..{rows[-3:] if rows else ''}] "
                   f"heads{heads} cols[{cols[:4]}..{cols[-4:] if cols else ''}]")
    print(N, H, sigma, D, " | ".join(msg), flush=True)
