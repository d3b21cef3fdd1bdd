"""Probe: Delta = rowsum(dO * O) as computed in the P=1 backward workspace (debug aid)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2405_15780_b200 as ua  # noqa: E402
import synth  # noqa: E402

ctx = ua.Context(P=1)
for N, H, sigma, D in [(1000, 3, 2.0, 72), (1000, 3, 2.0, 64), (1000, 3, 1.0, 72)]:
    q, k, v, do = synth.qkv(1, N, H, D, seed=100 + N, sigma_qk=sigma, with_do=True)
    qc, kc, vc, dc = (t.cuda() for t in (q, k, v, do))
    r = ua.ulysses_attn_fwd(ctx, qc, kc, vc)
    g = ua.ulysses_attn_bwd(ctx, qc, kc, vc, r.out, r.lse, dc)
    torch.cuda.synchronize()
    ws = ctx._ws["buf"]
    delta = ws[: N * H * 4].view(torch.float32).view(N, H).cpu().numpy()
    ref = (dc.float() * r.out.float()).sum(-1)[0].cpu().numpy()     # [N][H]
    e = np.abs(delta - ref)
    print(N, H, sigma, D, "delta max err", e.max(), "ref max", np.abs(ref).max(), "argmax", np.unravel_index(e.argmax(), e.shape), flush=True)
