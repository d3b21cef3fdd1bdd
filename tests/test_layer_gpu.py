"""GPU parity of the attention layer (projections + Ulysses attention, P=1)
against the fp64 oracle (oracle/layer.py), through the C ABI.  Tolerance
(R16): relative L2 <= 1e-2 per output -- the GPU rounds q, k, v, o,
do (and, inside the attention, P and dS) to bf16 once each (2^-9 relative),
the oracle rounds nothing."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import layer as olayer
from tests.parity import rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ua():
    import paper_2405_15780_b200 as m
    from paper_2405_15780_b200 import build
    build.build()
    return m


@pytest.mark.parametrize("B,N,H,D", [(1, 512, 4, 64), (2, 300, 2, 72), (1, 1000, 2, 128), (1, 256, 8, 32)])
def test_layer_parity(ua, B, N, H, D):
    ctx = ua.Context(P=1)
    x, dy, w_qkv, w_o = synth.layer_inputs(B, N, H, D, seed=200 + N)
    xc, dyc, wqc, woc = (t.cuda() for t in (x, dy, w_qkv, w_o))
    y, saved = ua.layer_fwd(ctx, xc, wqc, woc, H)
    dx, dwq, dwo = ua.layer_bwd(ctx, xc, wqc, woc, saved, dyc, H)
    torch.cuda.synchronize()
    c0, _ = ctx.comm_stats()
    assert c0 == 0                                      # P = 1: no collectives
    f64 = [synth.to_f64(t) for t in (x, w_qkv, w_o, dy)]
    ry, _ = olayer.layer_fwd(f64[0], f64[1], f64[2], H)
    rdx, rdwq, rdwo = olayer.layer_bwd(*f64, H)
    for name, got, ref in (("y", y, ry), ("dx", dx, rdx), ("dw_qkv", dwq, rdwq), ("dw_o", dwo, rdwo)):
        r = rel_l2(got.float().cpu().numpy(), ref)
        assert r <= 1e-2, f"{name}: relL2 {r:.3e}"
    ctx.close()


def test_layer_repeatable(ua):
    """Forward bitwise repeatable; saved state is all the backward needs."""
    ctx = ua.Context(P=1)
    x, dy, w_qkv, w_o = (t.cuda() for t in synth.layer_inputs(1, 384, 2, 64, seed=9))
    y1, s1 = ua.layer_fwd(ctx, x, w_qkv, w_o, 2)
    y2, s2 = ua.layer_fwd(ctx, x, w_qkv, w_o, 2)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2) and torch.equal(s1, s2)
    ctx.close()
