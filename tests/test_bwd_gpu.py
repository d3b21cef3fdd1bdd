"""GPU parity of the Ulysses backward at P=1 against the fp64 oracle, through
the C ABI (dq, dk, dv for the loss <out, dout>).  Inputs from synth only."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests.parity import gate_grad

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ua():
    import paper_2405_15780_b200 as m
    from paper_2405_15780_b200 import build
    build.build()
    return m


@pytest.fixture(scope="module")
def ctx(ua):
    c = ua.Context(P=1)
    yield c
    c.close()


@pytest.fixture(scope="module")
def dctx(ua):
    c = ua.Context(P=1)
    c.set_deterministic(True)
    assert c.deterministic()
    yield c
    c.close()


def run_fwd_bwd(ua, ctx, q, k, v, do):
    qc, kc, vc, dc = (t.cuda() for t in (q, k, v, do))
    r = ua.ulysses_attn_fwd(ctx, qc, kc, vc)
    dq, dk, dv = ua.ulysses_attn_bwd(ctx, qc, kc, vc, r.out, r.lse, dc)
    torch.cuda.synchronize()
    return tuple(t.float().cpu().numpy() for t in (dq, dk, dv))


def check(ua, ctx, B, N, H, D, sigma, seed):
    q, k, v, do = synth.qkv(B, N, H, D, seed=seed, sigma_qk=sigma, with_do=True)
    got = run_fwd_bwd(ua, ctx, q, k, v, do)
    dq, dk, dv, _, _, gabs = oracle.attn_bwd(*(synth.to_f64(t) for t in (q, k, v, do)), with_abs=True)
    stats = {}
    for name, g, ref, a in zip(("dq", "dk", "dv"), got, (dq, dk, dv), gabs):
        stats[name] = gate_grad(g, ref, gate_a=sigma == 1.0, gabs=a)
    return stats


@pytest.mark.parametrize("N,H,D,sigma", [
    (256, 4, 32, 1.0),      # c1
    (256, 4, 32, 2.0),
    (1, 2, 64, 1.0),        # one token: dV = dO, dQ = dK = 0
    (127, 2, 64, 1.0),
    (129, 2, 64, 2.0),
    (384, 2, 64, 1.0),
    (640, 2, 128, 1.0),
    (1000, 2, 128, 2.0),
    (4050, 2, 64, 1.0),     # P:263 seq 4050 (ragged tail)
    (2048, 2, 32, 2.0),
    (300, 2, 72, 1.0),      # D=72 (ViT-10B)
    (1000, 3, 72, 2.0),
    (129, 2, 72, 1.0),
    (1000, 2, 64, 4.0),     # sigma_qk = 4: row maxima move by >> 2^8, the lazy rescale fires on most tiles
    (2048, 2, 128, 4.0),
    (777, 2, 32, 4.0),
])
def test_bwd_parity_small(ua, ctx, N, H, D, sigma):
    check(ua, ctx, 1, N, H, D, sigma, seed=100 + N)


def test_bwd_batch2(ua, ctx):
    check(ua, ctx, 2, 384, 2, 64, 1.0, seed=5)


@pytest.mark.parametrize("sigma", [1.0, 2.0])
def test_bwd_parity_c2(ua, ctx, sigma):
    """c2: N=8192, H=16, D=64, full oracle backward on 4 of the 16 heads
    (heads are independent; the GPU runs all 16)."""
    B, N, H, D = 1, 8192, 16, 64
    q, k, v, do = synth.qkv(B, N, H, D, seed=synth.BASE_SEED, sigma_qk=sigma, with_do=True)
    got = run_fwd_bwd(ua, ctx, q, k, v, do)
    heads = [0, 5, 10, 15]
    sub = [synth.to_f64(t)[:, :, heads] for t in (q, k, v, do)]
    dq, dk, dv, _, _, gabs = oracle.attn_bwd(*sub, with_abs=True)
    for g, ref, a in zip(got, (dq, dk, dv), gabs):
        gate_grad(g[:, :, heads], ref, gate_a=sigma == 1.0, gabs=a)


@pytest.mark.parametrize("det", [False, True])
@pytest.mark.parametrize("N,H,D,heads", [(8192, 16, 32, [0, 15]), (8192, 8, 72, [3, 7])])
def test_bwd_more_items_than_sms(ua, ctx, dctx, N, H, D, heads, det):
    """D = 32 (1,024 work items) and D = 72 (512 items) on 148 SMs: every CTA of
    the persistent backward runs several items, so the cross-item hand-offs
    (K/V reload, TMEM accumulator reuse, DQ_LATE issue order) are exercised at
    these head dims too.  Oracle on a subset of the heads."""
    q, k, v, do = synth.qkv(1, N, H, D, seed=900 + D, with_do=True)
    got = run_fwd_bwd(ua, dctx if det else ctx, q, k, v, do)
    sub = [synth.to_f64(t)[:, :, heads] for t in (q, k, v, do)]
    dq, dk, dv, _, _, gabs = oracle.attn_bwd(*sub, with_abs=True)
    for g, ref, a in zip(got, (dq, dk, dv), gabs):
        gate_grad(g[:, :, heads], ref, gate_a=True, gabs=a)


def sample_rows(N, rng, extra=12):
    """Both ends, both sides of 128-row tile boundaries near the ends and the
    middle, the boundary of the persistent grid's first item wave (148 key
    tiles), and random rows."""
    fixed = [0, 1, 127, 128, 129, 255, 256, 148 * 128 - 1, 148 * 128, N // 2 - 1, N // 2, N - 129, N - 128, N - 2,
             N - 1]
    return np.unique(np.array([r for r in fixed if 0 <= r < N] + list(rng.integers(0, N, extra))))


_FULL_REF = {}   # (cfg, head) -> fp64 oracle rows: the c4 reference (minutes of CPU) serves both modes


@pytest.mark.slow
@pytest.mark.parametrize("cfg,head,det", [("c3", 9, False), ("c4", 17, False), ("c4", 17, True)])
def test_bwd_full_size_sampled_rows(ua, ctx, dctx, cfg, head, det):
    """Full-size backward at P = 1 (c3: N = 65,536, D = 128; c4: N = 188,416,
    D = 64; c4 also in the deterministic mode): exact fp64 dK, dV for sampled
    KEY rows of one head (oracle.attn_bwd_kv_rows, which recomputes every lse_i
    and Delta_i) and dQ for sampled query rows, element by element (Gate A +
    relL2 + elementwise)."""
    c = synth.CONFIGS[cfg]
    B, N, H, D = c["B"], c["N"], c["H"], c["D"]
    q, k, v, do = synth.qkv(B, N, H, D, seed=synth.BASE_SEED, with_do=True)
    dq, dk, dv = run_fwd_bwd(ua, dctx if det else ctx, q, k, v, do)
    for t in (dq, dk, dv):
        assert np.isfinite(t).all()
    rows = sample_rows(N, np.random.default_rng(17))
    if (cfg, head) not in _FULL_REF:
        qh, kh, vh, doh = (synth.to_f64(t[0, :, head]) for t in (q, k, v, do))
        dk_ref, dv_ref = oracle.attn_bwd_kv_rows(qh, kh, vh, doh, rows)
        bh = np.array([(0, 0)] * len(rows))
        dq_ref = oracle.attn_bwd_dq_rows(qh[rows], doh[rows], bh, kh[None, :, None, :], vh[None, :, None, :])
        _FULL_REF[(cfg, head)] = (dk_ref, dv_ref, dq_ref)
    dk_ref, dv_ref, dq_ref = _FULL_REF[(cfg, head)]
    gate_grad(dk[0, rows, head], dk_ref)
    gate_grad(dv[0, rows, head], dv_ref)
    gate_grad(dq[0, rows, head], dq_ref)


def test_bwd_invariants(ua, ctx):
    """Exact-math invariants on the GPU gradients (oracle-free): sum_j dK_j = 0,
    sum_j dV_j = sum_i dO_i, <Q,dQ> = <K,dK> per head; constant V -> dQ = dK = 0."""
    N, H, D = 2048, 4, 64
    q, k, v, do = synth.qkv(1, N, H, D, seed=9, with_do=True)
    dq, dk, dv = run_fwd_bwd(ua, ctx, q, k, v, do)
    qf, kf, dof = (synth.to_f64(t) for t in (q, k, do))
    scale_k = np.abs(dk).sum(axis=1)
    assert np.all(np.abs(dk.sum(axis=1)) <= 2e-2 * scale_k + 1e-3)
    assert np.all(np.abs(dv.sum(axis=1) - dof.sum(axis=1)) <= 1e-2 * np.abs(dv).sum(axis=1) + 1e-2)
    lhs = np.einsum("bnhd,bnhd->h", qf, dq)
    rhs = np.einsum("bnhd,bnhd->h", kf, dk)
    assert np.all(np.abs(lhs - rhs) <= 2e-2 * (np.abs(lhs) + np.abs(rhs)) + 1.0)
    vc = torch.broadcast_to(v[:, :1], v.shape).contiguous()
    dq0, dk0, _ = run_fwd_bwd(ua, ctx, q, k, vc, do)
    assert np.abs(dq0).max() < 2e-2 and np.abs(dk0).max() < 2e-2


def test_bwd_deterministic_dkdv(ua, ctx):
    """dK, dV are computed without atomics: bitwise reproducible."""
    q, k, v, do = synth.qkv(1, 1024, 2, 64, seed=13, with_do=True)
    a = run_fwd_bwd(ua, ctx, q, k, v, do)
    b = run_fwd_bwd(ua, ctx, q, k, v, do)
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


# ------------------------------------------------------------ deterministic mode

@pytest.mark.parametrize("B,N,H,D,sigma", [
    (1, 256, 4, 32, 1.0),      # c1
    (1, 2, 2, 64, 1.0),        # two tokens
    (1, 129, 2, 64, 2.0),      # ragged query and key tails
    (1, 1000, 2, 128, 2.0),
    (1, 4050, 2, 64, 1.0),
    (2, 384, 2, 64, 1.0),      # B > 1
    (1, 1000, 3, 72, 2.0),     # D = 72 (padded 80-wide tiles)
])
def test_bwd_deterministic_parity(ua, dctx, B, N, H, D, sigma):
    """Query-stationary dQ + dQ-less KV-stationary kernel against the fp64 oracle."""
    check(ua, dctx, B, N, H, D, sigma, seed=300 + N)


def test_bwd_deterministic_one_token(ua, dctx):
    """N = 1: dV = dO, dQ = dK = 0.  dQ is dS k with dS = dP - Delta, two
    fp32 sums of the same D products in different orders, so it is zero only up
    to fp32 rounding (the relative gate is undefined for an all-zero reference)."""
    q, k, v, do = synth.qkv(1, 1, 2, 64, seed=3, with_do=True)
    dq, dk, dv = run_fwd_bwd(ua, dctx, q, k, v, do)
    assert np.abs(dq).max() <= 1e-4 and np.abs(dk).max() <= 1e-4
    assert np.array_equal(dv, do.float().numpy())


@pytest.mark.parametrize("N,H,D", [(2048, 2, 64), (1000, 2, 128), (777, 2, 32)])
def test_bwd_deterministic_bitwise(ua, ctx, dctx, N, H, D):
    """Deterministic mode: dq, dk, dv bitwise equal run to run, and within
    bf16 rounding of the default mode's (which sums the same per-tile partials
    in another order: staggered query sweeps, concurrent dQ reduce-adds)."""
    q, k, v, do = synth.qkv(1, N, H, D, seed=21, with_do=True)
    a = run_fwd_bwd(ua, dctx, q, k, v, do)
    b = run_fwd_bwd(ua, dctx, q, k, v, do)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    ref = run_fwd_bwd(ua, ctx, q, k, v, do)
    for x, y in zip(a, ref):
        assert np.abs(x - y).max() <= 2 ** -7 * np.abs(y).max() + 1e-6


def test_bwd_deterministic_c2(ua, dctx):
    """c2 (N=8192, H=16, D=64) in deterministic mode: oracle on 4 of the 16 heads."""
    B, N, H, D = 1, 8192, 16, 64
    q, k, v, do = synth.qkv(B, N, H, D, seed=synth.BASE_SEED, with_do=True)
    got = run_fwd_bwd(ua, dctx, q, k, v, do)
    heads = [0, 7, 15]
    sub = [synth.to_f64(t)[:, :, heads] for t in (q, k, v, do)]
    dq, dk, dv, _, _, gabs = oracle.attn_bwd(*sub, with_abs=True)
    for g, ref, a in zip(got, (dq, dk, dv), gabs):
        gate_grad(g[:, :, heads], ref, gate_a=True, gabs=a)
