"""GPU parity of the Ulysses forward at P=1 (and LSS segments) against the fp64
oracle, through the C ABI.  Inputs come from synth (never from the CUDA path)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests.parity import gate_lse, gate_out

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


def run_fwd(ua, ctx, q, k, v):
    r = ua.ulysses_attn_fwd(ctx, q.cuda(), k.cuda(), v.cuda())
    torch.cuda.synchronize()
    return r.out.float().cpu().numpy(), r.lse.cpu().numpy()


@pytest.mark.parametrize("N,H,D,sigma", [
    (256, 4, 32, 1.0),      # c1
    (256, 4, 32, 2.0),
    (1, 2, 64, 1.0),        # degenerate: one token
    (127, 2, 64, 1.0),      # ragged, less than one tile
    (129, 2, 64, 2.0),      # one tile + 1
    (300, 3, 64, 1.0),
    (640, 2, 128, 1.0),
    (1000, 2, 128, 2.0),    # ragged, D=128
    (4050, 2, 64, 1.0),     # P:263 seq 4050
    (2048, 2, 32, 2.0),
    (300, 2, 72, 1.0),      # D=72 (ViT-10B): padded 80-wide MMA tiles, SW32 atoms
    (1000, 3, 72, 2.0),
    (129, 2, 72, 1.0),
    (1000, 2, 64, 4.0),     # sigma_qk = 4: row maxima move by >> 2^8, the lazy rescale fires on most tiles
    (2048, 2, 128, 4.0),
    (777, 2, 32, 4.0),
    (300, 2, 72, 4.0),
])
def test_fwd_parity_small(ua, ctx, N, H, D, sigma):
    q, k, v = synth.qkv(1, N, H, D, seed=7 + N, sigma_qk=sigma)
    out, lse = run_fwd(ua, ctx, q, k, v)
    ref, ref_lse, absv = oracle.attn_fwd(synth.to_f64(q), synth.to_f64(k), synth.to_f64(v), with_abs=True)
    gate_out(out, ref, gate_a=sigma == 1.0, absv=absv)
    gate_lse(lse, ref_lse)


def test_fwd_batch2(ua, ctx):
    q, k, v = synth.qkv(2, 384, 2, 64, seed=11)
    out, lse = run_fwd(ua, ctx, q, k, v)
    ref, ref_lse = oracle.attn_fwd(synth.to_f64(q), synth.to_f64(k), synth.to_f64(v))
    gate_out(out, ref)
    gate_lse(lse, ref_lse)


@pytest.mark.parametrize("sigma", [1.0, 2.0])
def test_fwd_parity_c2(ua, ctx, sigma):
    """c2: N=8192, H=16, D=64 — full oracle on every head."""
    q, k, v = synth.qkv(1, 8192, 16, 64, seed=synth.BASE_SEED, sigma_qk=sigma)
    out, lse = run_fwd(ua, ctx, q, k, v)
    ref, ref_lse, absv = oracle.attn_fwd(synth.to_f64(q), synth.to_f64(k), synth.to_f64(v), with_abs=True)
    gate_out(out, ref, gate_a=sigma == 1.0, absv=absv)
    gate_lse(lse, ref_lse)


def test_fwd_invariants_and_determinism(ua, ctx):
    N, H, D = 1536, 4, 64
    q, k, v = synth.qkv(1, N, H, D, seed=3)
    out1, lse1 = run_fwd(ua, ctx, q, k, v)
    out2, lse2 = run_fwd(ua, ctx, q, k, v)
    assert np.array_equal(out1, out2) and np.array_equal(lse1, lse2)        # bitwise deterministic
    ones = torch.ones_like(v)
    o1, _ = run_fwd(ua, ctx, q, k, ones)                                       # rows of P sum to 1
    assert np.abs(o1 - 1).max() <= 2 ** -8
    perm = torch.randperm(N, generator=torch.Generator().manual_seed(0))
    o_p, l_p = run_fwd(ua, ctx, q[:, perm].contiguous(), k, v)               # query permutation equivariance
    assert np.array_equal(o_p, out1[:, perm.numpy()])


@pytest.mark.parametrize("N,H,D,seg", [(1024, 2, 64, 256), (1000, 2, 128, 384), (4050, 2, 64, 1024)])
def test_lss_segments_merge(ua, N, H, D, seg):
    q, k, v = synth.qkv(1, N, H, D, seed=21, sigma_qk=2.0)
    out, lse = ua.lss_chunked_fwd(q.cuda(), k.cuda(), v.cuda(), seg)
    torch.cuda.synchronize()
    ref, ref_lse, absv = oracle.attn_fwd(synth.to_f64(q), synth.to_f64(k), synth.to_f64(v), with_abs=True)
    gate_out(out.float().cpu().numpy(), ref, gate_a=False, absv=absv)
    gate_lse(lse.cpu().numpy(), ref_lse)
    # a single segment equals the oracle's segment (P:166 partial attention)
    o_s, l_s = ua.attn_fwd_segment(q.cuda(), k.cuda(), v.cuda(), seg, min(2 * seg, N))
    torch.cuda.synchronize()
    kf, vf = synth.to_f64(k), synth.to_f64(v)
    ro, rl, ra = oracle.attn_fwd(synth.to_f64(q), kf[:, seg:min(2 * seg, N)], vf[:, seg:min(2 * seg, N)], with_abs=True)
    gate_out(np.transpose(o_s.cpu().numpy(), (0, 2, 1, 3)), ro, gate_a=False, absv=ra)
    gate_lse(l_s.cpu().numpy(), rl)


@pytest.mark.slow
def test_fwd_c4_sampled_rows(ua, ctx):
    """c4 at P=1 (N=188,416, H=32, D=64): exact oracle on sampled rows of every
    head, including both ends and tile boundaries."""
    B, N, H, D = 1, 188416, 32, 64
    q, k, v = synth.qkv(B, N, H, D, seed=synth.BASE_SEED)
    out, lse = run_fwd(ua, ctx, q, k, v)
    rows = np.unique(np.array([0, 1, 127, 128, 255, 256, N // 2, N - 129, N - 128, N - 2, N - 1,
                               *np.random.default_rng(0).integers(0, N, 21)]))
    heads = np.arange(H)
    bh = np.array([(0, h) for h in heads for _ in rows])
    idx = np.tile(rows, len(heads))
    qf = synth.to_f64(q)
    o_r, l_r = oracle.attn_fwd_rows(qf[0, idx, bh[:, 1]], bh, synth.to_f64(k), synth.to_f64(v))
    gate_out(out[0, idx, bh[:, 1]], o_r)
    gate_lse(lse[0, bh[:, 1], idx], l_r)
    assert np.isfinite(out).all()


@pytest.mark.parametrize("D", [32, 64, 72, 128])
def test_fwd_lazy_rescale_ramp(ua, ctx, D):
    """Keys whose norms grow along the sequence make every query's running max
    rise tile after tile, so the lazy O / l rescale (threshold 2^8) fires often
    in both query tiles of a CTA; the result must still be the exact softmax."""
    N, H = 1536, 2
    q, k, v = synth.qkv(1, N, H, D, seed=31, sigma_qk=1.0)
    ramp = torch.linspace(0.2, 3.0, N).view(1, N, 1, 1)
    k = (k.float() * ramp).to(torch.bfloat16)          # deterministic transform of synth inputs
    out, lse = run_fwd(ua, ctx, q, k, v)
    ref, ref_lse, absv = oracle.attn_fwd(synth.to_f64(q), synth.to_f64(k), synth.to_f64(v), with_abs=True)
    gate_out(out, ref, gate_a=False, absv=absv)
    gate_lse(lse, ref_lse)
