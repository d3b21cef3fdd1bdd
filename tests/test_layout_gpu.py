"""Single-GPU checks of the Ulysses steps that only run at P > 1 (SURVEY §8(a)
rows A1, A5/A6, B1, B6, and the P-way composition), through the C ABI's
rank-local entry points (include/ulysses_attn.h "rank-local steps").

One GPU simulates P ranks: every rank's buffers live on cuda:0, the library's
own kernels do the packing, attention and unpacking, and the all-to-all between
them is performed by the test as plain byte copies with SPEC.md S:122's
semantics (output[j] on rank i == input[i] on rank j) -- the only step these
tests do not exercise is the NCCL transport itself (tests/test_multigpu.py
covers it whenever >= 2 GPUs are present).

Bars (R13): the layout round trip is BIT-EXACT against
oracle/ulysses.py (compared as raw bf16 bits); Delta is within fp32 rounding of
oracle.delta; the P-way forward is bitwise equal to the P = 1 forward; the
deterministic P-way backward is bitwise equal to the P = 1 deterministic
backward; both are within the oracle gates at sizes the oracle finishes.
Inputs from synth only."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import ulysses as oul
from tests.parity import gate_grad, gate_lse, gate_out

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ua():
    import paper_2405_15780_b200 as m
    from paper_2405_15780_b200 import build
    build.build()
    return m


@pytest.fixture(scope="module")
def ctx1(ua):
    c = ua.Context(P=1)
    yield c
    c.close()


@pytest.fixture(scope="module")
def dctx1(ua):
    c = ua.Context(P=1)
    c.set_deterministic(True)
    yield c
    c.close()


def bits(t):
    """Raw bf16 bits as an int16 numpy array (bitwise comparisons)."""
    return t.contiguous().view(torch.int16).cpu().numpy()


def shards_of(x, P):
    Nl = x.shape[1] // P
    return [x[:, r * Nl:(r + 1) * Nl].contiguous() for r in range(P)]


# ---- the all-to-all as byte copies ---------------------------------------------
def a2a_seq_to_head(sends, P):
    """sends[i] = rank i's send buffer [P][Nl][B][Hl][D] (chunk j -> rank j).
    Rank j receives chunk j of every rank in source order: [P][Nl][B][Hl][D] ==
    the head-shard tensor [N][B][Hl][D]."""
    _, Nl, B, Hl, D = sends[0].shape
    return [torch.cat([sends[i][j] for i in range(P)], dim=0) for j in range(P)]


def a2a_head_to_seq(heads, P):
    """heads[j] = rank j's [N][B][Hl][D] tensor, whose token block i goes to rank i.
    Rank i receives [P][Nl][B][Hl][D], chunk s from rank s."""
    N, B, Hl, D = heads[0].shape
    Nl = N // P
    return [torch.stack([heads[j].view(P, Nl, B, Hl, D)[i] for j in range(P)]) for i in range(P)]


def a2a_delta(sends, P):
    """Delta send buffers [P][Nl][B][Hl] -> rank j's [N][B][Hl]."""
    return [torch.cat([sends[i][j] for i in range(P)], dim=0) for j in range(P)]


LAYOUT_CASES = [
    # P, B, N, H, D
    (2, 1, 256, 4, 32),        # c1 shape at P = 2
    (4, 1, 256, 4, 32),        # c1 at P = H = 4
    (8, 1, 4096, 8, 64),
    (2, 1, 4050, 4, 64),       # ragged per-rank length N/P = 2025 (P:263's 4050)
    (4, 2, 2048, 8, 72),       # D = 72 (rows of 9 vectors), B = 2
    (2, 2, 1000, 4, 128),      # B = 2, D = 128
    (8, 1, 65536, 16, 128),    # c3 at P = 8 (full size)
]


@pytest.mark.parametrize("P,B,N,H,D", LAYOUT_CASES)
def test_pack_a2a_unpack_bit_exact(ua, P, B, N, H, D):
    """A1 (pack), the exchange, A6 (unpack): recv == oracle seq_to_head bitwise;
    head_to_seq(seq_to_head(x)) == x bitwise; B1's Delta vs oracle.delta."""
    q, k, v, do = synth.qkv(B, N, H, D, seed=500 + N + P, with_do=True)
    xs = [q, k, v]
    gsh = [shards_of(t.cuda(), P) for t in xs]                    # [tensor][rank]
    do_sh, o_sh = shards_of(do.cuda(), P), shards_of(v.flip(1).contiguous().cuda(), P)  # O stand-in: any bf16 [B][Nl][H][D]
    sends, dsends = [], []
    for r in range(P):
        s, dl = ua.pack_seq_to_head([gsh[w][r] for w in range(3)], P, dout=do_sh[r], out=o_sh[r])
        sends.append(s)
        dsends.append(dl)
    torch.cuda.synchronize()
    recv = [a2a_seq_to_head([sends[i][w] for i in range(P)], P) for w in range(3)]  # [tensor][rank j]
    for w, x in enumerate(xs):
        ref = oul.seq_to_head(oul.shard_seq(bits(x), P), P)                        # [B][N][Hl][D] per rank
        for j in range(P):
            got = bits(recv[w][j]).transpose(1, 0, 2, 3)
            assert np.array_equal(got, ref[j]), f"tensor {w} rank {j}: a2a #1 layout differs from the oracle"
    # Delta (fp32 in sequence space, shipped with the exchange) against the oracle
    rd = a2a_delta(dsends, P)
    dref = oracle.delta(synth.to_f64(do), synth.to_f64(v.flip(1)))                # [B][N][H]
    mag = np.abs(synth.to_f64(do) * synth.to_f64(v.flip(1))).sum(-1)
    Hl = H // P
    for j in range(P):
        got = rd[j].cpu().numpy().transpose(1, 0, 2)                               # [B][N][Hl]
        ref = dref[:, :, j * Hl:(j + 1) * Hl]
        assert np.all(np.abs(got - ref) <= 2.0 ** -22 * D * mag[:, :, j * Hl:(j + 1) * Hl] + 1e-30)
    # return trip: every rank's head shard back to sequence shards (A5 exchange + A6 unpack)
    for w, x in enumerate(xs):
        back_recv = a2a_head_to_seq(recv[w], P)
        back = [ua.unpack_head_to_seq([back_recv[i]], P)[0] for i in range(P)]
        torch.cuda.synchronize()
        heads_ref = oul.seq_to_head(oul.shard_seq(bits(x), P), P)
        seq_ref = oul.head_to_seq(heads_ref, P)
        for i in range(P):
            assert np.array_equal(bits(back[i]), seq_ref[i])                        # == oracle head_to_seq
            assert np.array_equal(bits(back[i]), bits(gsh[w][i]))                   # round trip is the identity
    # unpack of several tensors per launch (B6: dq, dk, dv in one call)
    back_recv = [a2a_head_to_seq(recv[w], P) for w in range(3)]
    for i in range(P):
        outs = ua.unpack_head_to_seq([back_recv[w][i] for w in range(3)], P)
        for w in range(3):
            assert torch.equal(outs[w].view(torch.int16), gsh[w][i].view(torch.int16))


@pytest.mark.parametrize("P,B,N,H,D", [c for c in LAYOUT_CASES if c[0] <= 8])
def test_push_equals_pack_plus_exchange(ua, P, B, N, H, D):
    """The peer transport's fused pack + all-to-all (every rank's chunks stored
    straight into each destination's receive buffer): receive buffers equal the
    pack -> exchange result bitwise, Delta included (same arithmetic)."""
    q, k, v, do = synth.qkv(B, N, H, D, seed=600 + N + P, with_do=True)
    sh = [shards_of(t.cuda(), P) for t in (q, k, v, do)]
    o_sh = shards_of(k.flip(1).contiguous().cuda(), P)
    Hl = H // P
    tens = B * N * Hl * D * 2
    bufs = [torch.zeros(4 * tens + B * N * Hl * 4, dtype=torch.uint8, device="cuda") for _ in range(P)]
    sends, dsends = [], []
    for r in range(P):
        ua.push_seq_to_head([sh[w][r] for w in range(4)], bufs, P, r, dout=sh[3][r], out=o_sh[r])
        s, dl = ua.pack_seq_to_head([sh[w][r] for w in range(4)], P, dout=sh[3][r], out=o_sh[r])
        sends.append(s)
        dsends.append(dl)
    torch.cuda.synchronize()
    recv = [a2a_seq_to_head([sends[i][w] for i in range(P)], P) for w in range(4)]
    rd = a2a_delta(dsends, P)
    for j in range(P):
        for w in range(4):
            got = bufs[j][w * tens:(w + 1) * tens].view(torch.int16)
            assert torch.equal(got, recv[w][j].reshape(-1).view(torch.int16)), f"rank {j} tensor {w}"
        got_d = bufs[j][4 * tens:].view(torch.float32)
        assert torch.equal(got_d, rd[j].reshape(-1)), f"rank {j} Delta"


# ---- the whole Ulysses path on P simulated ranks ---------------------------------------
def sim_fwd(ua, q, k, v, P, transport):
    """pack -> a2a #1 -> head attention -> a2a #2 -> unpack on P simulated ranks.
    Returns (per-rank out [B][Nl][H][D], per-rank lse [B][Hl][N], head shards)."""
    sh = [shards_of(t.cuda(), P) for t in (q, k, v)]
    sends = [ua.pack_seq_to_head([sh[w][r] for w in range(3)], P)[0] for r in range(P)]
    recv = [a2a_seq_to_head([sends[i][w] for i in range(P)], P) for w in range(3)]
    lses = []
    if transport == "peer":            # A3 + A5 fused: rows stored straight into the token owners
        outs = [torch.empty_like(sh[0][r]) for r in range(P)]
        for j in range(P):
            _, lse = ua.head_attn_fwd(recv[0][j], recv[1][j], recv[2][j], P, j, o_owner=outs)
            lses.append(lse)
    else:
        o_heads = []
        for j in range(P):
            o, lse = ua.head_attn_fwd(recv[0][j], recv[1][j], recv[2][j], P, j)
            o_heads.append(o)
            lses.append(lse)
        back = a2a_head_to_seq(o_heads, P)
        outs = [ua.unpack_head_to_seq([back[i]], P)[0] for i in range(P)]
    torch.cuda.synchronize()
    return outs, lses, recv


def sim_bwd(ua, q, k, v, do, outs, lses, P, transport, deterministic):
    """pack + Delta -> a2a #3 -> head backward -> a2a #4 -> unpack."""
    sh = [shards_of(t.cuda(), P) for t in (q, k, v, do)]
    packed = [ua.pack_seq_to_head([sh[w][r] for w in range(4)], P, dout=sh[3][r], out=outs[r]) for r in range(P)]
    recv = [a2a_seq_to_head([packed[i][0][w] for i in range(P)], P) for w in range(4)]
    rdelta = a2a_delta([packed[i][1] for i in range(P)], P)
    if transport == "peer":            # B3 + B5 fused
        grads = [[torch.empty_like(sh[0][r]) for r in range(P)] for _ in range(3)]
        owners = grads[0] + grads[1] + grads[2]
        for j in range(P):
            ua.head_attn_bwd(recv[0][j], recv[1][j], recv[2][j], recv[3][j], lses[j], rdelta[j], P, j, owners=owners,
                             deterministic=deterministic)
        torch.cuda.synchronize()
        return grads
    g_heads = [ua.head_attn_bwd(recv[0][j], recv[1][j], recv[2][j], recv[3][j], lses[j], rdelta[j], P, j,
                                deterministic=deterministic) for j in range(P)]
    back = [a2a_head_to_seq([g_heads[j][w] for j in range(P)], P) for w in range(3)]
    grads = [[None] * P for _ in range(3)]
    for i in range(P):
        dq, dk, dv = ua.unpack_head_to_seq([back[0][i], back[1][i], back[2][i]], P)
        grads[0][i], grads[1][i], grads[2][i] = dq, dk, dv
    torch.cuda.synchronize()
    return grads


def gather(shards):
    return torch.cat(shards, dim=1)


SIM_CASES = [
    # P, B, N, H, D, sigma
    (2, 1, 256, 4, 32, 1.0),       # c1 at P = 2
    (4, 1, 256, 4, 32, 2.0),       # c1 at P = 4
    (2, 1, 4050, 4, 64, 1.0),      # ragged N/P = 2025
    (8, 1, 4096, 16, 64, 1.0),
    (4, 2, 1024, 8, 128, 2.0),     # B = 2
    (2, 1, 2048, 4, 72, 1.0),      # D = 72
    (8, 1, 2048, 8, 32, 4.0),      # sigma_qk = 4: the lazy rescale fires on most tiles
]


@pytest.mark.parametrize("transport", ["nccl", "peer"])
@pytest.mark.parametrize("P,B,N,H,D,sigma", SIM_CASES)
def test_sim_ulysses_fwd(ua, ctx1, P, B, N, H, D, sigma, transport):
    """P-way forward == P = 1 forward bitwise ("all matrices are the same";
    DESIGN R13) and within the oracle gates."""
    q, k, v = synth.qkv(B, N, H, D, seed=700 + N + P, sigma_qk=sigma)
    outs, lses, _ = sim_fwd(ua, q, k, v, P, transport)
    r1 = ua.ulysses_attn_fwd(ctx1, q.cuda(), k.cuda(), v.cuda())
    torch.cuda.synchronize()
    assert torch.equal(gather(outs).view(torch.int16), r1.out.view(torch.int16))
    assert torch.equal(torch.cat(lses, dim=1), r1.lse)
    ref, ref_lse, absv = oracle.attn_fwd(synth.to_f64(q), synth.to_f64(k), synth.to_f64(v), with_abs=True)
    gate_out(gather(outs).float().cpu().numpy(), ref, gate_a=sigma == 1.0, absv=absv)
    gate_lse(torch.cat(lses, dim=1).cpu().numpy(), ref_lse)


@pytest.mark.parametrize("transport", ["nccl", "peer"])
@pytest.mark.parametrize("P,B,N,H,D,sigma", SIM_CASES)
def test_sim_ulysses_bwd(ua, ctx1, dctx1, P, B, N, H, D, sigma, transport):
    """P-way backward within the oracle gates (default mode) and, in
    deterministic mode, bitwise equal to the P = 1 deterministic backward."""
    q, k, v, do = synth.qkv(B, N, H, D, seed=800 + N + P, sigma_qk=sigma, with_do=True)
    outs, lses, _ = sim_fwd(ua, q, k, v, P, transport)
    dq, dk, dv, _, _, gabs = oracle.attn_bwd(*(synth.to_f64(t) for t in (q, k, v, do)), with_abs=True)
    g = sim_bwd(ua, q, k, v, do, outs, lses, P, transport, deterministic=False)
    for got, ref, a in zip(g, (dq, dk, dv), gabs):
        gate_grad(gather(got).float().cpu().numpy(), ref, gate_a=sigma == 1.0, gabs=a)
    gd = sim_bwd(ua, q, k, v, do, outs, lses, P, transport, deterministic=True)
    qc, kc, vc, dc = (t.cuda() for t in (q, k, v, do))
    r1 = ua.ulysses_attn_fwd(dctx1, qc, kc, vc)
    ref1 = ua.ulysses_attn_bwd(dctx1, qc, kc, vc, r1.out, r1.lse, dc)
    torch.cuda.synchronize()
    for got, ref in zip(gd, ref1):
        assert torch.equal(gather(got).view(torch.int16), ref.view(torch.int16))


@pytest.mark.slow
def test_sim_ulysses_c3_p8_full_size(ua, ctx1, dctx1):
    """c3 (N = 65,536, H = 16, D = 128) on 8 simulated ranks at full size: the
    P-way forward (both transports) bitwise equal to the P = 1 forward; the
    deterministic P-way backward bitwise equal to the P = 1 deterministic one;
    the default backward within bf16 rounding of it."""
    cfg = synth.CONFIGS["c3"]
    B, N, H, D, P = cfg["B"], cfg["N"], cfg["H"], cfg["D"], 8
    q, k, v, do = synth.qkv(B, N, H, D, seed=synth.BASE_SEED, with_do=True)
    qc, kc, vc, dc = (t.cuda() for t in (q, k, v, do))
    r1 = ua.ulysses_attn_fwd(dctx1, qc, kc, vc)
    ref = ua.ulysses_attn_bwd(dctx1, qc, kc, vc, r1.out, r1.lse, dc)
    torch.cuda.synchronize()
    for transport in ("nccl", "peer"):
        outs, lses, _ = sim_fwd(ua, q, k, v, P, transport)
        assert torch.equal(gather(outs).view(torch.int16), r1.out.view(torch.int16)), transport
        assert torch.equal(torch.cat(lses, dim=1), r1.lse), transport
    gd = sim_bwd(ua, q, k, v, do, outs, lses, P, "nccl", deterministic=True)
    for got, r in zip(gd, ref):
        assert torch.equal(gather(got).view(torch.int16), r.view(torch.int16))
    g = sim_bwd(ua, q, k, v, do, outs, lses, P, "peer", deterministic=False)
    for got, r in zip(g, ref):
        x, y = gather(got).float(), r.float()
        assert ((x - y).abs() <= 2 ** -7 * y.abs() + 2 ** -7 * y.abs().max()).all()


@pytest.mark.slow
def test_layout_c4_p8_bit_exact(ua):
    """c4 (N = 188,416, H = 32, D = 64) at P = 8: pack -> exchange -> unpack of
    one full-size tensor, bitwise against oracle/ulysses.py."""
    cfg = synth.CONFIGS["c4"]
    B, N, H, D, P = cfg["B"], cfg["N"], cfg["H"], cfg["D"], 8
    x = synth.normal_bf16(B, N, H, D, synth.BASE_SEED, "q")
    xb = bits(x)
    sh = shards_of(x.cuda(), P)
    sends = [ua.pack_seq_to_head([sh[r]], P)[0][0] for r in range(P)]
    recv = a2a_seq_to_head(sends, P)
    ref = oul.seq_to_head(oul.shard_seq(xb, P), P)
    for j in range(P):
        assert np.array_equal(bits(recv[j]).transpose(1, 0, 2, 3), ref[j])
    back = a2a_head_to_seq(recv, P)
    for i in range(P):
        assert torch.equal(ua.unpack_head_to_seq([back[i]], P)[0].view(torch.int16), sh[i].view(torch.int16))
