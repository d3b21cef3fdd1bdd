"""Pins for the fp64 oracle (CPU only).  Each check is independent of the
oracle's own code: a library implementation (torch fp64 SDPA + autograd),
central finite differences, closed forms / worked examples from SPEC.md, and
invariants that hold for the exact mathematics.  A dropped term, wrong sign,
wrong index or transposed operand in oracle.c fails at least one of these.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from oracle import layer, lss, ulysses

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def rnd(shape, seed, sigma=1.0):
    return np.random.default_rng(seed).standard_normal(shape) * sigma


def torch_sdpa(q, k, v):
    """Library routine: torch's fp64 CPU scaled_dot_product_attention on
    [B][N][H][D] arrays (transposed to its [B][H][N][D] convention)."""
    tq, tk, tv = (torch.from_numpy(np.ascontiguousarray(x)).permute(0, 2, 1, 3) for x in (q, k, v))
    o = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv)
    return o.permute(0, 2, 1, 3).numpy()


# ---------------------------------------------------------------- forward pins
@pytest.mark.parametrize("B,N,H,D", [(1, 7, 1, 4), (2, 33, 3, 8), (1, 130, 2, 32), (1, 257, 2, 64)])
def test_fwd_matches_torch_sdpa_fp64(B, N, H, D):
    q, k, v = rnd((B, N, H, D), 1), rnd((B, N, H, D), 2), rnd((B, N, H, D), 3)
    out, lse = oracle.attn_fwd(q, k, v)
    assert np.abs(out - torch_sdpa(q, k, v)).max() < 1e-12
    # lse against torch.logsumexp of the materialised scaled score matrix
    s = torch.einsum("bihd,bjhd->bhij", torch.from_numpy(q), torch.from_numpy(k)) / math.sqrt(D)
    assert np.abs(lse - torch.logsumexp(s, dim=-1).numpy()).max() < 1e-12


def test_fwd_abs_helper():
    """absv = sum_j P_ij |v_jd|: equals out for V >= 0 and out(|V|) always."""
    q, k, v = rnd((1, 40, 2, 8), 23), rnd((1, 40, 2, 8), 24), rnd((1, 40, 2, 8), 25)
    out, lse, absv = oracle.attn_fwd(q, k, v, with_abs=True)
    out2, lse2 = oracle.attn_fwd(q, k, v)
    assert np.array_equal(out, out2) and np.array_equal(lse, lse2)
    o_abs, _ = oracle.attn_fwd(q, k, np.abs(v))
    assert np.abs(absv - o_abs).max() < 1e-14
    assert np.all(absv >= np.abs(out) - 1e-14)


def test_fwd_cross_attention_shapes():
    """Nq != Nk (used by the segment tests) against torch SDPA."""
    q, k, v = rnd((1, 9, 2, 8), 4), rnd((1, 21, 2, 8), 5), rnd((1, 21, 2, 8), 6)
    out, _ = oracle.attn_fwd(q, k, v)
    assert np.abs(out - torch_sdpa(q, k, v)).max() < 1e-12


def test_golden_single_token():
    g = GOLD["mha_forward_single_token"]
    q, k, v = (np.array(g[n]).reshape(1, 1, 1, 4) for n in ("q", "k", "v"))
    out, lse = oracle.attn_fwd(q, k, v)
    assert np.array_equal(out.ravel(), np.array(g["out"]))
    assert abs(lse.item() - g["lse"]) < 1e-15


def test_golden_softmax_rows():
    """S:50-51.  Scores [c, c+ln2] are realised with D=1: s_j = q k_j / 1,
    so q = 1 and k_j = the row entries.  With V = identity columns the output
    equals the probability row."""
    for ex in GOLD["row_softmax"]:
        row = np.array(ex["row"])
        n = len(row)
        q = np.ones((1, 1, 1, 1))
        k = row.reshape(1, n, 1, 1)
        for c in range(n):                      # one-hot V picks P_{0c}
            v = np.zeros((1, n, 1, 1))
            v[0, c, 0, 0] = 1.0
            out, lse = oracle.attn_fwd(q, k, v)
            assert abs(out.item() - ex["probs"][c]) < 1e-15
        assert abs(lse.item() - (row.max() + np.log(np.exp(row - row.max()).sum()))) < 1e-14
        if n == 2:                              # lse = c + ln 3 exactly
            assert abs(lse.item() - (row[0] + math.log(3.0))) < 1e-14


def test_identical_keys_uniform():
    """identical K rows -> uniform weights, out = mean(V), lse = s + ln N."""
    N, D = 37, 16
    q, v = rnd((1, N, 1, D), 7), rnd((1, N, 1, D), 8)
    k = np.broadcast_to(rnd((1, 1, 1, D), 9), (1, N, 1, D)).copy()
    out, lse = oracle.attn_fwd(q, k, v)
    assert np.abs(out - v.mean(axis=1, keepdims=True)).max() < 1e-13
    s = (q[0, :, 0] @ k[0, 0, 0]) / math.sqrt(D)
    assert np.abs(lse[0, 0] - (s + math.log(N))).max() < 1e-12


def test_constant_v_and_rows_sum_to_one():
    N, D = 50, 8
    q, k = rnd((1, N, 2, D), 10, 3.0), rnd((1, N, 2, D), 11, 3.0)
    c = rnd((1, 1, 2, D), 12)
    out, _ = oracle.attn_fwd(q, k, np.broadcast_to(c, (1, N, 2, D)).copy())
    assert np.abs(out - c).max() < 1e-13
    out1, _ = oracle.attn_fwd(q, k, np.ones((1, N, 2, D)))
    assert np.abs(out1 - 1).max() < 1e-13


def test_permutation_equivariance_and_shift_invariance():
    N, H, D = 41, 2, 8
    q, k, v = rnd((1, N, H, D), 13), rnd((1, N, H, D), 14), rnd((1, N, H, D), 15)
    out, lse = oracle.attn_fwd(q, k, v)
    perm = np.random.default_rng(0).permutation(N)
    o2, l2 = oracle.attn_fwd(q[:, perm], k, v)                   # permute queries
    assert np.abs(o2 - out[:, perm]).max() < 1e-14
    o3, _ = oracle.attn_fwd(q, k[:, perm], v[:, perm])           # permute keys jointly
    assert np.abs(o3 - out).max() < 1e-13
    u = rnd((1, 1, H, D), 16)
    o4, l4 = oracle.attn_fwd(q, k + u, v)                         # S:72 shift invariance
    assert np.abs(o4 - out).max() < 1e-12
    shift = np.einsum("bnhd,bhd->bhn", q, u[:, 0]) / math.sqrt(D)
    assert np.abs(l4 - (lse + shift)).max() < 1e-12


def test_lse_bounds_and_convex_hull():
    N, H, D = 64, 2, 16
    q, k, v = rnd((1, N, H, D), 17, 2.0), rnd((1, N, H, D), 18, 2.0), rnd((1, N, H, D), 19)
    out, lse = oracle.attn_fwd(q, k, v)
    s = np.einsum("bihd,bjhd->bhij", q, k) / math.sqrt(D)
    assert np.all(lse >= s.max(-1) - 1e-12) and np.all(lse <= s.max(-1) + math.log(N) + 1e-12)
    vmin, vmax = v.min(axis=1, keepdims=True), v.max(axis=1, keepdims=True)
    assert np.all(out >= vmin - 1e-12) and np.all(out <= vmax + 1e-12)


def test_fwd_rows_matches_dense():
    B, N, H, D = 2, 90, 3, 16
    q, k, v = rnd((B, N, H, D), 20), rnd((B, N, H, D), 21), rnd((B, N, H, D), 22)
    out, lse = oracle.attn_fwd(q, k, v)
    bh = np.array([[0, 0], [1, 2], [1, 0], [0, 1]])
    idx = np.array([0, 89, 45, 7])
    qrows = q[bh[:, 0], idx, bh[:, 1]]
    o_r, l_r = oracle.attn_fwd_rows(qrows, bh, k, v)
    assert np.abs(o_r - out[bh[:, 0], idx, bh[:, 1]]).max() == 0.0
    assert np.abs(l_r - lse[bh[:, 0], bh[:, 1], idx]).max() == 0.0


# --------------------------------------------------------------- backward pins
def _loss(q, k, v, w):
    out, _ = oracle.attn_fwd(q, k, v)
    return float((out * w).sum())


@pytest.mark.parametrize("N,H,D", [(5, 1, 4), (12, 2, 3), (16, 1, 8)])
def test_bwd_central_finite_differences(N, H, D):
    """central differences, h=1e-6, fp64.  dout = w is the
    gradient of L = <out, w>."""
    q, k, v, w = (rnd((1, N, H, D), s, 1.5) for s in (30, 31, 32, 33))
    dq, dk, dv, _, _ = oracle.attn_bwd(q, k, v, w)
    h = 1e-6
    for x, g in ((q, dq), (k, dk), (v, dv)):
        num = np.zeros_like(x)
        it = np.nditer(x, flags=["multi_index"])
        for _ in it:
            i = it.multi_index
            old = x[i]
            x[i] = old + h
            fp = _loss(q, k, v, w)
            x[i] = old - h
            fm = _loss(q, k, v, w)
            x[i] = old
            num[i] = (fp - fm) / (2 * h)
        rel = np.abs(num - g).max() / max(1.0, np.abs(g).max())
        assert rel < 1e-7, rel


@pytest.mark.parametrize("B,N,H,D", [(1, 65, 2, 16), (2, 31, 1, 32)])
def test_bwd_matches_torch_autograd_fp64(B, N, H, D):
    q, k, v, do = (rnd((B, N, H, D), s) for s in (40, 41, 42, 43))
    dq, dk, dv, out, lse = oracle.attn_bwd(q, k, v, do)
    tq, tk, tv = (torch.from_numpy(x.copy()).permute(0, 2, 1, 3).requires_grad_() for x in (q, k, v))
    o = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv)
    o.backward(torch.from_numpy(do).permute(0, 2, 1, 3))
    for mine, ref in ((dq, tq.grad), (dk, tk.grad), (dv, tv.grad)):
        assert np.abs(mine - ref.permute(0, 2, 1, 3).numpy()).max() < 1e-12
    assert np.abs(out - o.detach().permute(0, 2, 1, 3).numpy()).max() < 1e-12


def test_bwd_closed_forms():
    g = GOLD["mha_backward_single_token"]
    q = rnd((1, 1, 1, 4), 50)
    k = rnd((1, 1, 1, 4), 51)
    v = rnd((1, 1, 1, 4), 52)
    do = np.array(g["dout"]).reshape(1, 1, 1, 4)
    dq, dk, dv, _, _ = oracle.attn_bwd(q, k, v, do)
    assert np.array_equal(dv.ravel(), np.array(g["dv"]))
    assert np.abs(dq).max() < 1e-15 and np.abs(dk).max() < 1e-15
    # dOut = 0 -> zero grads
    q, k, v = (rnd((1, 20, 2, 8), s) for s in (53, 54, 55))
    z = oracle.attn_bwd(q, k, v, np.zeros_like(q))
    assert all(np.abs(t).max() == 0.0 for t in z[:3])
    # constant V -> dQ = dK = 0 ; identical K rows -> dQ = 0
    c = np.broadcast_to(rnd((1, 1, 2, 8), 56), v.shape).copy()
    dq, dk, _, _, _ = oracle.attn_bwd(q, k, c, rnd(q.shape, 57))
    assert np.abs(dq).max() < 1e-13 and np.abs(dk).max() < 1e-13
    kc = np.broadcast_to(rnd((1, 1, 2, 8), 58), k.shape).copy()
    dq, _, _, _, _ = oracle.attn_bwd(q, kc, v, rnd(q.shape, 59))
    assert np.abs(dq).max() < 1e-13


def test_bwd_invariants():
    """sum_j dK_j = 0 ; sum_j dV_j = sum_i dO_i ; <Q,dQ> = <K,dK> per head;
    linearity in dO."""
    N, H, D = 70, 3, 16
    q, k, v, do = (rnd((1, N, H, D), s, 1.5) for s in (60, 61, 62, 63))
    dq, dk, dv, _, _ = oracle.attn_bwd(q, k, v, do)
    assert np.abs(dk.sum(axis=1)).max() < 1e-12
    assert np.abs(dv.sum(axis=1) - do.sum(axis=1)).max() < 1e-12
    assert np.abs(np.einsum("bnhd,bnhd->h", q, dq) - np.einsum("bnhd,bnhd->h", k, dk)).max() < 1e-10
    do2 = rnd(do.shape, 64)
    a = oracle.attn_bwd(q, k, v, do)
    b = oracle.attn_bwd(q, k, v, do2)
    c = oracle.attn_bwd(q, k, v, 2.0 * do - 3.0 * do2)
    for i in range(3):
        assert np.abs(c[i] - (2.0 * a[i] - 3.0 * b[i])).max() < 1e-12


# ------------------------------------------------------------- Ulysses pins
def test_all_to_all_golden_p2():
    g = GOLD["all_to_all_p2"]
    assert ulysses.all_to_all(g["send"]) == g["recv"]


def test_all_to_all_identity_and_involution():
    x = [[np.full(3, 10 * i + j) for j in range(1)] for i in range(1)]
    assert ulysses.all_to_all(x)[0][0] is x[0][0]          # P=1 identity
    P = 4
    sends = [[rnd(5, 100 * i + j) for j in range(P)] for i in range(P)]
    back = ulysses.all_to_all(ulysses.all_to_all(sends))     # S:126 involution
    assert all(np.array_equal(back[i][j], sends[i][j]) for i in range(P) for j in range(P))


@pytest.mark.parametrize("P", [1, 2, 4])
def test_seq_head_round_trip(P):
    x = rnd((2, 16, 4, 8), 70)
    shards = ulysses.shard_seq(x, P)
    heads = ulysses.seq_to_head(shards, P)
    assert heads[0].shape == (2, 16, 4 // P, 8)
    for j in range(P):   # rank j holds all tokens of head block j
        assert np.array_equal(heads[j], x[:, :, j * (4 // P):(j + 1) * (4 // P)])
    back = ulysses.head_to_seq(heads, P)
    assert all(np.array_equal(back[r], shards[r]) for r in range(P))


@pytest.mark.parametrize("P", [1, 2, 4])
def test_ulysses_equals_dense(P):
    """S:247 (S=16,H=4,d_h=8,P=4) and P:414 ("all matrices are the same")."""
    N, H, D = 16, 4, 8
    q, k, v, do = (rnd((1, N, H, D), s) for s in (80, 81, 82, 83))
    out, lse = oracle.attn_fwd(q, k, v)
    shards = [ulysses.shard_seq(x, P) for x in (q, k, v, do)]
    o_sh, lse_sh = ulysses.ulysses_fwd(shards[0], shards[1], shards[2], P)
    assert np.abs(ulysses.gather_seq(o_sh) - out).max() < 1e-14
    assert np.abs(np.concatenate(lse_sh, axis=1) - lse).max() < 1e-14
    dq, dk, dv, _, _ = oracle.attn_bwd(q, k, v, do)
    g = ulysses.ulysses_bwd(*shards, P)
    for mine, ref in zip(g, (dq, dk, dv)):
        assert np.abs(ulysses.gather_seq(mine) - ref).max() < 1e-14


def test_head_limit_errors():
    g = GOLD["head_limit"]
    with pytest.raises(ulysses.HeadDivisibilityError):
        ulysses.check(g["N"], g["H"], g["P"])
    with pytest.raises(ulysses.HeadDivisibilityError):
        ulysses.check(12, 6, 4)
    with pytest.raises(ulysses.SeqDivisibilityError):
        ulysses.check(10, 4, 4)
    ulysses.check(16, 4, 4)


# ------------------------------------------------------------------ LSS pins
@pytest.mark.parametrize("bounds", [[0, 64], [0, 1, 64], [0, 16, 32, 48, 64], [0, 5, 40, 63, 64]])
def test_lss_chunked_equals_full(bounds):
    q, k, v = (rnd((1, 64, 2, 16), s, 2.0) for s in (90, 91, 92))
    out, lse = oracle.attn_fwd(q, k, v)
    o2, l2 = lss.chunked_fwd(q, k, v, bounds)
    assert np.abs(o2 - out).max() < 1e-13
    assert np.abs(l2 - lse).max() < 1e-13


def test_lss_merge_weights_are_segment_mass():
    """exp(lse_s - lse) = softmax mass of segment s (sums to 1 over s)."""
    q, k, v = (rnd((1, 30, 1, 8), s) for s in (93, 94, 95))
    parts = [lss.segment_fwd(q, k, v, a, b) for a, b in ((0, 10), (10, 30))]
    _, lse = lss.merge(parts)
    mass = sum(np.exp(l - lse) for _, l in parts)
    assert np.abs(mass - 1).max() < 1e-14


@pytest.mark.parametrize("P,B,N,H,D", [(1, 1, 24, 2, 8), (2, 1, 24, 2, 8), (3, 2, 27, 1, 4), (4, 1, 32, 3, 16),
                                       (6, 1, 24, 2, 8)])
def test_lss_sp_equals_dense(P, B, N, H, D):
    """LSS sequence parallelism: per-rank forward over gathered keys and
    the reduce-scattered partial dK, dV reproduce the dense fp64 oracle (the C
    implementation, a different code path) -- including P > H."""
    q, k, v, do = (rnd((B, N, H, D), s, 1.5) for s in (110, 111, 112, 113))
    out, lse = oracle.attn_fwd(q, k, v)
    dq, dk, dv, _, _ = oracle.attn_bwd(q, k, v, do)
    outs, lses = lss.sp_fwd(q, k, v, P)
    assert np.abs(np.concatenate(outs, 1) - out).max() < 1e-12
    assert np.abs(np.concatenate(lses, 2) - lse).max() < 1e-12
    dqs, dks, dvs = lss.sp_bwd(q, k, v, do, P)
    for got, ref in ((dqs, dq), (dks, dk), (dvs, dv)):
        assert np.abs(np.concatenate(got, 1) - ref).max() < 1e-11


def test_lss_sp_partials_are_partial():
    """A single rank's dK partial is NOT the full dK (P > 1) -- the reduce is
    needed -- and the partials of the ranks sum to it."""
    P, N, H, D = 2, 16, 1, 4
    q, k, v, do = (rnd((1, N, H, D), s) for s in (120, 121, 122, 123))
    _, dk, _, out, lse = oracle.attn_bwd(q, k, v, do)
    Nl = N // P
    parts = [lss.sp_bwd_partial(q[:, r * Nl:(r + 1) * Nl], do[:, r * Nl:(r + 1) * Nl], out[:, r * Nl:(r + 1) * Nl],
                                lse[:, :, r * Nl:(r + 1) * Nl], k, v)[1] for r in range(P)]
    assert np.abs(parts[0] - dk).max() > 1e-3
    assert np.abs(parts[0] + parts[1] - dk).max() < 1e-12


def test_bwd_abs_helpers():
    """gabs = (scale (|dS|+E)|K|, scale (|dS|+E)^T|Q|, P^T|dO|): the third equals dV
    computed with |dO| (dV is linear in dO); all bound |grad| from above; the
    first two against materialised numpy on a tiny case."""
    N, H, D = 23, 2, 8
    q, k, v, do = (rnd((1, N, H, D), s) for s in (100, 101, 102, 103))
    dq, dk, dv, out, lse, (aq, ak, av) = oracle.attn_bwd(q, k, v, do, with_abs=True)
    _, _, dv_abs, _, _ = oracle.attn_bwd(q, k, v, np.abs(do))
    assert np.abs(av - dv_abs).max() < 1e-13
    for g, a in ((dq, aq), (dk, ak), (dv, av)):
        assert np.all(a >= np.abs(g) - 1e-13)
    sc = 1 / math.sqrt(D)
    for h in range(H):
        S = q[0, :, h] @ k[0, :, h].T * sc
        P = np.exp(S - S.max(1, keepdims=True))
        P /= P.sum(1, keepdims=True)
        dP = do[0, :, h] @ v[0, :, h].T
        O = P @ v[0, :, h]
        dS = P * (dP - (do[0, :, h] * O).sum(1, keepdims=True))
        E = P * np.abs(do[0, :, h] * O).sum(1, keepdims=True)
        assert np.abs(aq[0, :, h] - sc * (np.abs(dS) + E) @ np.abs(k[0, :, h])).max() < 1e-12
        assert np.abs(ak[0, :, h] - sc * (np.abs(dS) + E).T @ np.abs(q[0, :, h])).max() < 1e-12


def test_bwd_dq_rows_matches_dense():
    B, N, H, D = 2, 70, 3, 16
    q, k, v, do = (rnd((B, N, H, D), s) for s in (110, 111, 112, 113))
    dq, _, _, _, _ = oracle.attn_bwd(q, k, v, do)
    bh = np.array([[0, 0], [1, 2], [1, 1], [0, 2]])
    idx = np.array([0, 69, 33, 5])
    got = oracle.attn_bwd_dq_rows(q[bh[:, 0], idx, bh[:, 1]], do[bh[:, 0], idx, bh[:, 1]], bh, k, v)
    assert np.abs(got - dq[bh[:, 0], idx, bh[:, 1]]).max() < 1e-13


def test_bwd_kv_rows_matches_dense():
    """Sampled key rows (first, last, interior) of two heads against the dense
    backward, which torch autograd and finite differences pin above."""
    B, N, H, D = 1, 75, 3, 16
    q, k, v, do = (rnd((B, N, H, D), s, 1.5) for s in (120, 121, 122, 123))
    _, dk, dv, _, _ = oracle.attn_bwd(q, k, v, do)
    keys = np.array([0, 74, 37, 8, 8])
    for h in (0, 2):
        gk, gv = oracle.attn_bwd_kv_rows(q[0, :, h], k[0, :, h], v[0, :, h], do[0, :, h], keys)
        assert np.abs(gk - dk[0, keys, h]).max() < 1e-13
        assert np.abs(gv - dv[0, keys, h]).max() < 1e-13


def test_bwd_kv_rows_against_torch_autograd():
    """Independent of oracle.c's dense backward: torch fp64 autograd of
    <softmax(QK^T/sqrt(D)) V, dO> for one head."""
    N, D = 40, 8
    q, k, v, do = (rnd((N, D), s) for s in (130, 131, 132, 133))
    tq, tk, tv = (torch.tensor(x, requires_grad=True) for x in (q, k, v))
    p = torch.softmax(tq @ tk.T / math.sqrt(D), dim=-1)
    ((p @ tv) * torch.from_numpy(do)).sum().backward()
    keys = np.arange(N)
    gk, gv = oracle.attn_bwd_kv_rows(q, k, v, do, keys)
    assert np.abs(gk - tk.grad.numpy()).max() < 1e-12
    assert np.abs(gv - tv.grad.numpy()).max() < 1e-12


def test_delta_is_probability_weighted_dp():
    """Delta_i = dO_i . o_i = sum_j P_ij (dO_i . v_j) (rows of P sum to 1), with
    o from torch SDPA and P from a materialised torch softmax; dO = 0 -> 0."""
    B, N, H, D = 1, 30, 2, 8
    q, k, v, do = (rnd((B, N, H, D), s) for s in (140, 141, 142, 143))
    o = torch_sdpa(q, k, v)
    got = oracle.delta(do, o)
    s = torch.einsum("bihd,bjhd->bhij", torch.from_numpy(q), torch.from_numpy(k)) / math.sqrt(D)
    p = torch.softmax(s, dim=-1).numpy()
    dp = np.einsum("bihd,bjhd->bhij", do, v)
    ref = np.einsum("bhij,bhij->bih", p, dp)
    assert got.shape == (B, N, H)
    assert np.abs(got - ref).max() < 1e-12
    assert np.array_equal(oracle.delta(np.zeros_like(do), o), np.zeros((B, N, H)))


# ------------------------------------------------------------------ layer pins
@pytest.mark.parametrize("B,N,H,D", [(1, 12, 2, 4), (2, 7, 3, 2)])
def test_layer_matches_torch_autograd(B, N, H, D):
    """oracle.layer (numpy matmuls + oracle.c attention) against torch fp64
    autograd through matmuls and scaled_dot_product_attention (library routines)."""
    import torch
    E = H * D
    x, dy = rnd((B, N, E), 130), rnd((B, N, E), 131)
    w_qkv, w_o = rnd((3 * E, E), 132, 0.5), rnd((E, E), 133, 0.5)
    y, _ = layer.layer_fwd(x, w_qkv, w_o, H)
    dx, dwq, dwo = layer.layer_bwd(x, w_qkv, w_o, dy, H)
    tx, twq, two = (torch.tensor(t, dtype=torch.float64, requires_grad=True) for t in (x, w_qkv, w_o))
    qkv = [(tx @ twq[i * E:(i + 1) * E].T).reshape(B, N, H, D).transpose(1, 2) for i in range(3)]
    o = torch.nn.functional.scaled_dot_product_attention(*qkv).transpose(1, 2).reshape(B, N, E)
    ty = o @ two.T
    ty.backward(torch.tensor(dy, dtype=torch.float64))
    assert np.abs(y - ty.detach().numpy()).max() < 1e-12
    for a, b in ((dx, tx.grad), (dwq, twq.grad), (dwo, two.grad)):
        assert np.abs(a - b.numpy()).max() < 1e-11


def test_layer_weight_grads_are_sums_over_tokens():
    """The SP all-reduce sums per-shard weight gradients: the gradient
    of a token-sharded layer's weights equals the sum over shards' own."""
    B, N, H, D, P = 1, 12, 2, 4, 3
    E = H * D
    x, dy = rnd((B, N, E), 140), rnd((B, N, E), 141)
    w_qkv, w_o = rnd((3 * E, E), 142, 0.5), rnd((E, E), 143, 0.5)
    _, dwq, dwo = layer.layer_bwd(x, w_qkv, w_o, dy, H)
    _, (q, k, v, o, _) = layer.layer_fwd(x, w_qkv, w_o, H)
    Nl = N // P
    parts = [np.einsum("bnj,bni->ji", dy[:, r * Nl:(r + 1) * Nl], o[:, r * Nl:(r + 1) * Nl]) for r in range(P)]
    assert np.abs(sum(parts) - dwo).max() < 1e-12
