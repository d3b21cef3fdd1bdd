"""GPU parity of the projection GEMM (ua_gemm_bf16: TMA + tcgen05 + TMEM,
SURVEY §8(f)-3) against the plain definition C = sum_s op(A_s) op(B_s)
computed by numpy in fp64 on the same bf16 inputs (a library matmul as the
oracle's one step).  Inputs from synth.

Tolerance: the kernel multiplies bf16 values exactly and accumulates in fp32
(error <= K u32 sum |a||b|, u32 = 2^-24); a bf16 output adds one rounding
(<= 2^-9 |C|).  Gate: |err| <= 2^-14 (|A| |B|) + 2^-8 |ref| (bf16 out) or
2^-14 (|A| |B|) (fp32 out), elementwise."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ua():
    import paper_2405_15780_b200 as m
    from paper_2405_15780_b200 import build
    build.build()
    return m


def draw(rows, cols, seed, name):
    return synth.normal_bf16(1, rows, 1, cols, seed, name).reshape(rows, cols)


def ref_and_scale(As, Bs, a_mn, b_mn):
    ref, mag = 0.0, 0.0
    for A, B in zip(As, Bs):
        a = synth.to_f64(A)
        b = synth.to_f64(B)
        a = a.T if a_mn else a          # op(A) [M][K]
        b = b if b_mn else b.T          # op(B) [K][N]
        ref = ref + a @ b
        mag = mag + np.abs(a) @ np.abs(b)
    return ref, mag


def check(got, ref, mag, out_f32):
    err = np.abs(got.float().cpu().numpy().astype(np.float64) - ref)
    bound = 2.0 ** -14 * mag + (0.0 if out_f32 else 2.0 ** -8 * np.abs(ref))
    assert (err <= bound + 1e-30).all(), f"max excess {(err - bound).max():.3e}"


@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, True)])
@pytest.mark.parametrize("M,N,K,nseg,out_f32", [
    (128, 256, 64, 1, False),        # one tile, one k-block
    (296, 256, 200, 1, False),       # ragged M and K (TMA zero fill, masked rows)
    (1000, 384, 136, 3, True),       # N = 384 -> 128-wide tiles, three K segments
    (256, 512, 1024, 2, False),
    (72, 144, 520, 1, True),         # E = 144 (H = 2, D = 72): ragged everything
])
def test_gemm_parity(ua, M, N, K, nseg, out_f32, a_mn, b_mn):
    As = [draw(K, M, 10 + s, "x") if a_mn else draw(M, K, 10 + s, "x") for s in range(nseg)]
    Bs = [draw(K, N, 20 + s, "dy") if b_mn else draw(N, K, 20 + s, "dy") for s in range(nseg)]
    got = ua.gemm([t.cuda() for t in As], [t.cuda() for t in Bs], a_mn, b_mn, out_f32=out_f32)
    torch.cuda.synchronize()
    assert got.shape == (M, N)
    ref, mag = ref_and_scale(As, Bs, a_mn, b_mn)
    check(got, ref, mag, out_f32)


@pytest.mark.slow
def test_gemm_c4_projection_shapes(ua):
    """The c4 layer's shapes (P = 1: M = 188,416 tokens, E = 2,048): q = x Wq^T,
    dx = sum of three segments g_i W_i, and dW = g^T x (K = 188,416), checked on
    sampled output rows."""
    M, E = 188416, 2048
    x = draw(M, E, 1, "x").cuda()
    w = [draw(E, E, 2 + i, "w_qkv").cuda() for i in range(3)]
    g = [draw(M, E, 5 + i, "dy").cuda() for i in range(3)]
    rows_np = np.array([0, 1, 127, 128, 4095, M // 2, M - 129, M - 1])
    rows = torch.from_numpy(rows_np).cuda()
    wf = [synth.to_f64(t.cpu()) for t in w]
    # y = x W^T
    y = ua.gemm([x], [w[0]], False, False)
    xr = synth.to_f64(x[rows].cpu())
    check(y[rows], xr @ wf[0].T, np.abs(xr) @ np.abs(wf[0]).T, False)
    # dx = sum_i g_i W_i
    dx = ua.gemm(g, w, False, True)
    gr = [synth.to_f64(t[rows].cpu()) for t in g]
    check(dx[rows], sum(a @ b for a, b in zip(gr, wf)), sum(np.abs(a) @ np.abs(b) for a, b in zip(gr, wf)), False)
    # dW = g^T x (fp32), rows of dW = columns of g
    dw = ua.gemm([g[0]], [x], True, True, out_f32=True)
    cols = torch.tensor([0, 1, 1000, E - 1]).cuda()
    gc = synth.to_f64(g[0][:, cols].cpu())        # [M][4]
    xf = synth.to_f64(x.cpu())
    check(dw[cols], gc.T @ xf, np.abs(gc).T @ np.abs(xf), True)
    torch.cuda.synchronize()
