"""Single-GPU checks of the LSS sequence-parallel strategy (
PAPER.md P:72; R14) at P > 1, through the C ABI's LSS
rank-local entry points (include/ulysses_attn.h "LSS rank-local steps").

One GPU simulates P ranks: each rank's compute (its N/P queries of every head
over all N gathered keys; the backward's complete local dQ and PARTIAL dK, dV
over all keys) runs in the library's kernels, and the collectives between them
are performed by the test as plain copies / sums: the all-gather of K, V is a
concatenation in rank order, the reduce-scatter a sum over ranks in fp64
followed by each rank's row block.  Checked against oracle/lss.py per rank
(forward rows, per-rank fp32 partials) and after the reduction, and the
forward bitwise against the P = 1 run.  Inputs from synth."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import lss as olss
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


CASES = [
    # P, B, N, H, D, sigma
    (2, 1, 4096, 8, 64, 1.0),
    (4, 1, 4096, 2, 64, 1.0),      # P > H: no head limit
    (2, 1, 4050, 4, 64, 1.0),      # ragged segment N/P = 2025
    (2, 2, 2048, 4, 64, 1.0),      # B = 2
    (8, 1, 8192, 4, 64, 1.0),
    (2, 1, 2048, 3, 72, 2.0),      # D = 72
    (4, 1, 2048, 4, 128, 2.0),
    (4, 1, 2048, 2, 32, 4.0),      # sigma_qk = 4
]


@pytest.mark.parametrize("P,B,N,H,D,sigma", CASES)
def test_lss_sim(ua, ctx1, P, B, N, H, D, sigma):
    q, k, v, do = synth.qkv(B, N, H, D, seed=1100 + N + P, sigma_qk=sigma, with_do=True)
    Nl = N // P
    qc, kc, vc, dc = (t.cuda() for t in (q, k, v, do))
    sh = [[t[:, r * Nl:(r + 1) * Nl].contiguous() for r in range(P)] for t in (qc, kc, vc, dc)]
    # the all-gather: every rank's [B][Nl][H][D] shard re-laid [Nl][B][H][D], concatenated in rank order
    kf = torch.cat([x.permute(1, 0, 2, 3) for x in sh[1]]).contiguous()
    vf = torch.cat([x.permute(1, 0, 2, 3) for x in sh[2]]).contiguous()
    fw = [ua.lss_rank_fwd(sh[0][r], kf, vf, P) for r in range(P)]
    bw = [ua.lss_rank_bwd(sh[0][r], kf, vf, fw[r][0], fw[r][1], sh[3][r], P) for r in range(P)]
    torch.cuda.synchronize()

    f64 = [synth.to_f64(t) for t in (q, k, v, do)]
    o_ref, l_ref = olss.sp_fwd(*f64[:3], P)
    # error scales of the elementwise gates (R7): the dense oracle's magnitude sums; for a rank's
    # partial dK, dV (a sum over a subset of the queries) the full sum bounds the partial's
    _, _, absv = oracle.attn_fwd(*f64[:3], with_abs=True)
    _, _, _, _, _, gabs = oracle.attn_bwd(*f64, with_abs=True)
    # forward: per rank against the oracle, and bitwise against the P = 1 run
    out = torch.cat([f[0] for f in fw], dim=1)
    lse = torch.cat([f[1] for f in fw], dim=2)
    gate_out(out.float().cpu().numpy(), np.concatenate(o_ref, axis=1), gate_a=sigma == 1.0, absv=absv)
    gate_lse(lse.cpu().numpy(), np.concatenate(l_ref, axis=2))
    r1 = ua.lss_attn_fwd(ctx1, qc, kc, vc)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), r1.out.view(torch.int16))
    assert torch.equal(lse, r1.lse)

    # backward: each rank's fp32 partial dK, dV against the oracle's partial (S:181-183 restricted to its queries)
    dqs_ref, dks_ref, dvs_ref = olss.sp_bwd(*f64, P)
    for r in (0, P - 1):
        _, pk, pv = olss.sp_bwd_partial(f64[0][:, r * Nl:(r + 1) * Nl], f64[3][:, r * Nl:(r + 1) * Nl], o_ref[r],
                                        l_ref[r], f64[1], f64[2])
        gate_grad(bw[r][1].permute(1, 0, 2, 3).cpu().numpy(), pk, gate_a=False, gabs=gabs[1])
        gate_grad(bw[r][2].permute(1, 0, 2, 3).cpu().numpy(), pv, gate_a=False, gabs=gabs[2])
    # the reduce-scatter: sum of the partials over ranks, rank r's key rows
    dk_sum = sum(b[1].double() for b in bw).permute(1, 0, 2, 3).cpu().numpy()
    dv_sum = sum(b[2].double() for b in bw).permute(1, 0, 2, 3).cpu().numpy()
    gate_grad(dk_sum, np.concatenate(dks_ref, axis=1), gate_a=sigma == 1.0, gabs=gabs[1])
    gate_grad(dv_sum, np.concatenate(dvs_ref, axis=1), gate_a=sigma == 1.0, gabs=gabs[2])
    dq = torch.cat([b[0] for b in bw], dim=1).float().cpu().numpy()
    gate_grad(dq, np.concatenate(dqs_ref, axis=1), gate_a=sigma == 1.0, gabs=gabs[0])
