"""Multi-rank Ulysses parity check, launched by tests/test_multigpu.py as
    torchrun --nproc-per-node P tests/mp_ulysses_check.py --N .. --H .. --D ..
Each rank feeds its sequence shard (sliced from the same synth global tensors)
through the C ABI with P ranks; rank 0 gathers and checks:
  * P-way forward == P=1 forward, bitwise ("all matrices are the same");
  * out / lse / dq / dk / dv against the fp64 oracle (gates of tests/parity.py);
  * the all-to-all call law: 2 in the forward, 2 in the backward;
  * an invalid shape (head limit) fails identically on every rank
    before any collective (no hang).
Prints "MP_OK" on success of each case; --cases '<json list of {N,H,D,sigma,mode,det}>' runs
several cases in one process group (one launch per P in the test suite)."""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2405_15780_b200 as ua  # noqa: E402
import synth  # noqa: E402
from tests.parity import gate_grad, gate_lse, gate_out  # noqa: E402


def run_case(a, P, rank, local, dev):
    B, N, H, D = 1, a.N, a.H, a.D
    Nl = N // P
    q, k, v, do = synth.qkv(B, N, H, D, seed=77, sigma_qk=a.sigma, with_do=True)
    sl = slice(rank * Nl, (rank + 1) * Nl)
    qs, ks, vs, ds = (t[:, sl].contiguous().to(dev) for t in (q, k, v, do))

    ctx = ua.Context(P=P, rank=rank, device=local)
    ctx.set_a2a_mode(a.mode)
    assert ctx.a2a_mode() == a.mode
    ctx.set_deterministic(bool(a.det))
    # head limit: every rank must get the same error, before any collective
    try:
        ua.ulysses_attn_fwd(ctx, *(torch.zeros(1, 4, 1, D, dtype=torch.bfloat16, device=dev) for _ in range(3)))
        err = "none"
    except ua.HeadDivisibilityError:
        err = "head"
    errs = [None] * P
    dist.all_gather_object(errs, err)
    assert all(e == "head" for e in errs), errs

    c0, _ = ctx.comm_stats()
    r = ua.ulysses_attn_fwd(ctx, qs, ks, vs)
    c1, bytes_f = ctx.comm_stats()
    dq, dk, dv = ua.ulysses_attn_bwd(ctx, qs, ks, vs, r.out, r.lse, ds)
    c2, bytes_b = ctx.comm_stats()
    torch.cuda.synchronize()
    assert c1 - c0 == 2 and c2 - c1 == 2, (c0, c1, c2)
    exp_f = 4 * Nl * H * D * 2 * (P - 1) // P          # q,k,v in + o out, off-rank
    assert bytes_f == exp_f, (bytes_f, exp_f)
    # a second step reuses the (peer) buffers and flag counters: same bits
    r2 = ua.ulysses_attn_fwd(ctx, qs, ks, vs)
    dq2, dk2, dv2 = ua.ulysses_attn_bwd(ctx, qs, ks, vs, r2.out, r2.lse, ds)
    torch.cuda.synchronize()
    assert torch.equal(r2.out, r.out) and torch.equal(r2.lse, r.lse)
    assert torch.equal(dk2, dk) and torch.equal(dv2, dv)
    assert (dq2.float() - dq.float()).abs().max().item() <= 2e-2
    if a.det:
        assert torch.equal(dq2, dq)

    def gather(t):
        parts = [torch.empty_like(t) for _ in range(P)]
        dist.all_gather(parts, t.contiguous())
        return parts

    outs, dqs, dks, dvs, lses = (gather(t) for t in (r.out, dq, dk, dv, r.lse))
    if rank == 0:
        out_g = torch.cat(outs, 1).float().cpu().numpy()
        lse_g = torch.cat(lses, 1).cpu().numpy()            # [B][H][N]: rank j holds heads block j
        dq_g, dk_g, dv_g = (torch.cat(x, 1).float().cpu().numpy() for x in (dqs, dks, dvs))
        # P=1 on the same inputs, same device: bitwise forward equality
        c1ctx = ua.Context(P=1, device=local)
        c1ctx.set_deterministic(bool(a.det))
        r1 = ua.ulysses_attn_fwd(c1ctx, q.to(dev), k.to(dev), v.to(dev))
        g1 = ua.ulysses_attn_bwd(c1ctx, q.to(dev), k.to(dev), v.to(dev), r1.out, r1.lse, do.to(dev))
        torch.cuda.synchronize()
        assert np.array_equal(out_g, r1.out.float().cpu().numpy()), "P-way forward != P=1 forward"
        assert np.array_equal(lse_g, r1.lse.cpu().numpy()), "P-way lse != P=1 lse"
        for x, y in zip((dq_g, dk_g, dv_g), g1):
            if a.det:   # same per-head arithmetic in a fixed order: bitwise
                assert np.array_equal(x, y.float().cpu().numpy()), "P-way grads != P=1 grads (deterministic)"
            else:
                assert np.abs(x - y.float().cpu().numpy()).max() <= 2e-2
        f64 = [synth.to_f64(t) for t in (q, k, v, do)]
        oracle.set_num_threads(len(os.sched_getaffinity(0)))   # torchrun sets OMP_NUM_THREADS=1 per rank
        ref, ref_lse, absv = oracle.attn_fwd(*f64[:3], with_abs=True)
        gate_out(out_g, ref, gate_a=a.sigma == 1.0, absv=absv)
        gate_lse(lse_g, ref_lse)
        rdq, rdk, rdv, _, _, gabs = oracle.attn_bwd(*f64, with_abs=True)
        for x, y, gb in zip((dq_g, dk_g, dv_g), (rdq, rdk, rdv), gabs):
            gate_grad(x, y, gate_a=a.sigma == 1.0, gabs=gb)
        c1ctx.close()
        print("MP_OK", vars(a), flush=True)
    ctx.close()
    dist.barrier()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=4096)
    ap.add_argument("--H", type=int, default=8)
    ap.add_argument("--D", type=int, default=64)
    ap.add_argument("--sigma", type=float, default=1.0)
    ap.add_argument("--mode", default="nccl", choices=["nccl", "peer"])
    ap.add_argument("--det", type=int, default=0, help="deterministic backward: P-way grads == P=1 grads bitwise")
    ap.add_argument("--cases", default="", help="JSON list of per-case overrides of the options above")
    a = ap.parse_args()
    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    base = {k: v for k, v in vars(a).items() if k != "cases"}
    for c in (json.loads(a.cases) if a.cases else [{}]):
        run_case(argparse.Namespace(**{**base, **c}), P, rank, local, dev)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
