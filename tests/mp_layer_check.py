"""Multi-rank attention-layer check (projections + Ulysses attention + the SP
weight-gradient all-reduce), launched by tests/test_multigpu.py as
    torchrun --nproc-per-node P tests/mp_layer_check.py --N .. --H .. --D ..
Every rank feeds its sequence shard of x, dy; checks: y, dx shards and the
all-reduced dW against the fp64 oracle (relL2 <= 1e-2), dW identical on every
rank, and the collective law: 2 calls forward, 3 backward (2 a2a + 1
all-reduce).  Prints "LAYER_OK" per case; --cases '<json list of {N,H,D}>' runs several cases
in one process group."""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2405_15780_b200 as ua  # noqa: E402
import synth  # noqa: E402
from oracle import layer as olayer  # noqa: E402
from tests.parity import rel_l2  # noqa: E402


def run_case(a, P, rank, local, dev):
    B, N, H, D = 1, a.N, a.H, a.D
    Nl = N // P
    x, dy, w_qkv, w_o = synth.layer_inputs(B, N, H, D, seed=300)
    sl = slice(rank * Nl, (rank + 1) * Nl)
    xs, dys = (t[:, sl].contiguous().to(dev) for t in (x, dy))
    wq, wo = w_qkv.to(dev), w_o.to(dev)
    ctx = ua.Context(P=P, rank=rank, device=local)
    c0, _ = ctx.comm_stats()
    y, saved = ua.layer_fwd(ctx, xs, wq, wo, H)
    c1, _ = ctx.comm_stats()
    dx, dwq, dwo = ua.layer_bwd(ctx, xs, wq, wo, saved, dys, H)
    c2, _ = ctx.comm_stats()
    torch.cuda.synchronize()
    assert (c1 - c0, c2 - c1) == (2, 3), (c0, c1, c2)

    def gather(t):
        parts = [torch.empty_like(t) for _ in range(P)]
        dist.all_gather(parts, t.contiguous())
        return parts

    ys, dxs, dwqs, dwos = gather(y), gather(dx), gather(dwq), gather(dwo)
    if rank == 0:
        assert all(torch.equal(dwqs[0], t) for t in dwqs) and all(torch.equal(dwos[0], t) for t in dwos)
        f64 = [synth.to_f64(t) for t in (x, w_qkv, w_o, dy)]
        import oracle
        oracle.set_num_threads(len(os.sched_getaffinity(0)))   # torchrun sets OMP_NUM_THREADS=1 per rank
        ry, _ = olayer.layer_fwd(f64[0], f64[1], f64[2], H)
        rdx, rdwq, rdwo = olayer.layer_bwd(*f64, H)
        got = {"y": torch.cat(ys, 1), "dx": torch.cat(dxs, 1), "dw_qkv": dwqs[0], "dw_o": dwos[0]}
        for name, ref in (("y", ry), ("dx", rdx), ("dw_qkv", rdwq), ("dw_o", rdwo)):
            r = rel_l2(got[name].float().cpu().numpy(), ref)
            assert r <= 1e-2, f"{name}: relL2 {r:.3e}"
        print("LAYER_OK", vars(a), flush=True)
    ctx.close()
    dist.barrier()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=1024)
    ap.add_argument("--H", type=int, default=4)
    ap.add_argument("--D", type=int, default=64)
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
