#!/usr/bin/env python3
"""Benchmark of the Ulysses sequence-parallel exact-attention hot path on B200.

One step = the whole hot path of SURVEY.md §8(a) on one batch: the Ulysses
forward (pack -> a2a -> attention -> a2a -> unpack) and backward (pack + Delta
-> a2a -> attention backward -> dQ finalize -> a2a -> unpack) of one attention
layer at BASELINE.json's headline workload c4: N = 188,416 tokens (the paper's
188K full-attention climate run), H = 32, D = 64, batch 1, bf16, with
the sequence split over the N GPUs (P = --gpus).  The work is fixed as GPUs
are added (strong scaling).

    python bench.py [--gpus N --steps K --warmup W]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)
    python bench.py --impl reference                        (fp64 CPU oracle arm)

Rank 0 prints one JSON line.  value = aggregate attention TFLOP/s (fwd 4*N^2*H*D
+ bwd 10*N^2*H*D per step, FlashAttention accounting, no causal halving) over
the max-over-ranks device time; tokens/s and % of the measured bf16 peak ride
along.  Inputs are resident in HBM for `value`; `e2e` repeats the measurement
through the public API with pinned-host inputs copied in and results copied out
every step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "attention TFLOPS & tokens/s at 188K tokens, 1/2/4/8 B200 (% of BF16 peak)"
# The paper's own numbers for this path: context, not a target
# (another machine, another metric: no attention TFLOP/s is printed in its text).
PAPER_CONTEXT = {
    "hardware": "AMD MI250X GCDs on Frontier (64 GB HBM2e, ~191.5 TF dense bf16 per GCD), RCCL",
    "result": "94 % batch weak-scaling efficiency (real ERA5; 96 % synthetic) from 16 to 2,048 GCDs, "
              "ViT-Base Multi-Ch-ViT at 188,416 tokens with DeepSpeed-Ulysses + FlashAttention-2, local batch 4",
    "cite": "PAPER.md P:425 (section 6.1)",
}
UNIT = "TFLOP/s"
NVLINK_GBS = 900.0   # NVLink 5 per direction per GPU (B200_PROFILING.md / SURVEY §8(e))
WORKLOAD = dict(name="c4", B=1, N=188416, H=32, D=64)
# BASELINE.json configs by (N, H, D) (c1 is the oracle-sized parity case)
CONFIG_NAMES = {(256, 4, 32): "c1", (8192, 16, 64): "c2", (65536, 16, 128): "c3", (188416, 32, 64): "c4",
                (1048576, 32, 128): "c5"}


def flops_per_step(B, N, H, D):
    fwd = 4.0 * B * N * N * H * D
    return fwd, 2.5 * fwd


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(bf16_burst=d["bf16_tflops"], bf16_sustained=d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                    hbm_gbs=d["hbm_gbs"], source="MEASURED_PEAKS.json (measured)")
    return dict(bf16_burst=1590.0, bf16_sustained=1400.0, hbm_gbs=6650.0,
                source="B200_PROFILING.md fallback")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, enabled=True):
        self.proc = None
        self.enabled = enabled

    def __enter__(self):
        if self.enabled:
            try:
                self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                              "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                             text=True)
            except Exception:
                self.proc = None
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.proc is None:
            return
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                self.rows.append(f)

    def summary(self, devices):
        """Median SM clock over samples of the GPUs in use that were under
        load (power above 40 % of the max seen), and every throttle reason
        seen on those GPUs."""
        rows = [r for r in getattr(self, "rows", []) if r[0].isdigit() and int(r[0]) in devices]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        pw = [num(r[3]) or 0.0 for r in rows]
        thr = 0.4 * max(pw) if pw else 0.0
        loaded = [r for r, w in zip(rows, pw) if w >= thr] or rows
        sm = [num(r[1]) for r in loaded if num(r[1]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": num(rows[0][2]),
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(loaded),
                "power_w_max": max(pw) if pw else None}


def devices_in_use(P):
    """nvidia-smi indices of the GPUs the P local ranks use (local rank r ->
    CUDA device r, mapped through CUDA_VISIBLE_DEVICES when it is set)."""
    vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
    ids = [int(x) for x in vis.split(",") if x.strip().isdigit()]
    return set(ids[:P]) if ids else set(range(P))


def host_cpu():
    """lscpu model name and the host's logical CPU count."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return model, os.cpu_count()


def load_ncu(kind, D, N, P, det=False):
    """Pipe utilisations of the attention kernels from the committed ncu
    summary (profiles/ncu_metrics.json, written from `ncu --set full`
    captures; the file names its source reports)."""
    path = os.path.join(ROOT, "profiles", "ncu_metrics.json")
    if not os.path.exists(path):
        return None
    try:
        d = json.load(open(path))
        key = f"{kind}{'_det' if det else ''}_D{D}_N{N}"
        if f"{key}_P{P}" in d:
            return d[f"{key}_P{P}"]
        if f"{key}_P1" in d:   # the per-rank kernel at P > 1 is the same kernel on H/P heads
            return dict(d[f"{key}_P1"], note=f"P = 1 capture; at P = {P} each rank runs the same kernel on H/P heads")
        return None
    except Exception:
        return None


def cpu_baseline(steps=1, n_sample=24576, D=64):
    """The fp64 oracle as it stands: fwd + bwd of one head over the first
    n_sample tokens (same D), timed on this host's cores."""
    import numpy as np
    import oracle
    import synth
    q, k, v, do = synth.qkv(1, n_sample, 1, D, seed=synth.BASE_SEED, with_do=True)
    args = [synth.to_f64(t) for t in (q, k, v, do)]
    oracle.num_threads()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        oracle.attn_fwd(*args[:3])
        oracle.attn_bwd(*args)
        times.append(time.perf_counter() - t0)
    fwd, bwd = flops_per_step(1, n_sample, 1, D)
    t = float(np.mean(times))
    value = (fwd + bwd) / t / 1e12
    full_fwd, full_bwd = flops_per_step(WORKLOAD["B"], WORKLOAD["N"], WORKLOAD["H"], D)
    model, ncpu = host_cpu()
    return dict(value=value, unit=UNIT, cores=oracle.num_threads(), kind="oracle",
                sample=f"fwd+bwd of 1 of {WORKLOAD['H']} heads over the first {n_sample} of {WORKLOAD['N']} tokens "
                       f"(D={D}), fp64 oracle, {steps} run(s) of {t:.2f} s; algorithmic flops 14*n^2*D per head",
                seconds=t, cpu_model=model, host_logical_cpus=ncpu, threads=oracle.num_threads(),
                extrapolated_full_c4_s=(full_fwd + full_bwd) / (value * 1e12),
                extrapolated_note="EXTRAPOLATED, not measured: full c4 fwd+bwd (14*N^2*H*D = "
                                  f"{(full_fwd + full_bwd):.3e} flop) at the sampled rate")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        # torchrun sets OMP_NUM_THREADS=1 per rank; rank 0 runs the oracle alone, on all host cores
        import oracle
        oracle.set_num_threads(len(os.sched_getaffinity(0)))
    n_sample = 8192
    W, K = args.warmup, args.steps
    base = cpu_baseline(steps=1, n_sample=n_sample)  # warm-up compile / first touch
    for _ in range(max(0, W - 1)):
        cpu_baseline(steps=1, n_sample=n_sample)
    r = cpu_baseline(steps=K, n_sample=n_sample)
    out = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus,
           "steps": K, "warmup": W, "ms_per_step": r["seconds"] * 1e3, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": "c4 (sampled): fwd+bwd of one head, first 8192 of 188416 tokens, D=64",
                      "B": 1, "N": WORKLOAD["N"], "H": WORKLOAD["H"], "D": WORKLOAD["D"]},
           "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model", "threads",
                                              "extrapolated_full_c4_s", "extrapolated_note")},
           "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    del base
    print(json.dumps(out), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--N", type=int, default=WORKLOAD["N"])
    ap.add_argument("--H", type=int, default=WORKLOAD["H"])
    ap.add_argument("--D", type=int, default=WORKLOAD["D"])
    ap.add_argument("--B", type=int, default=WORKLOAD["B"], help="batch (the paper's local batch is 4, P:425)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--a2a", default="auto", choices=["auto", "nccl", "peer"],
                    help="all-to-all transport for P > 1: NCCL send/recv, or NVLink peer stores from the kernels; "
                         "auto = peer for P in {2, 4} (validated on hardware, +0.8 / +1.2 %% at c4), NCCL otherwise")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--deterministic", action="store_true",
                    help="bitwise-reproducible backward (query-stationary dQ kernel; same algorithmic flop count)")
    ap.add_argument("--strategy", default="ulysses", choices=["ulysses", "lss"],
                    help="sequence-parallel strategy: Ulysses all-to-all (headline) or LSS gather-KV / reduce-scatter")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import paper_2405_15780_b200 as ua
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    P = world
    if args.a2a == "auto":
        args.a2a = "peer" if P in (2, 4) else "nccl"
    if args.gpus != world:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using {world}", file=sys.stderr)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    B, N, H, D = args.B, args.N, args.H, args.D
    lss = args.strategy == "lss"
    (ua.lss_validate if lss else ua.validate)(B, N, H, D, P)
    Nl = N // P
    fwd_fn = ua.lss_attn_fwd if lss else ua.ulysses_attn_fwd
    bwd_fn = ua.lss_attn_bwd if lss else ua.ulysses_attn_bwd
    ctx = ua.Context(P=P, rank=rank, device=local)
    if P > 1 and not lss:
        ctx.set_a2a_mode(args.a2a)
    if args.deterministic:
        ctx.set_deterministic(True)
    dev = torch.device("cuda", local)
    shape = (B, Nl, H, D)
    import synth
    # counter-based draws of this rank's sequence shard of the global tensors: the data are
    # identical for every P (synth/__init__.py); drawn on the host once, before any timing
    host_in = synth.qkv(B, N, H, D, seed=synth.BASE_SEED, with_do=True, n0=rank * Nl, n1=(rank + 1) * Nl)
    q, k, v, do = (t.to(dev) for t in host_in)
    fb, bb = (ua.lss_workspace_size if lss else ua.workspace_size)(B, N, H, D, P)
    ctx.workspace(max(fb, bb))
    out = torch.empty_like(q)
    lse = torch.empty((B, H, Nl) if lss else (B, H // P, N), dtype=torch.float32, device=dev)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    stream = torch.cuda.current_stream()

    def step(qq=q, kk=k, vv=v, dd=do):
        fwd_fn(ctx, qq, kk, vv, out=out, lse=lse)
        bwd_fn(ctx, qq, kk, vv, out, lse, dd, dq=dq, dk=dk, dv=dv)

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ctx.phase_times()  # drop warm-up records
    calls0, bytes0 = ctx.comm_stats()

    # ---------------------------------------------------------------- timed
    ctx.enable_timing(True)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(enabled=(rank == 0)) as clk:
        evs[0].record(stream)
        for i in range(args.steps):
            step()
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
    barrier()
    ms_total = max_over_ranks(evs[0].elapsed_time(evs[-1]))
    per_step = torch.tensor([evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)], dtype=torch.float64,
                            device=dev)
    if dist is not None:
        dist.all_reduce(per_step, op=dist.ReduceOp.MAX)
    per_step = per_step.cpu().tolist()
    ctx.enable_timing(False)
    phases = ctx.phase_times()
    calls1, bytes1 = ctx.comm_stats()
    ms_step = ms_total / args.steps

    fwd_f, bwd_f = flops_per_step(B, N, H, D)
    tflops = (fwd_f + bwd_f) / (ms_step * 1e-3) / 1e12
    peaks = load_peaks()

    # roofline of the dominant kernel (attention backward), per launch on this rank
    def kstats(name, flops_total):
        ms, n = phases[name]
        if n == 0:
            return None
        avg = ms / n
        fl = flops_total / P  # this rank's heads
        return dict(avg_ms=avg, launches=n, tflops=fl / (avg * 1e-3) / 1e12)

    kb = kstats("attn_bwd", bwd_f)
    kf = kstats("attn_fwd", fwd_f)
    ncu_b = None if lss or B != 1 else load_ncu("attn_bwd", D, N, P, args.deterministic)
    ncu_f = None if lss or B != 1 else load_ncu("attn_fwd", D, N, P)
    traffic = ncu_b.get("dram_bytes") if (ncu_b and "note" not in ncu_b) else None   # per launch, this shape only
    roofline = {"bound": "tensor", "kernel": "attn_bwd_kernel", "achieved": kb["tflops"],
                "peak": peaks["bf16_sustained"], "unit": UNIT, "frac": kb["tflops"] / peaks["bf16_sustained"],
                "frac_of_burst": kb["tflops"] / peaks["bf16_burst"], "peak_source": peaks["source"] + " sustained",
                "traffic": traffic, "traffic_source": ncu_b.get("source") if ncu_b else None,
                "flops_per_launch": bwd_f / P, "flops_formula": "10*B*N^2*(H/P)*D per launch (5 GEMMs incl. recompute)"}
    fwd_roof = {"kernel": "attn_fwd_kernel", "achieved": kf["tflops"], "frac": kf["tflops"] / peaks["bf16_sustained"],
                "avg_ms": kf["avg_ms"], "traffic": ncu_f.get("dram_bytes") if (ncu_f and "note" not in ncu_f) else None}
    ncu = {"attn_bwd": ncu_b, "attn_fwd": ncu_f,
           "note": "from the committed ncu --set full captures named in each entry's source (not this run)"}
    # our kernels per phase call: attn_bwd = bwd_prep + the backward kernel (+ the dQ kernel in
    # deterministic mode); the other non-a2a phases launch one kernel each (a2a phases: NCCL)
    per_call = {"attn_bwd": 3 if args.deterministic else 2}
    launches = sum(n * per_call.get(name, 1) for name, (ms, n) in phases.items() if not name.startswith("a2a"))
    phase_ms = {name: ms / args.steps for name, (ms, n) in phases.items() if n}
    a2a_ms = sum(ms for name, (ms, n) in phases.items() if name.startswith("a2a"))
    comm_ms = sum(ms for name, (ms, n) in phases.items() if name.startswith(("a2a", "pack", "unpack")))
    # peer transport: the NVLink stores happen in the pack / attention / finaliser kernels, so the
    # transfer time is the data-movement phases, not the (flag-wait only) a2a phases
    xfer_ms = comm_ms if (P > 1 and not lss and args.a2a == "peer") else a2a_ms
    a2a_bytes = bytes1 - bytes0

    # ---------------------------------------------------------------- e2e
    e2e = None
    if not args.no_e2e:
        # End to end through the public API with host buffers: every step copies its q, k, v, dO
        # from pinned host memory and its out, dq, dk, dv back.  Copies run on their own stream,
        # double-buffered: step i+1's inputs upload and step i-1's results download while step i
        # computes (what a training loop's prefetcher does).  The timed region spans the first
        # upload to the last download.
        hq, hk, hv, hd = (t.pin_memory() for t in host_in)
        hout = [[torch.empty(shape, dtype=torch.bfloat16).pin_memory() for _ in range(4)] for _ in range(2)]
        dins = [[torch.empty_like(q) for _ in range(4)] for _ in range(2)]
        douts = [[torch.empty_like(q) for _ in range(4)] for _ in range(2)]
        lses = [torch.empty_like(lse) for _ in range(2)]
        cstream = torch.cuda.Stream(device=dev)
        uploaded = [torch.cuda.Event() for _ in range(2)]      # inputs of buffer b are on the device
        computed = [torch.cuda.Event() for _ in range(2)]      # step on buffer b finished
        downloaded = [torch.cuda.Event() for _ in range(2)]    # results of buffer b are on the host

        def upload(b):
            with torch.cuda.stream(cstream):
                cstream.wait_event(computed[b])                  # buffer b's previous step is done
                for dst, src in zip(dins[b], (hq, hk, hv, hd)):
                    dst.copy_(src, non_blocking=True)
                uploaded[b].record(cstream)

        def download(b):
            with torch.cuda.stream(cstream):
                cstream.wait_event(computed[b])
                for dst, src in zip(hout[b], douts[b]):
                    dst.copy_(src, non_blocking=True)
                downloaded[b].record(cstream)

        def compute(b):
            stream.wait_event(uploaded[b])
            stream.wait_event(downloaded[b])                     # buffer b's previous results are out
            q_, k_, v_, d_ = dins[b]
            o_, dq_, dk_, dv_ = douts[b]
            fwd_fn(ctx, q_, k_, v_, out=o_, lse=lses[b])
            bwd_fn(ctx, q_, k_, v_, o_, lses[b], d_, dq=dq_, dk=dk_, dv=dv_)
            computed[b].record(stream)

        def run(nsteps):
            for b in range(2):
                computed[b].record(stream)
                downloaded[b].record(stream)
            upload(0)
            for i in range(nsteps):
                b = i % 2
                if i + 1 < nsteps:
                    upload(1 - b)
                compute(b)
                download(b)
            stream.wait_stream(cstream)

        run(2)
        torch.cuda.synchronize()
        barrier()
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        run(args.steps)
        b_.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms_e2e = max_over_ranks(a.elapsed_time(b_)) / args.steps
        nbytes = q.numel() * 2
        e2e = {"value": (fwd_f + bwd_f) / (ms_e2e * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": ms_e2e,
               "h2d_bytes_per_step": 4 * nbytes, "d2h_bytes_per_step": 4 * nbytes,
               "tokens_per_s": B * N / (ms_e2e * 1e-3),
               "path": f"pinned host q,k,v,dO -> H2D -> ua_{args.strategy}_attn_fwd/bwd -> D2H out,dq,dk,dv "
                       "(per rank; copies on a second stream, double-buffered across steps)"}

    if rank == 0:
        res = {
            "metric": METRIC, "value": tflops, "unit": UNIT, "n_gpus": P, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"{CONFIG_NAMES.get((N, H, D), 'custom')}: {'LSS' if lss else 'Ulysses'} attention fwd+bwd, N={N} tokens, H={H}, D={D}, B={B}, P={P}",
                       "B": B, "N": N, "H": H, "D": D, "P": P, "parallelism": f"{args.strategy}-sp{P}",
                       "a2a": ("nccl all-gather/reduce-scatter" if lss else args.a2a) if P > 1 else "none",
                       "l2": "inputs larger than L2 (each q/k/v/dO shard "
                             f"{q.numel() * 2 / 1e6:.0f} MB; working set > 126 MB)",
                       "inputs": "N(0,1) bf16 from synth/ (counter-based PCG64 blocks keyed by seed, tensor, b, h and "
                                 "1024-token block: the global data are identical for every P), seed 1234",
                       "deterministic_bwd": bool(args.deterministic)},
            "tokens_per_s": B * N / (ms_step * 1e-3),
            "paper_context": PAPER_CONTEXT,
            "pct_of_bf16_peak": tflops / (P * peaks["bf16_sustained"]) * 100,
            "pct_of_bf16_burst_peak": tflops / (P * peaks["bf16_burst"]) * 100,
            "pct_of_bf16_datasheet_2250": tflops / (P * 2250.0) * 100,
            "fwd_only_tokens_per_s": B * N / (sum(v for k_, v in phase_ms.items() if k_.endswith("_fwd")
                                                    or k_ == "a2a_fwd_in" or k_ == "a2a_fwd_out") * 1e-3)
            if phase_ms.get("attn_fwd") else None,
            "a2a_call_law_ok": (calls1 - calls0) == (0 if P == 1 else (3 if lss else 4)) * args.steps,
            "fwd_tflops_per_gpu_kernel": kf["tflops"], "bwd_tflops_per_gpu_kernel": kb["tflops"],
            "roofline": roofline, "roofline_fwd": fwd_roof,
            "phases_ms_per_step": phase_ms,
            "a2a": {"calls": calls1 - calls0, "bytes_sent_per_rank": a2a_bytes, "ms_per_step": a2a_ms / args.steps,
                    "comm_ms_per_step": comm_ms / args.steps,
                    "comm_share_of_step": (comm_ms / args.steps) / ms_step if P > 1 else 0.0,
                    "GBps": (a2a_bytes / (xfer_ms * 1e-3) / 1e9) if xfer_ms > 0 else None,
                    "frac_of_nvlink": (a2a_bytes / (xfer_ms * 1e-3) / 1e9 / NVLINK_GBS) if xfer_ms > 0 else None,
                    "nvlink_gbs": NVLINK_GBS,
                    "note": ("bytes this rank sent to other ranks / device time of the phases that move them: "
                             + ("the a2a phases (NCCL send/recv incl. launch and wait)" if args.a2a == "nccl" or lss
                                else "pack_push + flag waits + copy-out (the peer stores happen inside the pack and "
                                     "attention kernels)")
                             + "; per direction.  comm_ms = pack + a2a + unpack phases per step")},
            "ncu": ncu,
            "ms_per_step_median": statistics.median(per_step), "ms_per_step_min": min(per_step),
            "ms_per_step_max": max(per_step),
            "gpu_launches": launches,
            "clocks": clk.summary(devices_in_use(P)),
            "e2e": e2e,
        }
        if P == 1 and not args.no_cpu_baseline:
            cb = cpu_baseline(steps=1)
            res["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model", "threads",
                                                      "extrapolated_full_c4_s", "extrapolated_note")}
        print(json.dumps(res), flush=True)
    ctx.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
