# Bench lines for the BASELINE.json configs (run on a 4-GPU box): python bench.py at P=1, torchrun at P=2, 4.
o=gpurun_out
b1() { name=$1; shift; timeout 400 python bench.py --no-cpu-baseline "$@" > $o/cfg_$name.json 2> $o/cfg_$name.err; echo "$name rc=$?"; }
bn() { n=$1; name=$2; shift 2; timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $n --no-cpu-baseline "$@" > $o/cfg_$name.json 2> $o/cfg_$name.err; echo "$name rc=$?"; }
b1 c2_p1 --N 8192 --H 16 --D 64 --no-e2e
b1 c3_p1 --N 65536 --H 16 --D 128 --no-e2e
b1 c4_p1_det --deterministic --no-e2e
b1 c4_p1_h16 --H 16 --no-e2e
b1 c4_p1_b4 --B 4 --steps 3 --no-e2e
bn 2 c4_p2
bn 4 c4_p4
bn 2 c3_p2 --N 65536 --H 16 --D 128 --no-e2e
bn 4 c3_p4 --N 65536 --H 16 --D 128 --no-e2e
bn 4 c4_p4_det --deterministic --no-e2e
bn 4 c5_p4 --N 1048576 --H 32 --D 128 --steps 3 --warmup 3 --no-e2e
for f in $o/cfg_*.json; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    print(f.split("cfg_")[1][:-5], round(d["value"], 1), d["unit"], round(d["ms_per_step"], 1), "ms/step",
          "fwd", round(d.get("fwd_tflops_per_gpu_kernel", 0), 1), "bwd", round(d.get("bwd_tflops_per_gpu_kernel", 0), 1),
          "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"], "e2e", (d["e2e"] or {}).get("value"))
except Exception as e:
    print("parse failed", f, e)
PY
done
