#!/bin/bash
# Multi-GPU validation + scaling run (used under gpurun --gpus N).
NG=$(nvidia-smi -L | wc -l)
echo "GPUs: $NG"
# env: STRATEGY=ulysses|lss (bench), TESTS=-k expression for the multi-GPU tests ("" = all, "none" = skip)
STRATEGY=${STRATEGY:-ulysses}
TESTS=${TESTS-}
if [ "$TESTS" != "none" ]; then
  timeout 1200 python -m pytest tests/test_multigpu.py -q -m gpu -x ${TESTS:+-k "$TESTS"} 2>&1 | tail -3
fi
for n in 1 2 4 8; do
  if [ $n -le $NG ]; then
    if [ $n -eq 1 ]; then
      timeout 600 python bench.py --no-cpu-baseline --strategy $STRATEGY > gpurun_out/scale_${STRATEGY}_$n.json 2> gpurun_out/scale_${STRATEGY}_$n.err
    else
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $((29600 + n)) bench.py --gpus $n --no-cpu-baseline --strategy $STRATEGY > gpurun_out/scale_${STRATEGY}_$n.json 2> gpurun_out/scale_${STRATEGY}_$n.err
    fi
    echo "n=$n rc=$? bytes=$(wc -c < gpurun_out/scale_${STRATEGY}_$n.json)"
    python - "$n" "$STRATEGY" <<'PY'
import json, sys
n, st = sys.argv[1], sys.argv[2]
try:
    d = json.loads([l for l in open(f"gpurun_out/scale_{st}_{n}.json") if l.startswith("{")][-1])
    print(n, round(d["value"], 1), "TFLOP/s", round(d["ms_per_step"], 1), "ms/step",
          {k: round(v, 2) for k, v in d["phases_ms_per_step"].items()}, d["a2a"],
          "e2e", d["e2e"]["value"] if d["e2e"] else None, d["clocks"])
except Exception as e:
    print("parse failed", n, e)
PY
  fi
done
