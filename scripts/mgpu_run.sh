#!/bin/bash
# Multi-GPU validation + scaling run (used under gpurun --gpus N).
set -x
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_multigpu.py -q -m gpu -x 2>&1 | tail -5
for n in 1 2 4 8; do
  if [ $n -le $NG ]; then
    if [ $n -eq 1 ]; then
      timeout 600 python bench.py --no-cpu-baseline > gpurun_out/scale_$n.json 2> gpurun_out/scale_$n.err
    else
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --no-cpu-baseline > gpurun_out/scale_$n.json 2> gpurun_out/scale_$n.err
    fi
    tail -2 gpurun_out/scale_$n.err
    python -c "import json;d=json.load(open('gpurun_out/scale_$n.json'));print($n, round(d['value'],1), round(d['ms_per_step'],1), d['phases_ms_per_step'], d['a2a'], d['e2e']['value'] if d['e2e'] else None)"
  fi
done
