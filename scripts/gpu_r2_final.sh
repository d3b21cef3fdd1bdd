# Final round-2 pass on a 4-GPU box: every multi-rank test (P = 2, 4) on the final code, then the
# driver's bench command (default arguments) at P = 1, 2, 4.
set -x
mkdir -p gpurun_out
nvidia-smi -L
timeout 3300 python -m pytest tests/test_multigpu.py -m gpu -q -rf --durations=10 > gpurun_out/r02_mgpu_final.log 2>&1; echo mgpu rc=$?
tail -16 gpurun_out/r02_mgpu_final.log
timeout 900 python bench.py > gpurun_out/r02_final_1.json 2> gpurun_out/r02_final_1.err; echo "n=1 rc=$?"
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29800 + n)) bench.py --gpus $n > gpurun_out/r02_final_$n.json 2> gpurun_out/r02_final_$n.err
  echo "n=$n rc=$?"
done
for n in 1 2 4; do python -c "
import json,sys; d=json.loads([l for l in open('gpurun_out/r02_final_$n.json') if l.startswith('{')][-1])
print($n, round(d['value'],1), round(d['ms_per_step'],1), d['config']['a2a'], 'e2e', round(d['e2e']['value'],1), 'comm', round(d['a2a']['comm_share_of_step'],4), d['clocks']['sm_mhz'])"; done
