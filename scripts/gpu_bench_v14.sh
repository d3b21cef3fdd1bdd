o=gpurun_out
timeout 600 python bench.py --no-cpu-baseline > $o/bench_v14_p1.json 2> $o/b14_1.err; echo p1 rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29688 bench.py --gpus 2 > $o/bench_v14_p2.json 2> $o/b14_2.err; echo p2 rc=$?
timeout 600 python -m pytest tests/test_multigpu.py -m gpu -q -x -k "test_ulysses_p_way and 4096 and 8 and 64" 2>&1 | tail -2
for n in 1 2; do python -c "
import json; d=json.loads([l for l in open('$o/bench_v14_p$n.json') if l.startswith('{')][-1]); print($n, round(d['value'],1), d['ms_per_step'], 'fwd', round(d['fwd_tflops_per_gpu_kernel'],1), 'bwd', round(d['bwd_tflops_per_gpu_kernel'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"; done
