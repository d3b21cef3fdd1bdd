o=gpurun_out
timeout 600 python bench.py > $o/bench_v13.json 2> $o/bench_v13.err; echo bench rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_v13.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $o/ncu13.log 2>&1; echo ncu rc=$?
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file $o/traffic_v13.csv python scripts/prof_kernel.py --N 188416 --iters 1 > /dev/null 2>&1; echo traffic rc=$?
python -c "
import json; d=json.loads([l for l in open('$o/bench_v13.json') if l.startswith('{')][-1]); print(round(d['value'],1), d['ms_per_step'], 'fwd', round(d['fwd_tflops_per_gpu_kernel'],1), 'bwd', round(d['bwd_tflops_per_gpu_kernel'],1), 'e2e', round(d['e2e']['value'],1), d['clocks'])"
