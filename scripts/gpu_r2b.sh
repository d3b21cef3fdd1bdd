set -x
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo bench rc=$?
tail -c 300 gpurun_out/bench_r2b.json
bash scripts/gpu_ncu_r2.sh
