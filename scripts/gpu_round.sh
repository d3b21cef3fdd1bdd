set -x
nvidia-smi -L
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 600 python bench.py > gpurun_out/bench_v10.json 2> gpurun_out/bench_v10.err; echo bench rc=$?
tail -2 gpurun_out/bench_v10.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2>gpurun_out/ref.err; echo ref rc=$?
tail -1 gpurun_out/ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v10.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo ncu rc=$?
