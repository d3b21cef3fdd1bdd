# The whole single-GPU suite as the driver runs it (timed), parity margins logged, then the bench.
set -x
mkdir -p gpurun_out
export UA_PARITY_LOG=gpurun_out/parity_r2d.jsonl
rm -f $UA_PARITY_LOG
start=$(date +%s)
timeout 2400 python -m pytest tests/ -x -q -m gpu -rs --durations=25 > gpurun_out/pytest_r2d.log 2>&1; echo pytest rc=$? secs=$(( $(date +%s) - start ))
tail -40 gpurun_out/pytest_r2d.log
unset UA_PARITY_LOG
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke rc=$?
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2d.json 2> gpurun_out/bench_r2d.err; echo bench rc=$?
tail -c 400 gpurun_out/bench_r2d.json
