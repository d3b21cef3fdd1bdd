# Round 2, first GPU pass: new single-GPU layout / simulated-rank tests, full-size
# dK/dV rows, sigma_qk = 4 cases; parity margins logged; then one bench line.
set -x
mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build()"
export UA_PARITY_LOG=gpurun_out/parity_r2a.jsonl
rm -f $UA_PARITY_LOG
timeout 2400 python -m pytest tests/test_layout_gpu.py tests/test_fwd_gpu.py tests/test_bwd_gpu.py -m gpu -q -rf \
  --durations=15 > gpurun_out/pytest_r2a.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_r2a.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; echo bench rc=$?
tail -c 600 gpurun_out/bench_r2a.json
