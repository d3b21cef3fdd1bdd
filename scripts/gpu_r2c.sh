# LSS single-GPU simulated-rank tests, the layout tests, then compute-sanitizer
# (memcheck, racecheck, synccheck) on small forward / backward / layout calls.
set -x
mkdir -p gpurun_out
export UA_PARITY_LOG=gpurun_out/parity_r2c.jsonl
rm -f $UA_PARITY_LOG
timeout 900 python -m pytest tests/test_lss_sim_gpu.py tests/test_layout_gpu.py -m gpu -q -rf > gpurun_out/pytest_r2c.log 2>&1; echo pytest rc=$?
tail -8 gpurun_out/pytest_r2c.log
unset UA_PARITY_LOG
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_run.py > gpurun_out/r02_sanitize_$tool.log 2>&1
  echo $tool rc=$?
  tail -4 gpurun_out/r02_sanitize_$tool.log
done
