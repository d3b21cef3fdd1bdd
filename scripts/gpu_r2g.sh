# Final single-GPU sanity on the final code: shape fuzz, GEMM / layer, ABI-level smoke.
set -x
mkdir -p gpurun_out
export UA_PARITY_LOG=gpurun_out/parity_r2g.jsonl
rm -f $UA_PARITY_LOG
timeout 1200 python -m pytest tests/test_fuzz_gpu.py tests/test_gemm_gpu.py tests/test_layer_gpu.py -m gpu -q -rf > gpurun_out/pytest_r2g.log 2>&1; echo pytest rc=$?
tail -6 gpurun_out/pytest_r2g.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke rc=$?
