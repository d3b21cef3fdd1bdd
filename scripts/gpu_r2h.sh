set -x
timeout 900 python -m pytest tests/test_fuzz_gpu.py -m gpu -q -rf > gpurun_out/pytest_r2h.log 2>&1; echo pytest rc=$?
tail -4 gpurun_out/pytest_r2h.log
