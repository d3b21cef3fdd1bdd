# tcgen05 projection GEMM: parity (standalone + layer), throughput at c4 shapes.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py -m gpu -q -x > gpurun_out/pytest_gemm.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gemm.log
timeout 300 python scripts/gemm_bench.py 2>&1 | tail -4
