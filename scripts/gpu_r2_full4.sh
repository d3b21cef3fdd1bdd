# Every multi-rank test including the full-size BASELINE matrix (UA_MGPU_FULL=1) on a 4-GPU box.
set -x
mkdir -p gpurun_out
start=$(date +%s)
UA_MGPU_FULL=1 timeout 3000 python -m pytest tests/test_multigpu.py -m gpu -q -rs --durations=12 > gpurun_out/r02_mgpu_full4.log 2>&1; echo mgpu rc=$? secs=$(( $(date +%s) - start ))
tail -24 gpurun_out/r02_mgpu_full4.log
