# The driver's GPUTEST command on a 4-GPU box (timed): every -m gpu test, default subset.
set -x
mkdir -p gpurun_out
nvidia-smi -L
start=$(date +%s)
timeout 3300 python -m pytest tests/ -x -q -m gpu -rs --durations=15 > gpurun_out/r02_suite4.log 2>&1; echo pytest rc=$? secs=$(( $(date +%s) - start ))
tail -32 gpurun_out/r02_suite4.log
