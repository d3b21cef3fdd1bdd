# Peer transport on NCCL symmetric windows: multi-rank tests at P = 2 and the default bench at P = 2.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q -x -k "ulysses_p_way or layer" > gpurun_out/r02_ncclwin_tests.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/r02_ncclwin_tests.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29741 \
  bench.py --gpus 2 --no-cpu-baseline > gpurun_out/r02_ncclwin_bench2.json 2> gpurun_out/r02_ncclwin_bench2.err; echo bench rc=$?
tail -c 600 gpurun_out/r02_ncclwin_bench2.json; grep -i "error\|warn" gpurun_out/r02_ncclwin_bench2.err | head -5
