# Peer transport on NCCL symmetric windows at P = 4: multi-rank tests (incl. full-size peer cases), bench.
set -x
mkdir -p gpurun_out
UA_MGPU_FULL=1 timeout 1800 python -m pytest tests/test_multigpu.py -m gpu -q -x -k "ulysses_p_way or peer or layer" > gpurun_out/r02_ncclwin4_tests.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/r02_ncclwin4_tests.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29742 \
  bench.py --gpus 4 --no-cpu-baseline > gpurun_out/r02_ncclwin_bench4.json 2> gpurun_out/r02_ncclwin_bench4.err; echo bench rc=$?
tail -c 300 gpurun_out/r02_ncclwin_bench4.json
