# The driver's bench command at P = 2 (default arguments: --a2a auto -> peer) and P = 1.
set -x
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29731 \
  bench.py --gpus 2 > gpurun_out/r02_bench_default_2.json 2> gpurun_out/r02_bench_default_2.err; echo rc=$?
tail -c 1500 gpurun_out/r02_bench_default_2.json
tail -5 gpurun_out/r02_bench_default_2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29732 \
  bench.py --gpus 2 --impl reference > gpurun_out/r02_ref_2.json 2> gpurun_out/r02_ref_2.err; echo ref rc=$?
tail -c 300 gpurun_out/r02_ref_2.json
