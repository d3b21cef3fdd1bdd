# c3 (N = 65,536, H = 16, D = 128) and c5 (N = 1,048,576, H = 32, D = 128) on 4 GPUs, final code.
set -x
mkdir -p gpurun_out
for cfg in "65536 16 128 c3" "1048576 32 128 c5"; do
  set -- $cfg
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29911 bench.py --gpus 4 --N $1 --H $2 --D $3 --steps 3 --warmup 3 --no-e2e \
    > gpurun_out/r02_bench_$4_p4.json 2> gpurun_out/r02_bench_$4_p4.err
  echo "$4 rc=$?"
  tail -c 300 gpurun_out/r02_bench_$4_p4.json
done
