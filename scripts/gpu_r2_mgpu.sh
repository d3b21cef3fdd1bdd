# Round 2 multi-GPU pass (gpurun --gpus 4): LSS simulated-rank tests, the torchrun
# multi-rank tests (P = 2, 4; NCCL and peer transports; full-size c3 / c4 / c5),
# then the c4 bench at P = 1, 2, 4 for both transports.
set -x
mkdir -p gpurun_out
nvidia-smi -L
timeout 900 python -m pytest tests/test_lss_sim_gpu.py -m gpu -q -rf > gpurun_out/pytest_lss_sim.log 2>&1; echo lss_sim rc=$?
tail -3 gpurun_out/pytest_lss_sim.log
timeout 3000 python -m pytest tests/test_multigpu.py -m gpu -q -rf --durations=20 > gpurun_out/r02_mgpu.log 2>&1; echo mgpu rc=$?
tail -30 gpurun_out/r02_mgpu.log
for mode in nccl peer; do
  for n in 2 4; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29700 + n)) bench.py --gpus $n --steps 5 --warmup 3 --no-cpu-baseline --a2a $mode \
      > gpurun_out/r02_scale_${mode}_$n.json 2> gpurun_out/r02_scale_${mode}_$n.err
    echo "$mode n=$n rc=$?"
    tail -c 400 gpurun_out/r02_scale_${mode}_$n.json
  done
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_scale_nccl_1.json 2> gpurun_out/r02_scale_nccl_1.err; echo "n=1 rc=$?"
