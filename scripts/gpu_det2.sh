timeout 300 python -m pytest tests/test_bwd_gpu.py -m gpu -q -x -k "deterministic" 2>&1 | tail -5
for i in 1 2; do
timeout 60 python scripts/prof_kernel.py --N 32768 --det | grep attn_bwd
timeout 60 python scripts/prof_kernel.py --N 32768 | grep attn_bwd
done
timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/det2_launches.csv python scripts/prof_kernel.py --N 32768 --det --iters 1 > /dev/null 2>&1
grep -E "attn_bwd" gpurun_out/det2_launches.csv | cut -c1-20,100-400 | head
