python scripts/prof_kernel.py --N 32768 --det
python scripts/prof_kernel.py --N 32768
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/det_launches.csv python scripts/prof_kernel.py --N 32768 --det --iters 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd" -c 2 -o gpurun_out/det_bwd python scripts/prof_kernel.py --N 32768 --det --iters 0 > gpurun_out/det_ncu.log 2>&1; echo ncu rc=$?
