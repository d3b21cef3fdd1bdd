o=gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 300 ncu --metrics $M --clock-control none --csv --log-file $o/traffic_c4.csv python scripts/prof_kernel.py --N 188416 --iters 1 > /dev/null 2>&1; echo traffic rc=$?
timeout 300 ncu --metrics $M --clock-control none --csv --log-file $o/traffic_c4_det.csv python scripts/prof_kernel.py --N 188416 --iters 1 --det > /dev/null 2>&1; echo traffic_det rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd_split" -c 1 -o $o/v11_fwd_c4 python scripts/prof_kernel.py --N 188416 --iters 0 --fwd-only > $o/v11_fwd.log 2>&1; echo fwd rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd" -c 1 -o $o/v11_bwd_65k python scripts/prof_kernel.py --N 65536 --iters 0 > $o/v11_bwd.log 2>&1; echo bwd rc=$?
