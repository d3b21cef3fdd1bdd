# Bounded-skew pacing of the persistent backward (UA_BWD_SKEW): parity, interleaved A/B, DRAM traffic.
set -x
mkdir -p gpurun_out
V=paper_2405_15780_b200/variants
L=paper_2405_15780_b200/libulysses_attn.so
timeout 900 python -m pytest tests/test_bwd_gpu.py tests/test_lss_sim_gpu.py -m gpu -q -x -k "not full_size" > gpurun_out/pytest_skew.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_skew.log
timeout 900 python scripts/ab.py --what bwd --rounds 4 --N 188416 --libs $L $V/libskew0.so $V/libskew16.so $V/libskew256.so 2>&1 | tail -5
timeout 400 python scripts/ab.py --what bwd --rounds 6 --libs $L $V/libskew0.so $V/libskew16.so 2>&1 | tail -4
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:attn_bwd_ws --csv --log-file gpurun_out/r02_traffic_skew.csv python scripts/prof_kernel.py --N 188416 --iters 1 > /dev/null 2>&1; echo traffic rc=$?
