# Round 2 profiles: launch list of the bench command, DRAM traffic per launch at
# full c4 (H = 32), and one `ncu --set full` capture per attention kernel at the
# c4 sequence length with one head (N = 188,416, H = 1; the full-H backward does
# not replay under --set full).
set -x
o=gpurun_out
mkdir -p $o
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/r02_launches_c4_p1.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $o/r02_ncu_launch.log 2>&1; echo launches rc=$?
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $o/r02_traffic_c4.csv \
  python scripts/prof_kernel.py --N 188416 --iters 1 > /dev/null 2>&1; echo traffic rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd_split" -c 1 -o $o/r02_fwd_c4h1 \
  python scripts/prof_kernel.py --N 188416 --H 1 --iters 0 --fwd-only > $o/r02_fwd.log 2>&1; echo fwd rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd_ws" -c 1 -o $o/r02_bwd_c4h1 \
  python scripts/prof_kernel.py --N 188416 --H 1 --iters 0 > $o/r02_bwd.log 2>&1; echo bwd rc=$?
for r in r02_fwd_c4h1 r02_bwd_c4h1; do
  ncu -i $o/$r.ncu-rep --page raw --csv > $o/$r.raw.csv 2>/dev/null
done
ls -la $o
