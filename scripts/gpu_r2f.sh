# c2 (N = 8192, H = 16, D = 64) ncu full captures, and the deterministic-backward bench at c4.
set -x
o=gpurun_out
mkdir -p $o
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd_split" -c 1 -o $o/r02_fwd_c2 \
  python scripts/prof_kernel.py --N 8192 --H 16 --iters 0 --fwd-only > $o/r02_fwd_c2.log 2>&1; echo fwd rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd_ws" -c 1 -o $o/r02_bwd_c2 \
  python scripts/prof_kernel.py --N 8192 --H 16 --iters 0 > $o/r02_bwd_c2.log 2>&1; echo bwd rc=$?
for r in r02_fwd_c2 r02_bwd_c2; do ncu -i $o/$r.ncu-rep --page raw --csv > $o/$r.raw.csv 2>/dev/null; done
timeout 900 python bench.py --steps 5 --warmup 3 --deterministic --no-cpu-baseline > $o/r02_bench_det.json 2> $o/r02_bench_det.err; echo det rc=$?
tail -c 300 $o/r02_bench_det.json
timeout 900 python bench.py --steps 3 --warmup 3 --N 65536 --H 16 --D 128 --no-cpu-baseline > $o/r02_bench_c3_p1.json 2> $o/r02_bench_c3.err; echo c3 rc=$?
tail -c 200 $o/r02_bench_c3_p1.json
