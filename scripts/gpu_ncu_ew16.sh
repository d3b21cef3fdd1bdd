# ncu --set full of the backward at the c4 sequence length, one head: EW16 (default build) vs 32x32b.
set -x
o=gpurun_out
V=paper_2405_15780_b200/variants
for lib in paper_2405_15780_b200/libulysses_attn.so $V/libnoew16.so; do
  n=$(basename $lib .so)
  timeout 900 ncu --set full --clock-control none -k regex:"attn_bwd_ws" -c 1 -o $o/ew_$n \
    python scripts/ab.py --libs $lib --what bwd --rounds 1 --N 188416 --H 1 > $o/ew_$n.log 2>&1; echo $n rc=$?
  ncu -i $o/ew_$n.ncu-rep --page raw --csv > $o/ew_$n.raw.csv 2>/dev/null
  rm -f $o/ew_$n.ncu-rep
done
