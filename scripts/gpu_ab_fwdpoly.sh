cd paper_2405_15780_b200
for v in "sp3 UA_FWD_SPLIT_POLY16=3" "sp5 UA_FWD_SPLIT_POLY16=5" "sp6 UA_FWD_SPLIT_POLY16=6"; do set -- $v; python build.py --variant $1 $2 > /dev/null & done; wait
cd ..
V=paper_2405_15780_b200/variants
timeout 300 python scripts/ab.py --what fwd --rounds 10 --N 65536 --libs paper_2405_15780_b200/libulysses_attn.so $V/libsp3.so $V/libsp5.so $V/libsp6.so
