set -x
V=paper_2405_15780_b200/variants
L=paper_2405_15780_b200/libulysses_attn.so
timeout 1200 python scripts/ab.py --what fwd --rounds 4 --N 188416 --libs $L $V/libfpoly3.so $V/libfpoly5.so $V/libfpoly6.so 2>&1 | tail -5
timeout 600 python scripts/ab.py --what fwd --rounds 8 --libs $L $V/libfpoly3.so $V/libfpoly5.so $V/libfpoly6.so 2>&1 | tail -5
