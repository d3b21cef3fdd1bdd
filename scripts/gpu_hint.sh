set -x
V=paper_2405_15780_b200/variants
L=paper_2405_15780_b200/libulysses_attn.so
timeout 1200 python scripts/ab.py --what bwd --rounds 4 --N 188416 --libs $L $V/libqdonormal.so $V/libqdofirst.so 2>&1 | tail -4
