set -x
V=paper_2405_15780_b200/variants
L=paper_2405_15780_b200/libulysses_attn.so
timeout 1200 python scripts/ab.py --what fwd --rounds 5 --N 188416 --libs $L $V/libnoxchg.so 2>&1 | tail -3
timeout 600 python scripts/ab.py --what fwd --rounds 8 --libs $L $V/libnoxchg.so 2>&1 | tail -3
timeout 600 python scripts/ab.py --what fwd --rounds 8 --N 32768 --D 32 --H 16 --libs $L $V/libnoxchg.so 2>&1 | tail -3
