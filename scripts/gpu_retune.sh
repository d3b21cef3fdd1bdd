# Re-tune the backward's knobs under the pair multicast (interleaved A/B at c4 and N = 32K).
set -x
V=paper_2405_15780_b200/variants
L=paper_2405_15780_b200/libulysses_attn.so
timeout 1200 python scripts/ab.py --what bwd --rounds 3 --N 188416 --libs $L $V/libbox2off.so $V/libstag4.so $V/libstag64.so $V/libpoly0.so $V/libpoly8.so 2>&1 | tail -7
timeout 600 python scripts/ab.py --what bwd --rounds 5 --libs $L $V/libbox2off.so $V/libstag4.so $V/libstag64.so $V/libpoly0.so $V/libpoly8.so 2>&1 | tail -7
