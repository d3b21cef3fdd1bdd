# Backward elementwise stage in 16x32bx2 TMEM shapes (UA_BWD_EW16) vs 32x32b: parity tests, then
# interleaved A/B at c4, N = 32K, c3 (D = 128) and D = 32.
set -x
V=paper_2405_15780_b200/variants
L=paper_2405_15780_b200/libulysses_attn.so
timeout 1200 python -m pytest -x -q tests/test_bwd_gpu.py tests/test_fuzz_gpu.py tests/test_lss_sim_gpu.py 2>&1 | tail -3
timeout 1200 python scripts/ab.py --what bwd --rounds 4 --N 188416 --libs $L $V/libnoew16.so 2>&1 | tail -3
timeout 600 python scripts/ab.py --what bwd --rounds 6 --libs $L $V/libnoew16.so 2>&1 | tail -3
timeout 600 python scripts/ab.py --what bwd --rounds 4 --N 65536 --H 16 --D 128 --libs $L $V/libnoew16.so 2>&1 | tail -3
timeout 600 python scripts/ab.py --what bwd --rounds 6 --N 32768 --H 16 --D 32 --libs $L $V/libnoew16.so 2>&1 | tail -3
