# Forward column-split kernel: K / V ring depth 4 (new default) vs 3 / 5, after the forward parity tests.
V=paper_2405_15780_b200/variants
L=paper_2405_15780_b200/libulysses_attn.so
timeout 600 python -m pytest -x -q tests/test_fwd_gpu.py tests/test_fuzz_gpu.py 2>&1 | tail -2
timeout 600 python scripts/ab.py --what fwd --rounds 6 --N 188416 --libs $L $V/libfst3.so $V/libfst5.so 2>&1 | tail -3
timeout 300 python scripts/ab.py --what fwd --rounds 8 --libs $L $V/libfst3.so $V/libfst5.so 2>&1 | tail -3
timeout 300 python scripts/ab.py --what fwd --rounds 8 --N 32768 --H 16 --D 32 --libs $L $V/libfst3.so $V/libfst5.so 2>&1 | tail -3
