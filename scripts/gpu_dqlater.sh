# UA_BWD_DQ_LATER (the dQ GEMM of tile T behind tile T+1's first half) vs DQ_LATE alone: backward
# parity tests on the LATER build (swapped in for the run), then interleaved A/B.
V=paper_2405_15780_b200/variants
L=paper_2405_15780_b200/libulysses_attn.so
cp $L /tmp/ua_base.so && cp $V/liblater1.so $L
timeout 600 python -m pytest -x -q tests/test_bwd_gpu.py tests/test_fuzz_gpu.py -k "not full_size" 2>&1 | tail -2
cp /tmp/ua_base.so $L
timeout 600 python scripts/ab.py --what bwd --rounds 4 --N 188416 --libs $L $V/liblater1.so 2>&1 | tail -2
timeout 300 python scripts/ab.py --what bwd --rounds 6 --libs $L $V/liblater1.so 2>&1 | tail -2
timeout 300 python scripts/ab.py --what bwd --rounds 6 --N 32768 --H 16 --D 32 --libs $L $V/liblater1.so 2>&1 | tail -2
