# Forward D <= 64: deferred cross-half max exchange vs the blocking one (interleaved A/B), plus the
# forward parity tests on the new default.
set -x
V=paper_2405_15780_b200/variants
L=paper_2405_15780_b200/libulysses_attn.so
timeout 900 python -m pytest -x -q tests/test_fwd_gpu.py tests/test_fuzz_gpu.py tests/test_lss_sim_gpu.py tests/test_layout_gpu.py 2>&1 | tail -3
timeout 1200 python scripts/ab.py --what fwd --rounds 5 --N 188416 --libs $L $V/libnodefer.so 2>&1 | tail -3
timeout 600 python scripts/ab.py --what fwd --rounds 8 --libs $L $V/libnodefer.so 2>&1 | tail -3
timeout 600 python scripts/ab.py --what fwd --rounds 8 --N 32768 --D 32 --H 16 --libs $L $V/libnodefer.so 2>&1 | tail -3
