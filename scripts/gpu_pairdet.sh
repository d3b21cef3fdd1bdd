# Pair multicast for the dQ-less (deterministic) KV-stationary kernel: parity, bitwise P-way, A/B.
set -x
V=paper_2405_15780_b200/variants
L=paper_2405_15780_b200/libulysses_attn.so
timeout 900 python -m pytest tests/test_bwd_gpu.py tests/test_layout_gpu.py tests/test_fuzz_gpu.py -m gpu -q -x -k "deterministic or sim_ulysses_bwd or fuzz" > gpurun_out/pytest_pairdet.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_pairdet.log
timeout 1200 python scripts/ab.py --what bwd --det --rounds 3 --N 188416 --libs $L $V/libpairdet0.so 2>&1 | tail -3
timeout 600 python scripts/ab.py --what bwd --det --rounds 6 --libs $L $V/libpairdet0.so 2>&1 | tail -3
