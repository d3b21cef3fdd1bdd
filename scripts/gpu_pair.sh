# Paired CTAs sharing Q / dO via TMA multicast (UA_BWD_PAIR): parity, then interleaved A/B.
set -x
mkdir -p gpurun_out
V=paper_2405_15780_b200/variants
L=paper_2405_15780_b200/libulysses_attn.so
timeout 600 python -m pytest tests/test_bwd_gpu.py -m gpu -q -x -k "not full_size" > gpurun_out/pytest_pair.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_pair.log
timeout 400 python scripts/ab.py --what bwd --rounds 8 --libs $L $V/libpair0.so 2>&1 | tail -3
timeout 600 python scripts/ab.py --what bwd --rounds 4 --N 188416 --libs $L $V/libpair0.so 2>&1 | tail -3
timeout 300 python scripts/ab.py --what bwd --rounds 4 --N 65536 --H 16 --D 128 --libs $L $V/libpair0.so 2>&1 | tail -3
timeout 300 python scripts/ab.py --what bwd --rounds 4 --N 8192 --H 16 --D 64 --libs $L $V/libpair0.so 2>&1 | tail -3
