# Two-phase backward elementwise stage (UA_BWD_TWOPHASE) vs the one-pass stage: backward parity
# tests, then interleaved A/B at c4 and N = 32K.
V=paper_2405_15780_b200/variants
L=paper_2405_15780_b200/libulysses_attn.so
timeout 600 python -m pytest -x -q tests/test_bwd_gpu.py -k "not full_size" 2>&1 | tail -2
timeout 600 python scripts/ab.py --what bwd --rounds 4 --N 188416 --libs $L $V/libtwoph0.so 2>&1 | tail -2
timeout 300 python scripts/ab.py --what bwd --rounds 6 --libs $L $V/libtwoph0.so 2>&1 | tail -2
