# UA_BWD_DQ_LATE re-checked under the pair multicast (interleaved A/B at c4 and N = 32K).
V=paper_2405_15780_b200/variants
L=paper_2405_15780_b200/libulysses_attn.so
timeout 900 python scripts/ab.py --what bwd --rounds 4 --N 188416 --libs $L $V/libdqlate0.so 2>&1 | tail -2
timeout 400 python scripts/ab.py --what bwd --rounds 6 --libs $L $V/libdqlate0.so 2>&1 | tail -2
