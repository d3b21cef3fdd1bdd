cd paper_2405_15780_b200 && python build.py --variant dqearly UA_BWD_DQ_LATE=0 > /dev/null; cd ..
timeout 300 python -m pytest tests/test_bwd_gpu.py -m gpu -q -x 2>&1 | tail -2
V=paper_2405_15780_b200/variants
timeout 300 python scripts/ab.py --what bwd --rounds 8 --libs paper_2405_15780_b200/libulysses_attn.so $V/libdqearly.so
timeout 300 python scripts/ab.py --what bwd --rounds 4 --N 188416 --libs paper_2405_15780_b200/libulysses_attn.so $V/libdqearly.so
