cd paper_2405_15780_b200 && python build.py --variant nobatch UA_BWD_LDBATCH=0 > /dev/null; cd ..
timeout 300 python -m pytest tests/test_bwd_gpu.py -m gpu -q -x 2>&1 | tail -2
V=paper_2405_15780_b200/variants
timeout 300 python scripts/ab.py --what bwd --rounds 8 --libs paper_2405_15780_b200/libulysses_attn.so $V/libnobatch.so
timeout 300 python scripts/ab.py --what bwd --rounds 3 --N 188416 --libs paper_2405_15780_b200/libulysses_attn.so $V/libnobatch.so
timeout 300 python scripts/ab.py --what bwd --rounds 6 --N 65536 --H 16 --D 128 --libs paper_2405_15780_b200/libulysses_attn.so $V/libnobatch.so
