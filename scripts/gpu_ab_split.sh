cd paper_2405_15780_b200 && python build.py --variant nosplit UA_BWD_EW_SPLIT=0 > /dev/null; cd ..
timeout 60 python scripts/dbg_det.py 1024 2 64 | tail -1
timeout 400 python -m pytest tests/test_bwd_gpu.py tests/test_fwd_gpu.py -m gpu -q -x 2>&1 | tail -2
V=paper_2405_15780_b200/variants
timeout 300 python scripts/ab.py --what bwd --rounds 8 --libs paper_2405_15780_b200/libulysses_attn.so $V/libnosplit.so
timeout 300 python scripts/ab.py --what bwd --rounds 3 --N 188416 --libs paper_2405_15780_b200/libulysses_attn.so $V/libnosplit.so
