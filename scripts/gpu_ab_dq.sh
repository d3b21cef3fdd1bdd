cd paper_2405_15780_b200 && python build.py --variant g2 UA_BWD_DQ_GROUPS=2 > /dev/null; cd ..
timeout 60 python scripts/dbg_det.py 2 2 64 | tail -1
timeout 300 python -m pytest tests/test_bwd_gpu.py -m gpu -q -x -k "deterministic" 2>&1 | tail -2
V=paper_2405_15780_b200/variants
timeout 300 python scripts/ab.py --det --what bwd --rounds 8 --libs paper_2405_15780_b200/libulysses_attn.so $V/libg2.so
timeout 300 python scripts/ab.py --det --what bwd --rounds 3 --N 188416 --libs paper_2405_15780_b200/libulysses_attn.so $V/libg2.so
