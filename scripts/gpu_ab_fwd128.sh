cd paper_2405_15780_b200 && python build.py --variant poly128 UA_FWD_POLY_MAXD=128 > /dev/null; cd ..
V=paper_2405_15780_b200/variants
timeout 300 python scripts/ab.py --what fwd --rounds 8 --N 65536 --H 16 --D 128 --libs paper_2405_15780_b200/libulysses_attn.so $V/libpoly128.so
timeout 300 python scripts/ab.py --what fwd --rounds 8 --N 32768 --H 32 --D 128 --libs paper_2405_15780_b200/libulysses_attn.so $V/libpoly128.so
