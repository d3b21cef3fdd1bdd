cd paper_2405_15780_b200
for v in "p0 UA_BWD_POLY_MOD=0" "p8 UA_BWD_POLY_MOD=8" "st8 UA_BWD_STAGGER=8" "st32 UA_BWD_STAGGER=32" "kvs UA_BWD_KV_TMEM=0"; do set -- $v; python build.py --variant $1 $2 > /dev/null & done; wait
cd ..
V=paper_2405_15780_b200/variants
timeout 400 python scripts/ab.py --what bwd --rounds 8 --libs paper_2405_15780_b200/libulysses_attn.so $V/libp0.so $V/libp8.so $V/libst8.so $V/libst32.so $V/libkvs.so
timeout 400 python scripts/ab.py --what bwd --rounds 4 --N 188416 --libs paper_2405_15780_b200/libulysses_attn.so $V/libp0.so $V/libp8.so
