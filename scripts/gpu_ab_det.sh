cd paper_2405_15780_b200
for v in "nosep UA_BWD_SEP_P=0" "dqp0 UA_BWD_DQ_POLY_MOD=0" "dqp2 UA_BWD_DQ_POLY_MOD=2" "dqp8 UA_BWD_DQ_POLY_MOD=8" "wsp2 UA_BWD_POLY_MOD=2" "wsp0 UA_BWD_POLY_MOD=0"; do set -- $v; python build.py --variant $1 $2 > /dev/null & done; wait
cd ..
timeout 120 python -m pytest tests/test_bwd_gpu.py -m gpu -q -x -k "deterministic" 2>&1 | tail -2
V=paper_2405_15780_b200/variants
timeout 300 python scripts/ab.py --det --what bwd --rounds 8 --libs paper_2405_15780_b200/libulysses_attn.so $V/libnosep.so $V/libdqp0.so $V/libdqp2.so $V/libdqp8.so $V/libwsp2.so $V/libwsp0.so
