cd paper_2405_15780_b200 && python build.py --variant box2 UA_BWD_BOX2=1 > /dev/null; cd ..
V=paper_2405_15780_b200/variants
cp $V/libbox2.so /tmp/libbox2.so
timeout 300 python scripts/ab.py --what bwd --rounds 8 --libs paper_2405_15780_b200/libulysses_attn.so $V/libbox2.so
timeout 300 python scripts/ab.py --what bwd --rounds 4 --N 188416 --libs paper_2405_15780_b200/libulysses_attn.so $V/libbox2.so
