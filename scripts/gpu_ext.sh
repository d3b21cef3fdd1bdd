# Backward with -lse / -Delta as an extra MMA K step (UA_BWD_EXT): parity, then interleaved A/B.
set -x
mkdir -p gpurun_out
V=paper_2405_15780_b200/variants
L=paper_2405_15780_b200/libulysses_attn.so
export UA_PARITY_LOG=gpurun_out/parity_ext.jsonl
rm -f $UA_PARITY_LOG
timeout 1200 python -m pytest tests/test_bwd_gpu.py tests/test_layout_gpu.py tests/test_lss_sim_gpu.py -m gpu -q -x -k "not full_size and not c3_p8 and not c4_p8" > gpurun_out/pytest_ext.log 2>&1; echo pytest rc=$?
tail -4 gpurun_out/pytest_ext.log
unset UA_PARITY_LOG
timeout 400 python scripts/ab.py --what bwd --rounds 8 --libs $L $V/libext0.so $V/libextbox2.so 2>&1 | tail -4
timeout 700 python scripts/ab.py --what bwd --rounds 4 --N 188416 --libs $L $V/libext0.so $V/libextbox2.so 2>&1 | tail -4
timeout 300 python scripts/ab.py --what bwd --rounds 6 --N 8192 --H 16 --D 64 --libs $L $V/libext0.so 2>&1 | tail -3
timeout 300 python scripts/ab.py --what bwd --rounds 6 --N 32768 --H 16 --D 32 --libs $L $V/libext0.so 2>&1 | tail -3
timeout 700 python scripts/ab.py --what bwd --det --rounds 3 --N 188416 --libs $L $V/libdetslots0.so 2>&1 | tail -3
timeout 300 python scripts/ab.py --what bwd --det --rounds 6 --libs $L $V/libdetslots0.so 2>&1 | tail -3
