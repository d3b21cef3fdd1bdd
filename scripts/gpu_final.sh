o=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_multigpu.py 2>&1 | tail -2
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q -x -k "p_way and 4096 and 8 and 64 and not lss" 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" 2>&1 | tail -1
timeout 600 python bench.py > $o/final_p1.json 2> $o/final_p1.err; echo bench1 rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29655 bench.py --gpus 2 > $o/final_p2.json 2> $o/final_p2.err; echo bench2 rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29656 bench.py --gpus 2 --impl reference --steps 3 --warmup 3 > $o/final_ref_p2.json 2> $o/final_ref_p2.err; echo ref2 rc=$?
for f in final_p1 final_p2 final_ref_p2; do tail -c 600 $o/$f.json; echo; done
