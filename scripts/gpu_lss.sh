o=gpurun_out
timeout 400 python bench.py --strategy lss --no-cpu-baseline --no-e2e > $o/cfg_lss_c4_p1.json 2> $o/lss1.err; echo lss1 rc=$?
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29677 bench.py --gpus 2 --strategy lss --no-cpu-baseline --no-e2e > $o/cfg_lss_c4_p2.json 2> $o/lss2.err; echo lss2 rc=$?
for f in cfg_lss_c4_p1 cfg_lss_c4_p2; do python -c "
import json; d=json.loads([l for l in open('$o/$f.json') if l.startswith('{')][-1]); print('$f', round(d['value'],1), d['ms_per_step'], d['config']['workload'])"; done
