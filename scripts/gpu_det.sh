# deterministic-backward checks (GPUs visible: 1 or more)
timeout 900 python -m pytest tests/test_bwd_gpu.py -m gpu -q -k "deterministic" 2>&1 | tail -15
timeout 1200 python -m pytest tests/test_multigpu.py -m gpu -q -k "deterministic" 2>&1 | tail -15
