#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q 2>&1 | tail -3
timeout 300 python bench.py --sharded --steps 30 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sharded x1', round(d['ms_per_step'],4), d['roofline']['kernel_ms'], d['init'], d['e2e']['n_iter'], d['e2e']['td'], d['e2e']['seconds'])"
timeout 300 python bench.py --sharded --config 5 --variant fastpam2 --steps 5 --warmup 2 --no-e2e 2>&1 | tail -1 | cut -c1-300
