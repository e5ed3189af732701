#!/bin/bash
# stream kernel time vs row parts P and consumer variant (seg / seg2)
cd $GRAFT_REPO_ROOT
KM_STREAM=seg2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_seg2.log 2>&1; echo "seg2 parity rc=$?"
run() { # cfg P variant
  export KM_STREAM=$3; if [ $2 = 0 ]; then unset KM_PARTS; else export KM_PARTS=$2; fi
  python bench.py --config $1 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-fasterpam 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $1 P=$2 $3', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], flush=True)"
}
for v in seg seg2; do for P in 31 39 47 55 63 79; do run 4 $P $v; done; done
for v in seg seg2; do for P in 0 79 100 130 160; do run 3 $P $v; done; done
for v in seg seg2; do for P in 0 16 20 24 32; do run 5 $P $v; done; done
