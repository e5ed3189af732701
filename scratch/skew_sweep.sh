#!/bin/bash
# stream kernel time vs part-size tilt (KM_PART_SKEW, 16ths) and row parts P
cd $GRAFT_REPO_ROOT
KM_PART_SKEW=12 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fasterpam.py -x -q > gpurun_out/pytest_skew.log 2>&1; echo "skew12 parity rc=$?"
run() { # cfg P skew
  export KM_PART_SKEW=$3; if [ $2 = 0 ]; then unset KM_PARTS; else export KM_PARTS=$2; fi
  python bench.py --config $1 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-fasterpam --no-dissimilarity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg $1 P=$2 skew=$3', round(d['ms_per_step'],4), round(r['kernel_ms'],4), round(r['frac'],4), round(r['frac_of_read_only_peak'],4), d['clocks']['sm_mhz'], flush=True)"
}
for sk in 0 4 8 12 15; do run 4 0 $sk; done
for sk in 8 12; do for P in 31 39 63; do run 4 $P $sk; done; done
for sk in 0 6 12; do run 3 0 $sk; done
for sk in 0 6 12; do run 5 0 $sk; done
