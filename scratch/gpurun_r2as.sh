mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2as_gputest.log 2>&1; echo "tests rc=$?"
KM_STEP_PROF=1 timeout 300 python scratch/fp2prof.py 3 30 > gpurun_out/r2as_fp2prof_c3.log 2>&1
KM_STEP_PROF=1 timeout 300 python scratch/fp2prof.py 5 10 > gpurun_out/r2as_fp2prof_c5.log 2>&1
for spec in "3 fastpam2 3 10" "5 fastpam2 3 10"; do
  set -- $spec
  timeout 600 python bench.py --config $1 --variant $2 --warmup $3 --steps $4 --no-fasterpam --no-dissimilarity --no-clara --no-cpu-baseline > gpurun_out/r2as_bench_c$1_$2.log 2>&1
done
