# C2: D kept in L2 (evict_normal) vs streamed evict_first
mkdir -p gpurun_out
for mb in 0 112; do
  KM_L2_KEEP_MB=$mb KM_STEP_PROF=1 timeout 300 python scratch/stepprof.py 2 100 > gpurun_out/r2af_stepprof_c2_keep$mb.log 2>&1
  KM_L2_KEEP_MB=$mb timeout 300 python bench.py --config 2 --warmup 3 --steps 5 --no-fasterpam --no-dissimilarity --no-clara --no-cpu-baseline > gpurun_out/r2af_bench_c2_keep$mb.log 2>&1
done
echo done
