# per-phase step profile (KM_STEP_PROF) at C2/C3/C4 + every config at HEAD
mkdir -p gpurun_out
for c in 2 3 4; do
  KM_STEP_PROF=1 timeout 300 python scratch/stepprof.py $c 100 > gpurun_out/r2ae_stepprof_c$c.log 2>&1
done
bash scratch/all_configs.sh > gpurun_out/r2ae_all_configs.log 2>&1
echo done
