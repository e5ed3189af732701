# final round-2 evidence at HEAD: every config, phase splits, default bench, launch list, ncu capture
mkdir -p gpurun_out
bash scratch/all_configs.sh > gpurun_out/r2ay_all_configs.log 2>&1
for c in 2 3 4; do KM_STEP_PROF=1 timeout 300 python scratch/stepprof.py $c 100 > gpurun_out/r2ay_stepprof_c$c.log 2>&1; done
KM_STEP_PROF=1 timeout 300 python scratch/fp2prof.py 3 30 > gpurun_out/r2ay_fp2prof_c3.log 2>&1
KM_STEP_PROF=1 timeout 300 python scratch/fp2prof.py 5 10 > gpurun_out/r2ay_fp2prof_c5.log 2>&1
timeout 900 python bench.py > gpurun_out/r2ay_bench.log 2>&1; echo "bench rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-fasterpam --no-dissimilarity --no-cpu-baseline --no-clara"
timeout 600 $CMD > gpurun_out/r2ay_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2ay_launches.csv python bench.py > gpurun_out/r2ay_ncu1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_swap_stream_seg2|k_fp1_post" -s 12 -c 2 -o gpurun_out/r2ay_prof $CMD > gpurun_out/r2ay_ncu2.log 2>&1
echo "rc=$?"
