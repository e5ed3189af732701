mkdir -p gpurun_out
KM_STEP_PROF=1 timeout 300 python scratch/fp2prof.py 3 30 > gpurun_out/r2ar_fp2prof_c3.log 2>&1
KM_STEP_PROF=1 timeout 300 python scratch/fp2prof.py 5 10 > gpurun_out/r2ar_fp2prof_c5.log 2>&1

