mkdir -p gpurun_out
for c in 1 0 1 0; do KM_DIST_CENTER=$c timeout 300 python scratch/dist_c4.py 2>&1 | grep -v Warn; done > gpurun_out/r2av_dist.log
CMD="python scratch/dist_c4.py"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2av_dist_launches.csv $CMD > /dev/null 2>&1; echo rc=$?
