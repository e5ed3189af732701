# FastPAM2 launch lists at C3 and C5 (per-kernel durations; cold-cache, serialised)
mkdir -p gpurun_out
for c in 3 5; do
CMD="python bench.py --config $c --variant fastpam2 --steps 3 --warmup 3 --no-e2e --no-fasterpam --no-dissimilarity --no-cpu-baseline --no-clara"
timeout 600 $CMD > gpurun_out/r2ag_plain_c$c.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2ag_launches_c$c.csv $CMD > gpurun_out/r2ag_ncu_c$c.log 2>&1
echo "c$c rc=$?"
done
