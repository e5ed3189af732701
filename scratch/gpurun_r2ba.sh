mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2ba_1.csv python scratch/clara_repro.py 1 1 > gpurun_out/r2ba_ncu_ns1.log 2>&1; echo "ncu ns=1 rc=$?"
timeout 600 ncu --graph-profiling graph --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2ba_2.csv python scratch/clara_repro.py 1 5 > gpurun_out/r2ba_ncu_graph.log 2>&1; echo "ncu graph-profiling rc=$?"
KM_LIBRARY=checked timeout 600 python scratch/clara_repro.py 3 5 > gpurun_out/r2ba_checked.log 2>&1; echo "checked rc=$?"
