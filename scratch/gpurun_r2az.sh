mkdir -p gpurun_out
timeout 300 python scratch/clara_repro.py 5 > gpurun_out/r2az_plain.log 2>&1; echo "plain rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2az_l1.csv python scratch/clara_repro.py 1 > gpurun_out/r2az_ncu_head.log 2>&1; echo "ncu head rc=$?"
cp paper_2008_05171_b200/libkmedoids.so /tmp/head.so; cp scratch/libs/libkmedoids_b11.so paper_2008_05171_b200/libkmedoids.so
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2az_l2.csv python scratch/clara_repro.py 1 > gpurun_out/r2az_ncu_b11.log 2>&1; echo "ncu b11 rc=$?"
cp /tmp/head.so paper_2008_05171_b200/libkmedoids.so
