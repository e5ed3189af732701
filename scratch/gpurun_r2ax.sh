mkdir -p gpurun_out
for r in 1 2; do
timeout 300 python scratch/dist_c4.py 2>&1 | grep -v Warn | sed 's/^/nacc4 /'
cp paper_2008_05171_b200/libkmedoids.so /tmp/lib4.so; cp scratch/libs/libkm_nacc2.so paper_2008_05171_b200/libkmedoids.so
timeout 300 python scratch/dist_c4.py 2>&1 | grep -v Warn | sed 's/^/nacc2 /'
cp /tmp/lib4.so paper_2008_05171_b200/libkmedoids.so
done > gpurun_out/r2ax_dist.log
