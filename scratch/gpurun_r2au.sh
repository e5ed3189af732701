mkdir -p gpurun_out
for P in 0 12 20 30 40 60; do
  if [ $P = 0 ]; then unset KM_PARTS; else export KM_PARTS=$P; fi
  timeout 300 python scratch/evcost.py 2 4 2>&1 | grep -v Warn | sed "s/^/P=$P /"
done > gpurun_out/r2au_c2_parts.log
