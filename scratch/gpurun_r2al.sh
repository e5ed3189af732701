mkdir -p gpurun_out
for c in 2 3 4; do
  K=40; [ $c = 2 ] && K=4
  for m in 0 1 0 1; do KM_POST_PDL=$m timeout 300 python scratch/evcost.py $c $K 2>&1 | grep -v Warn | sed "s/^/pdl=$m /"; done
done > gpurun_out/r2am_evcost.log

