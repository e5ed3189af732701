mkdir -p gpurun_out
for c in 2 3 4; do
  K=40; [ $c = 2 ] && K=4
  for ge in 1 2 0 1 2 0; do KM_GRAPH_EVENTS=$ge timeout 300 python scratch/evcost.py $c $K 2>&1 | grep -v Warn; done
done > gpurun_out/r2ai_evcost.log
