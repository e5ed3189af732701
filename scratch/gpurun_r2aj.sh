mkdir -p gpurun_out
for c in 2 3 4; do
  K=40; [ $c = 2 ] && K=4
  for m in "1 0" "2 0" "2 1" "1 0" "2 0" "2 1"; do set -- $m; KM_GRAPH_EVENTS=$1 KM_DONE_POLL=$2 timeout 300 python scratch/evcost.py $c $K 2>&1 | grep -v Warn | sed "s/^/poll=$2 /"; done
done > gpurun_out/r2aj_evcost.log
