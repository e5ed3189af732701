# row-part count sweep on the current build (step = stream + post with phase-0 combine)
for c in 4 3 2; do for p in default 16 20 24 28 40; do
  if [ $p = default ]; then unset KM_PARTS; else export KM_PARTS=$p; fi
  echo "C$c KM_PARTS=$p"; timeout 300 python scratch/evcost.py $c 30
done; unset KM_PARTS; done
