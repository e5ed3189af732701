# part-output L2 store policy sweep (KM_PART_POL 0 last / 1 normal / 2 first), C4 and C3
for c in 4 3; do for p in 0 1 2 0; do
  echo "KM_PART_POL=$p"; KM_PART_POL=$p timeout 300 python scratch/evcost.py $c 30
done; done
