# side-chain threads vs one stream at small / medium sizes
for env in "" "B2L_OVERLAP_MIN=999999999" "B2L_SIDE_MIN=999999999" "B2L_OVERLAP_MIN=999999999 B2L_SIDE_MIN=999999999"; do
  echo "== $env"
  for cfg in "c2 10000 40" "c2 100000 30" "c2 1000000 30"; do
    set -- $cfg; env $env timeout 300 python tools/time_analysis.py --device --config $1 --n $2 --iters $3 2>&1 | tail -1
  done
done
