for cfg in "c2 1000000 8" "c2 10000000 4"; do
  set -- $cfg
  B2L_TRACE=1 timeout 600 python tools/time_analysis.py --device --config $1 --n $2 --iters $3 2>&1 | tail -24
done
for cfg in "c2 1000000 12" "c2 10000000 6"; do
  set -- $cfg
  timeout 600 python tools/time_analysis.py --device --config $1 --n $2 --iters $3 2>&1 | tail -1
done
