timeout 900 python -m pytest tests -m gpu -x -q -k "analysis or savings or standalone or reports or sharded or capture" 2>&1 | tail -2
for cfg in "c2 10000 30" "c2 1000000 16" "c2 10000000 6" "c2 100000000 5"; do
  set -- $cfg
  timeout 600 python tools/time_analysis.py --device --config $1 --n $2 --iters $3 2>&1 | tail -1
done
