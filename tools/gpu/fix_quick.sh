timeout 900 python -m pytest tests -m gpu -x -q -k "sort or analysis or savings or standalone or reports or sharded" 2>&1 | tail -2
timeout 600 python tools/sanitize_small.py 3000 --no-sharded 2>&1 | tail -3
for cfg in "c2 10000 30" "c2 1000000 16" "c4 1000000 12" "c4 10000000 6"; do
  set -- $cfg
  timeout 600 python tools/time_analysis.py --device --config $1 --n $2 --iters $3 2>&1 | tail -1
done
