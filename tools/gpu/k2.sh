timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "^E  |passed|failed" | head -20
timeout 300 python tools/bench_configs.py --configs c3 2>&1 | head -1
for cfg in "c2 10000000 6" "c4 10000000 6"; do
  set -- $cfg
  timeout 600 python tools/time_analysis.py --device --config $1 --n $2 --iters $3 2>&1 | tail -1
done
