timeout 900 python -m pytest tests/test_sort_gpu.py -q 2>&1 | grep -E "^E  |passed|failed" | head -20
for cfg in "c2 10000000 6" "c4 10000000 6"; do
  set -- $cfg
  B2L_TRACE=1 timeout 600 python tools/time_analysis.py --device --config $1 --n $2 --iters $3 2>&1 | tail -24
done
