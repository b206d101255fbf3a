# arena check: analysis parity subset, scratch-allocation trace, steady-state timing
timeout 900 python -m pytest tests -m gpu -x -q -k "analysis or savings or standalone or reports or sharded or capture" 2>&1 | tail -2
for cfg in "c2 10000" "c2 1000000" "c2 10000000" "c4 10000000"; do
  set -- $cfg
  B2L_TRACE=1 timeout 300 python tools/time_analysis.py --device --config $1 --n $2 --iters 3 2>&1 | grep -E "arena" | tail -2
  B2L_TRACE=1 timeout 300 python tools/time_analysis.py --config $1 --n $2 --iters 3 2>&1 | grep -E "savings arena" | tail -1
done
for cfg in "c2 10000 20" "c2 1000000 16" "c2 10000000 6" "c4 10000000 6" "c2 100000000 3"; do
  set -- $cfg
  timeout 600 python tools/time_analysis.py --device --config $1 --n $2 --iters $3 2>&1 | tail -1
done
