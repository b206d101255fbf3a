# analysis parity tests + steady-state timing at 1M / 10M (C2, C4) and 100M (C2)
timeout 900 python -m pytest tests -m gpu -x -q -k "analysis or standalone or reports or sharded or ingest" 2>&1 | tail -5
for cfg in "c2 1000000 12" "c2 10000000 6" "c4 10000000 6" "c2 100000000 4"; do
  set -- $cfg
  timeout 600 python tools/time_analysis.py --device --config $1 --n $2 --iters $3 2>&1 | tail -2
done
