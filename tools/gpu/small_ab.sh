# small traces (C1 10k, C3 30k): threaded side chains (default) vs serial on one stream (B2L_OVERLAP_MIN)
for mode in default serial; do
  if [ $mode = serial ]; then export B2L_OVERLAP_MIN=100000000; fi
  echo "== $mode"
  timeout -k 5 300 python tools/time_analysis.py --device --config c2 --n 10000 --iters 60 2>&1 | tail -1
  timeout -k 5 300 python tools/time_analysis.py --device --config c3 --n 10000 --iters 60 2>&1 | tail -1
  timeout -k 5 300 python tools/time_analysis.py --device --config c2 --n 100000 --iters 40 2>&1 | tail -1
done
