# one iteration of an analysis change: GPU analysis tests, the broad sweep, warm timings
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "analysis or savings or standalone or reports or sharded or capture" 2>&1 | tail -2
bash tools/gpu/sweep.sh 2>&1 | tail -2
for cfg in "c2 10000 30" "c3 30000 30" "c2 1000000 16" "c4 1000000 16" "c2 10000000 8" "c4 10000000 8"; do
  set -- $cfg
  timeout 600 python tools/time_analysis.py --device --config $1 --n $2 --iters $3 2>&1 | tail -1
done
