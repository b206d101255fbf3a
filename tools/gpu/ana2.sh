# analysis parity tests + steady-state timing + launch lists (1M, 10M C2)
timeout 900 python -m pytest tests -m gpu -x -q -k "analysis or standalone or reports or sharded or ingest" 2>&1 | tail -5
for cfg in "c2 1000000 12" "c2 10000000 6" "c4 10000000 6" "c2 100000000 4"; do
  set -- $cfg
  timeout 600 python tools/time_analysis.py --device --config $1 --n $2 --iters $3 2>&1 | tail -2
done
for n in 1000000 10000000; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c2_$n.csv python tools/time_analysis.py --device --config c2 --n $n --iters 2 > /dev/null 2>&1
done
