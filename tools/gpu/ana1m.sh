# analysis parity subset + steady-state timing (1M / 10M C2) + the 1M launch list
timeout 900 python -m pytest tests -m gpu -x -q -k "analysis or savings or standalone or reports" 2>&1 | tail -2
for cfg in "c2 1000000 16" "c2 10000000 6" "c4 10000000 6"; do
  set -- $cfg
  timeout 600 python tools/time_analysis.py --device --config $1 --n $2 --iters $3 2>&1 | tail -1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c2_1000000.csv python tools/time_analysis.py --device --config c2 --n 1000000 --iters 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launch_c2_1000000.csv 2 14
