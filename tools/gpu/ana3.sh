# full GPU tests + steady-state timing + 10M launch list
timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -E "^E  |passed|failed" | head -30
for cfg in "c2 1000000 12" "c2 10000000 6" "c4 10000000 6" "c2 100000000 6"; do
  set -- $cfg
  timeout 600 python tools/time_analysis.py --device --config $1 --n $2 --iters $3 2>&1 | tail -2
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c2_10000000.csv python tools/time_analysis.py --device --config c2 --n 10000000 --iters 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launch_c2_10000000.csv 2 30
