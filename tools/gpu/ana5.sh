timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "^E  |passed|failed" | head -20
for cfg in "c2 1000000 40" "c2 10000000 12" "c4 10000000 12"; do
  set -- $cfg
  timeout 600 python tools/time_analysis.py --device --config $1 --n $2 --iters $3 2>&1 | tail -1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c2_10000000.csv python tools/time_analysis.py --device --config c2 --n 10000000 --iters 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launch_c2_10000000.csv 2 12
