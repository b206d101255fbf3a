# analysis parity subset + steady-state device-resident timings (C2 10k/1M/10M, C4 1M/10M)
timeout 900 python -m pytest tests/test_analysis_gpu.py tests/test_parity_configs_gpu.py tests/test_reports_gpu.py tests/test_standalone_gpu.py -q -x -m gpu 2>&1 | tail -3
for cfg in "c2 10000" "c2 1000000" "c2 10000000" "c4 1000000" "c4 10000000"; do
  set -- $cfg
  timeout 300 python tools/time_analysis.py --device --config $1 --n $2 --iters 16 2>&1 | grep MEDIAN
done
