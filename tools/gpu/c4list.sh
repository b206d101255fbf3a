timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c4_10M.csv python tools/time_analysis.py --device --config c4 --n 10000000 --iters 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launch_c4_10M.csv 2 25
