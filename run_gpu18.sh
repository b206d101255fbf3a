B2L_TRACE=1 timeout 300 python tools/time_analysis.py --device --n 20000000 --iters 2 2>&1 | tail -16
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ana_launches_20m.csv python tools/time_analysis.py --device --n 20000000 --iters 1 > /dev/null 2>&1
