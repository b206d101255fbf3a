timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_r01c.json 2> gpurun_out/bench_r01c.err; tail -c 5000 gpurun_out/bench_r01c.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ana_launches4.csv python tools/time_analysis.py --device --iters 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_onesweep -s 10 -c 2 -o gpurun_out/onesweep_r01 python tools/time_analysis.py --device --iters 2 > /dev/null 2>&1
ls -la gpurun_out
