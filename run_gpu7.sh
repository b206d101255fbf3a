timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python tools/time_analysis.py --device --iters 4
timeout 300 python tools/time_analysis.py --device --config c4 --n 10000000 --iters 3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ana_launches.csv python tools/time_analysis.py --device --iters 2 > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err; tail -c 4000 gpurun_out/bench_r01b.json
