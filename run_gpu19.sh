timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_r01d.json 2> gpurun_out/bench_r01d.err; tail -c 3500 gpurun_out/bench_r01d.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r01.json 2>&1; tail -c 1500 gpurun_out/bench_ref_r01.json
timeout 900 python tools/bench_configs.py > gpurun_out/configs_r01b.jsonl 2> gpurun_out/configs_r01b.err; cat gpurun_out/configs_r01b.jsonl
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ana_launches5.csv python tools/time_analysis.py --device --iters 2 > /dev/null 2>&1
