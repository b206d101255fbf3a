timeout 900 python tools/bench_configs.py > gpurun_out/configs_r01.jsonl 2> gpurun_out/configs_r01.err; cat gpurun_out/configs_r01.jsonl; tail -3 gpurun_out/configs_r01.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_hash_planes -c 1 -o gpurun_out/k2_r01 python tools/bench_configs.py --configs c3 --c3-buffers 1 > /dev/null 2>&1
ls gpurun_out | tail -3
