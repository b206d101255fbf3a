timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_hash_planes -c 1 -o gpurun_out/k2_v5 -f python tools/bench_configs.py --configs c3 --c3-buffers 1 > /dev/null 2>&1
ls gpurun_out
