timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k_hash_warp" --launch-skip 3 -c 1 -o gpurun_out/prof_c1_warp -f python tools/bench_configs.py --configs c1 > /dev/null 2>&1
ls gpurun_out/prof_c1_warp*
