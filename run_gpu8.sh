CUDA_LAUNCH_BLOCKING=1 timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python tools/sanitize_small.py 100000 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_analysis_gpu.py -x -q 2>&1 | tail -3
timeout 300 python tools/time_analysis.py --device --iters 6
timeout 300 python tools/time_analysis.py --device --config c4 --n 10000000 --iters 4
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ana_launches3.csv python tools/time_analysis.py --device --iters 2 > /dev/null 2>&1
