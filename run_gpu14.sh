timeout 1200 python -m pytest tests/test_analysis_gpu.py -x -q -m gpu 2>&1 | tail -2
timeout 300 python tools/time_analysis.py --device --iters 6 2>&1 | tail -3
timeout 300 python tools/time_analysis.py --device --config c4 --n 10000000 --iters 4 2>&1 | tail -2
