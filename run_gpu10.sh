B2L_TRACE=1 timeout 300 python tools/time_analysis.py --device --iters 4 2>&1 | tail -16
timeout 300 python tools/time_analysis.py --device --iters 8 2>&1 | tail -5
timeout 300 python tools/time_analysis.py --iters 5 2>&1 | tail -3
timeout 600 python -m pytest tests/test_analysis_gpu.py -x -q 2>&1 | tail -2
