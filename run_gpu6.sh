timeout 900 python -m pytest tests/test_analysis_gpu.py -x -q 2>&1 | tail -5
timeout 300 python tools/time_analysis.py
