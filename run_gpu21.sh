timeout 300 python -m pytest tests/test_sharded.py -q -x -m gpu 2>&1 | tail -3
B2L_TRACE=1 timeout 300 python tools/time_analysis.py --device --n 100000000 --iters 3 2>&1 | grep -E "analyze|d2h|detectors|upload|validate|partition"
