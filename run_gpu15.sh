timeout 180 python -m pytest tests/test_hash_gpu.py -x -q -k "k2" 2>&1 | tail -15
