timeout 900 python -m pytest tests/test_hash_gpu.py -q -x 2>&1 | grep -E "^E  |passed|failed" | head -20
timeout 300 python tools/bench_configs.py --configs c3 2>&1 | head -1
