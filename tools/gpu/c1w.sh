timeout 900 python -m pytest tests/test_hash_gpu.py tests/test_capture.py -q 2>&1 | grep -E "^E  |passed|failed" | head
timeout 300 python tools/bench_configs.py --configs c1 2>&1 | head -1
B2L_HASH_CFG=11 timeout 300 python tools/bench_configs.py --configs c1 2>&1 | head -1
