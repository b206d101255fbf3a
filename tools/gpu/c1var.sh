for v in 11 14 15; do echo "variant $v"; B2L_HASH_CFG=$v timeout 300 python tools/bench_configs.py --configs c1 2>&1 | head -1; done
timeout 900 python -m pytest tests/test_hash_gpu.py -q -x 2>&1 | grep -E "^E  |passed|failed" | head
