timeout 300 python -m pytest tests/test_hash_gpu.py -x -q 2>&1 | tail -3
timeout 300 python tools/bench_configs.py --configs c1,c3 2>&1 | grep GB
for c in 6 11 12 13; do echo "cfg $c: $(B2L_HASH_CFG=$c timeout 120 python tools/bench_configs.py --configs c1 2>&1 | grep GB | cut -c1-140)"; done
