# K2 v7 (streamed groups) vs v6: parity tests, C3 timing
timeout 600 python -m pytest tests/test_hash_gpu.py tests/test_capture.py -q -x -k "k2 or single_buffer or device_copy or large" 2>&1 | tail -2
timeout 300 python bench.py --no-cpu --no-large --no-e2e --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); [print(c['name'], c['value'], c.get('ms_per_buffer'), c.get('verified')) for c in d['configs'] if c['name']=='C3-hash']"
B2L_K2=6 timeout 300 python bench.py --no-cpu --no-large --no-e2e --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); [print('v6', c['name'], c['value'], c.get('ms_per_buffer'), c.get('verified')) for c in d['configs'] if c['name']=='C3-hash']"
