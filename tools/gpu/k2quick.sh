# K2 tests + timing (single buffers and the C3 16 x 256 MiB call)
timeout -k 5 300 python -m pytest tests/test_hash_gpu.py -q -x -k "k2 or large or routing" 2>&1 | tail -1
timeout -k 5 200 python tools/k2_time.py $((256<<20)) $((16<<20)) $((1<<20))
