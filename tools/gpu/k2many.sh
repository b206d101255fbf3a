# K2 multi-buffer launches: tests, then a (jobs, teams) sweep on 16 x 256 MiB (C3)
timeout 600 python -m pytest tests/test_hash_gpu.py -q -x -k "k2 or large or routing" 2>&1 | tail -2
K2_MANY=0 timeout 300 python tools/k2_time.py
for j in 1 2 4 8 16; do for t in 1 2 4; do
  B2L_K2_JOBS=$j B2L_K2_TEAMS=$t timeout 300 python tools/k2_time.py 0 2>&1 | grep many
done; done
