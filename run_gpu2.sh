timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for c in 0 1 2 3 4 5 6 7; do
  echo "cfg $c: $(B2L_HASH_CFG=$c timeout 200 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu 2>&1 | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["roofline"]["frac"], d["verified"])')"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hash_seq -s 2 -c 1 -o gpurun_out/hash_r01_cfg0 python bench.py --steps 1 --warmup 2 --n-bufs 100000 --no-e2e --no-cpu > gpurun_out/ncu0.log 2>&1
tail -3 gpurun_out/ncu0.log
