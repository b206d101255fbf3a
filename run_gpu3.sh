timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for c in 0 1 2 3 4 5 6 7 8 9 10; do
  echo "cfg $c: $(B2L_HASH_CFG=$c timeout 200 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu 2>&1 | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["roofline"]["frac"], d["verified"])')"
done
