# round-2 closing evidence: GPU tests, smoke, both bench arms, the hash launch list, ncu --set full
# of K2 (one 16 x 256 MiB hash_large_many launch and one single-buffer launch), of the C1 split-pair
# batch and of the C2 hash kernel -- everything into gpurun_out/ (summaries copied to profiles/ after)
set -x
cat > /tmp/k2many.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch
from paper_2601_12713_b200 import hashing as H
k, n = 16, 256 << 20
t = torch.randint(0, 256, (k * n,), dtype=torch.uint8, device="cuda")
out = torch.empty(k, dtype=torch.int64, device="cuda")
ptrs = [t.data_ptr() + i * n for i in range(k)]
for _ in range(3): H.hash_large_many(ptrs, [n] * k, out.data_ptr())
torch.cuda.synchronize()
PY
timeout -k 10 900 ncu --set full --import-source on --clock-control none -k regex:k_hash_planes -s 2 -c 1 -o gpurun_out/k2_many_full -f python /tmp/k2many.py > gpurun_out/k2many_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/k2_many_full.ncu-rep gpurun_out/k2_many_ncu_summary.json --algo-bytes 4294967296 > /dev/null 2>&1
cp gpurun_out/k2_many_ncu_summary.json profiles/ 2>/dev/null
timeout -k 10 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout -k 10 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout -k 10 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout -k 10 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/hash_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-large --no-configs > gpurun_out/bench_ncu.log 2>&1
bash tools/gpu/k2ncu.sh > /dev/null 2>&1
sed -n '/^cat > \/tmp\/c1t.py/,/^PY$/p' tools/gpu/c1split.sh > /tmp/mk.sh; bash /tmp/mk.sh
timeout -k 10 600 ncu --set full --import-source on --clock-control none -k regex:k_hash_warp -s 3 -c 1 -o gpurun_out/c1_split -f python /tmp/c1t.py > /dev/null 2>&1
timeout -k 10 600 ncu --set full --clock-control none -k regex:k_hash_coop -s 2 -c 1 -o gpurun_out/hash_c2 -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-large --no-configs > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/c1_split.ncu-rep gpurun_out/c1_split_ncu_summary.json > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/hash_c2.ncu-rep gpurun_out/hash_c2_ncu_summary.json > /dev/null 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log
python - <<'PY'
import json
for f in ('gpurun_out/bench.json', 'gpurun_out/bench_ref.json'):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'unparsable', e); continue
    print(f, d.get('value'), d.get('unit'), 'e2e', (d.get('e2e') or {}).get('value'))
    a = d.get('analysis') or {}
    print('  analysis', a.get('value'), a.get('verified'), (a.get('e2e') or {}).get('value'))
    for c in d.get('configs') or []:
        print('  ', c.get('name'), c.get('value'), c.get('unit'), 'ver', c.get('verified'), 'e2e', (c.get('e2e') or {}).get('value'), 'cpu', (c.get('cpu_baseline') or {}).get('value'))
PY
