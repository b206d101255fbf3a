# C1 hash with and without the split pairs (+ digests vs the C oracle), then the hash GPU tests
cat > /tmp/c1t.py <<'PY'
import sys, os; sys.path.insert(0, ".")
import numpy as np, torch
from oracle import hash_ref
from paper_2601_12713_b200 import hash_device
dev = torch.device("cuda")
rng = np.random.default_rng(1)
lens = np.exp(rng.uniform(np.log(1024), np.log(1 << 20), 4000)).astype(np.int64)
if os.environ.get("ONE_LONG"): lens = np.full(2000, 1024, np.int64); lens[0] = 1 << 20
part = os.environ.get("PART")
if part:
    srt = np.sort(lens)[::-1]
    lens = np.concatenate([srt[:296], np.full(1000, 16)]) if part == "top" else np.concatenate([np.full(296, 16), srt[296:]])
n = lens.size
offs = np.zeros(n, np.int64); offs[1:] = np.cumsum((lens + 255) // 256 * 256)[:-1]
total = int(offs[-1] + lens[-1])
host = np.frombuffer(np.random.default_rng(5).bytes(total), np.uint8).copy()
slab = torch.from_numpy(host).to(dev)
o_d, l_d = torch.from_numpy(offs).to(dev), torch.from_numpy(lens).to(dev)
ptrs = o_d + slab.data_ptr()
order = torch.from_numpy(np.argsort(-lens, kind="stable").astype(np.int32)).to(dev)
out = torch.empty(n, dtype=torch.int64, device=dev)
for _ in range(3): hash_device(ptrs, l_d, out, order=order)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): hash_device(ptrs, l_d, out, order=order)
e1.record(); torch.cuda.synchronize()
dt = e0.elapsed_time(e1) / 20 * 1e-3
hp = offs.astype(np.uint64) + np.uint64(host.ctypes.data)
want = hash_ref.fold64_c_batch(hp, lens.astype(np.uint64), threads=os.cpu_count())
ok = np.array_equal(out.cpu().numpy().view(np.uint64), want)
print(f"{'one 1 MiB + 1999 x 1 KiB' if os.environ.get('ONE_LONG') else 'C1'} {part or ''} wps={os.environ.get('B2L_RAGGED_WPS','-')} lead={os.environ.get('B2L_LEAD_TICKET','-')} split={os.environ.get('B2L_HASH_NO_SPLIT') is None}: {dt*1e3:.3f} ms {lens.sum()/dt/1e9:.1f} GB/s digests ok={ok}")
PY
python /tmp/c1t.py
B2L_HASH_NO_DUAL=1 python /tmp/c1t.py
B2L_HASH_NO_SPLIT=1 python /tmp/c1t.py
B2L_RAGGED_WPS=3 python /tmp/c1t.py
PART=top python /tmp/c1t.py
PART=rest python /tmp/c1t.py
PART=rest B2L_HASH_NO_DUAL=1 python /tmp/c1t.py
bash tools/gpu/chain.sh 2>&1 | tail -1
timeout 600 python -m pytest tests/test_hash_gpu.py tests/test_capture.py -q -x 2>&1 | tail -2
