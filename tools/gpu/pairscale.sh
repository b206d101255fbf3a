# wall time of K concurrent 1 MiB split pairs (plus 16-B fillers so the ragged/lead path is taken)
cat > /tmp/ps.py <<'PY'
import sys, os; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2601_12713_b200 import hash_device
dev = torch.device("cuda")
for K in (1, 8, 37, 74, 148, 222, 296):
    lens = np.concatenate([np.full(K, 1 << 20), np.full(1300 - K, 16)]).astype(np.int64)
    n = lens.size
    offs = np.zeros(n, np.int64); offs[1:] = np.cumsum((lens + 255) // 256 * 256)[:-1]
    slab = torch.randint(0, 256, (int(offs[-1] + lens[-1]),), dtype=torch.uint8, device=dev)
    o_d, l_d = torch.from_numpy(offs).to(dev), torch.from_numpy(lens).to(dev)
    ptrs = o_d + slab.data_ptr()
    order = torch.from_numpy(np.argsort(-lens, kind="stable").astype(np.int32)).to(dev)
    out = torch.empty(n, dtype=torch.int64, device=dev)
    for _ in range(3): hash_device(ptrs, l_d, out, order=order)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): hash_device(ptrs, l_d, out, order=order)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"K={K:4d} pairs of 1 MiB: {ms:.3f} ms = {ms*1e-3*1.965e9/(1<<17):.2f} cycles/word at 1965 MHz", flush=True)
PY
python /tmp/ps.py
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
