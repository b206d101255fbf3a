# Lone FNV chain: cycles/word of the step formulations (tools/chain_bench.cu) and one 1 MiB
# buffer through the batch kernel (k_hash_warp, lone chain).
./tools/chain_bench
timeout 300 python - <<'PY'
import sys; sys.path.insert(0, ".")
import torch
from paper_2601_12713_b200 import hashing as H
dev = torch.device("cuda:0")
for n in (1 << 20,):
    t = torch.randint(0, 256, (n,), dtype=torch.uint8, device=dev)
    out = torch.empty(1, dtype=torch.int64, device=dev)
    ptrs = torch.tensor([t.data_ptr()], dtype=torch.int64, device=dev)
    lens = torch.tensor([n], dtype=torch.int64, device=dev)
    for _ in range(3): H.hash_device(ptrs, lens, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): H.hash_device(ptrs, lens, out)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    print(f"batch kernel, one {n} B buffer: {us:.1f} us = {us*1e-6*1.965e9/(n/8):.2f} cycles/word at 1965 MHz")
PY
