# Per-call latency of the HashFn drop-in (ours vs reference) and, on the device, one
# buffer through the batch kernel vs K2 (hash_large) -- picks the K2 single-buffer threshold.
timeout 300 python - <<'PY'
import sys, time, os
sys.path.insert(0, "."); sys.path.insert(0, "baseline/_ref")
import torch
import paper_2601_12713_b200 as b
from paper_2601_12713_b200 import hashing as H
from dmlens.hashing import hash_bytes as ref_hash
for n in (64, 1024, 16384, 65536, 262144, 1 << 20):
    p = os.urandom(n)
    assert b.hash_bytes(p) == ref_hash(p)
    for name, f in (("ours", b.hash_bytes), ("reference", ref_hash)):
        k = 200 if n <= 65536 else 20
        if name == "reference" and n >= 65536: k = 3
        t = time.perf_counter()
        for _ in range(k): f(p)
        dt = (time.perf_counter() - t) / k
        print(f"{n:>8} B  {name:9s} {dt*1e6:10.1f} us/call", flush=True)
dev = torch.device("cuda:0")
for n in (4096, 16384, 65536, 131072, 262144, 524288, 1 << 20, 4 << 20, 16 << 20):
    t = torch.randint(0, 256, (n,), dtype=torch.uint8, device=dev)
    out = torch.empty(1, dtype=torch.int64, device=dev)
    out2 = torch.empty(1, dtype=torch.int64, device=dev)
    ptrs = torch.tensor([t.data_ptr()], dtype=torch.int64, device=dev)
    lens = torch.tensor([n], dtype=torch.int64, device=dev)
    res = {}
    for name, f in (("batch", lambda: H.hash_device(ptrs, lens, out)),
                    ("k2", lambda: H.hash_large(t.data_ptr(), n, out2.data_ptr()))):
        for _ in range(3): f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): f()
        e1.record(); torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / 20 * 1e3
    assert int(out.item()) == int(out2.item())
    print(f"device {n:>9} B  batch {res['batch']:9.1f} us  k2 {res['k2']:9.1f} us", flush=True)
PY
