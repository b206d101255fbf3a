import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
dev = torch.device("cuda")
s = torch.cuda.Stream()
buf = torch.empty(8_000_000, dtype=torch.uint8, pin_memory=True)
v = buf.numpy().view(np.int64)
t_np = torch.from_numpy(v)
print("from_numpy is_pinned", t_np.is_pinned(), "buf pinned", buf.is_pinned())
for name, src in (("pinned tensor", buf.view(torch.int64)), ("from_numpy view", t_np)):
    for _ in range(3):
        with torch.cuda.stream(s):
            x = src.to(dev, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    with torch.cuda.stream(s):
        xs = [src.to(dev, non_blocking=True) for _ in range(10)]
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name}: host {1e3*(t1-t)/10:.3f} ms per .to, total {1e3*(t2-t):.3f} ms for 10 x 8 MB")
    del xs
# preallocated destination + copy_
dst = torch.empty(1_000_000, dtype=torch.int64, device=dev)
torch.cuda.synchronize(); t = time.perf_counter()
with torch.cuda.stream(s):
    for _ in range(10):
        dst.copy_(t_np, non_blocking=True)
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"copy_ into preallocated: host {1e3*(t1-t)/10:.3f} ms each, total {1e3*(t2-t):.3f}")
