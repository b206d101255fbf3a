"""K2 (b2l_hash_large) timing on one GPU: per-buffer ms and GB/s for a few sizes, each digest
checked against the C oracle.  Measurement helper, not on the product path."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import hash_ref  # noqa: E402  (the checker)
from paper_2601_12713_b200.hashing import hash_large  # noqa: E402

dev = torch.device("cuda:0")
sizes = [int(a) for a in sys.argv[1:] if int(a)] if sys.argv[1:] else [1 << 20, 16 << 20, 256 << 20, (256 << 20) + 3]
for n in sizes:
    g = torch.Generator(device=dev).manual_seed(n)
    buf = torch.randint(0, 256, (n + 5,), dtype=torch.uint8, device=dev, generator=g)
    out = torch.zeros(2, dtype=torch.int64, device=dev)
    ok = True
    for off in (0, 5):
        hash_large(buf.data_ptr() + off, n, out.data_ptr() + 8 * (off > 0))
    torch.cuda.synchronize()
    host = buf.cpu().numpy()
    for j, off in enumerate((0, 5)):
        want = hash_ref.fold64_c(host[off:off + n].tobytes())
        ok &= int(out[j].item()) & (2**64 - 1) == want
    iters = 20 if n >= (64 << 20) else 100
    for _ in range(3):
        hash_large(buf.data_ptr(), n, out.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        hash_large(buf.data_ptr(), n, out.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    print(f"K2 {n:>11} B  {ms:8.3f} ms  {n / ms / 1e6:8.1f} GB/s  match={ok}", flush=True)

# several huge buffers per call (b2l_hash_large_many): C3's 16 x 256 MiB stencil arrays
import os  # noqa: E402

from paper_2601_12713_b200.hashing import hash_large_many  # noqa: E402

k, size = int(os.environ.get("K2_MANY", "16")), int(os.environ.get("K2_MANY_BYTES", str(256 << 20)))
if k:
    slab = torch.randint(0, 256, (k * size,), dtype=torch.uint8, device=dev)
    ptrs = [slab.data_ptr() + i * size for i in range(k)]
    out = torch.zeros(k, dtype=torch.int64, device=dev)
    hash_large_many(ptrs, [size] * k, out.data_ptr())
    torch.cuda.synchronize()
    host = slab[:2 * size].cpu().numpy()
    ok = all(int(out[i].item()) & (2**64 - 1) == hash_ref.fold64_c(host[i * size:(i + 1) * size].tobytes())
             for i in range(2))
    one = torch.zeros(k, dtype=torch.int64, device=dev)
    for i in range(k):
        hash_large(ptrs[i], size, one.data_ptr() + 8 * i)
    torch.cuda.synchronize()
    ok &= bool(torch.equal(one, out))
    for name, f in (("many", lambda: hash_large_many(ptrs, [size] * k, out.data_ptr())),
                    ("one-by-one", lambda: [hash_large(p, size, one.data_ptr()) for p in ptrs])):
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"K2 {name:10s} {k} x {size} B  {ms:8.3f} ms  {k * size / ms / 1e6:8.1f} GB/s  match={ok} "
              f"jobs={os.environ.get('B2L_K2_JOBS', '16')} teams={os.environ.get('B2L_K2_TEAMS', '1')}", flush=True)
