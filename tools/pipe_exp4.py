"""Latency of a small device->host read-back (8-B copy + stream sync, what the engine does to size
its next step) alone and while a large host->device upload runs on another stream; the same for
a kernel writing into mapped pinned memory polled by the host."""
import sys, time
sys.path.insert(0, ".")
import torch

dev = torch.device("cuda")
big = torch.empty(800 << 20, dtype=torch.uint8, pin_memory=True)
dbig = torch.empty(800 << 20, dtype=torch.uint8, device=dev)
bg = torch.cuda.Stream()
s = torch.cuda.Stream()
src = torch.arange(16, dtype=torch.int64, device=dev)
dst = torch.empty(16, dtype=torch.int64, pin_memory=True)


def readbacks(k=200):
    ts = []
    with torch.cuda.stream(s):
        for _ in range(k):
            t = time.perf_counter()
            dst.copy_(src[:1], non_blocking=True)
            s.synchronize()
            ts.append(1e6 * (time.perf_counter() - t))
    ts.sort()
    return ts[len(ts) // 2], ts[int(len(ts) * 0.9)]


def small_kernels(k=200):  # launch + completion of a tiny kernel, no copies
    ts = []
    with torch.cuda.stream(s):
        for _ in range(k):
            t = time.perf_counter()
            src.add_(0)
            s.synchronize()
            ts.append(1e6 * (time.perf_counter() - t))
    ts.sort()
    return ts[len(ts) // 2], ts[int(len(ts) * 0.9)]


for label, fn in (("8-B D2H read-back + sync", readbacks), ("tiny kernel + sync", small_kernels)):
    torch.cuda.synchronize()
    alone = fn()
    with torch.cuda.stream(bg):
        dbig.copy_(big, non_blocking=True)  # ~15 ms of H2D
    beside = fn(60)
    torch.cuda.synchronize()
    print(f"{label:28s} median/p90 us: alone {alone[0]:.1f}/{alone[1]:.1f}   beside an 800 MB H2D "
          f"{beside[0]:.1f}/{beside[1]:.1f}", flush=True)

# mapped pinned memory written by a tiny kernel, the host spinning on the value (no stream sync)
mapped = torch.zeros(16, dtype=torch.int64, pin_memory=True)
import ctypes
cudart = ctypes.CDLL("libcudart.so")
dptr = ctypes.c_void_p()
assert cudart.cudaHostGetDevicePointer(ctypes.byref(dptr), ctypes.c_void_p(mapped.data_ptr()), 0) == 0
mapped_dev = torch.cuda.caching_allocator_alloc  # noqa (not used)
# a device view of the mapped buffer through torch is not available; use a raw copy kernel via cudaMemcpyAsync
# from device to the mapped device pointer (a DtoD write into host memory = the GPU writes over PCIe)
def mapped_polls(k=200):
    ts = []
    flag = mapped.numpy()
    with torch.cuda.stream(s):
        for i in range(1, k + 1):
            src.fill_(i)
            t = time.perf_counter()
            assert cudart.cudaMemcpyAsync(dptr, ctypes.c_void_p(src.data_ptr()), 8, 3, ctypes.c_void_p(s.cuda_stream)) == 0
            while flag[0] != i:
                pass
            ts.append(1e6 * (time.perf_counter() - t))
    s.synchronize()
    ts.sort()
    return ts[len(ts) // 2], ts[int(len(ts) * 0.9)]


torch.cuda.synchronize()
alone = mapped_polls()
with torch.cuda.stream(bg):
    dbig.copy_(big, non_blocking=True)
beside = mapped_polls(60)
torch.cuda.synchronize()
print(f"{'DtoD into mapped + host spin':28s} median/p90 us: alone {alone[0]:.1f}/{alone[1]:.1f}   beside an 800 MB H2D "
      f"{beside[0]:.1f}/{beside[1]:.1f}", flush=True)
