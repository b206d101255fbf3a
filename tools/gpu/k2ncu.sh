# ncu --set full (with source) of one K2 launch on a 256 MiB buffer (the shipping kernel)
cat > /tmp/k2one.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch
from paper_2601_12713_b200 import hashing as H
n = 256 << 20
t = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
out = torch.empty(1, dtype=torch.int64, device="cuda")
for _ in range(3): H.hash_large(t.data_ptr(), n, out.data_ptr())
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_hash_planes -s 2 -c 1 -o gpurun_out/k2_full -f python /tmp/k2one.py > gpurun_out/k2ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/k2_full.ncu-rep gpurun_out/k2_ncu_summary.json --algo-bytes 268435456 > /dev/null 2>&1
tail -3 gpurun_out/k2ncu.log
