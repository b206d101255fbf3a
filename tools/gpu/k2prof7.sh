cp tools/_exp/libb2l_k2w32.so paper_2601_12713_b200/libb2l.so; touch paper_2601_12713_b200/libb2l.so
cat > /tmp/k2one.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch
from paper_2601_12713_b200 import hashing as H
n = 256 << 20
t = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
out = torch.empty(1, dtype=torch.int64, device="cuda")
for _ in range(2): H.hash_large(t.data_ptr(), n, out.data_ptr())
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none -k regex:k_group -s 17 -c 2 -o gpurun_out/k2v7 -f python /tmp/k2one.py > /dev/null 2>&1
ls -la gpurun_out/k2v7.ncu-rep
