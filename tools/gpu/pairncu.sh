# ncu warp-state stats of the split pairs at K = 37 and K = 296 concurrent 1 MiB buffers
cat > /tmp/ps2.py <<'PY'
import sys, os; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2601_12713_b200 import hash_device
dev = torch.device("cuda")
K = int(sys.argv[1])
lens = np.concatenate([np.full(K, 1 << 20), np.full(1300 - K, 16)]).astype(np.int64)
n = lens.size
offs = np.zeros(n, np.int64); offs[1:] = np.cumsum((lens + 255) // 256 * 256)[:-1]
slab = torch.randint(0, 256, (int(offs[-1] + lens[-1]),), dtype=torch.uint8, device=dev)
o_d, l_d = torch.from_numpy(offs).to(dev), torch.from_numpy(lens).to(dev)
ptrs = o_d + slab.data_ptr()
order = torch.from_numpy(np.argsort(-lens, kind="stable").astype(np.int32)).to(dev)
out = torch.empty(n, dtype=torch.int64, device=dev)
for _ in range(2): hash_device(ptrs, l_d, out, order=order)
torch.cuda.synchronize()
PY
for K in 37 296; do
  ncu --set full --import-source on -k regex:k_hash_warp -s 1 -c 1 -o gpurun_out/pairs_$K python /tmp/ps2.py $K > /dev/null 2>&1
done
ls -la gpurun_out/
