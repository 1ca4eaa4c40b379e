"""Write-only HBM bandwidth on this GPU (the roofline denominator for a
store-only kernel): torch fill_ of 8 GiB, best of 10, CUDA events; plus a
read+write copy for comparison with MEASURED_PEAKS.json."""
import json

import torch

x = torch.empty(8 << 30, dtype=torch.uint8, device="cuda")
best = 1e9
for i in range(12):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    x.fill_(i)
    b.record()
    torch.cuda.synchronize()
    if i >= 2:
        best = min(best, a.elapsed_time(b))
cp = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
y = torch.empty_like(cp)
bc = 1e9
for i in range(12):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    y.copy_(cp)
    b.record()
    torch.cuda.synchronize()
    if i >= 2:
        bc = min(bc, a.elapsed_time(b))
print(json.dumps({"write_only_gbs": (8 << 30) / best / 1e6, "copy_rw_gbs": 2 * (4 << 30) / bc / 1e6}))
