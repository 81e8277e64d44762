"""Device-copy bandwidth of this box (torch copy of a 4 GiB buffer), to tell
a slow box from a slow kernel when comparing runs across boxes."""
import json

import torch

x = torch.empty(1 << 30, dtype=torch.float32, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    y.copy_(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    y.copy_(x)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(json.dumps({"copy_gbs": round(2 * x.numel() * 4 / (ms / 1e3) / 1e9, 1), "ms": round(ms, 3)}))
