import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2601_19489_b200 import binning
from paper_2601_19489_b200.synthetic import random_splat_batch
b = random_splat_batch(1000000, 8.0, 0, width=1920, height=1080)
out = {}
for st in (0, 1):
    b.counts = None
    binning._ensure_counts(b, st)
    torch.cuda.synchronize()
    out[st] = (b.spans.cpu().numpy().view(np.uint32).reshape(-1, 4).copy(), b.counts.cpu().numpy().copy())
s0, c0 = out[0]; s1, c1 = out[1]
print("counts equal", np.array_equal(c0, c1))
ov0 = (s0[:, 1] >> 31) & 1; ov1 = (s1[:, 1] >> 31) & 1
print("overflow seq", ov0.mean(), "lb", ov1.mean())
diff = np.flatnonzero((s0 != s1).any(1))
print("rows with different spans", len(diff))
for i in diff[:5]:
    print(i, [hex(x) for x in s0[i]], [hex(x) for x in s1[i]], c0[i], c1[i])
