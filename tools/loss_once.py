"""One fused photometric loss at 1080p (for ncu -k ssim)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_19489_b200.losses import photometric_device  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
r = torch.rand(1080, 1920, 3, device="cuda", generator=g)
t = torch.rand(1080, 1920, 3, device="cuda", generator=g)
for _ in range(2):
    out = photometric_device(r, t)
torch.cuda.synchronize()
print(out[0] if isinstance(out, tuple) else out)
