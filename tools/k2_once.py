"""One K2 launch on the canonical C2 batch (for ncu -k build_index)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2601_19489_b200 as ts  # noqa: E402
from paper_2601_19489_b200.synthetic import make_scene  # noqa: E402

n, clustered = {"c2": (1_000_000, False), "c3": (3_000_000, True)}[sys.argv[1] if len(sys.argv) > 1 else "c2"]
params, cam, _ = make_scene(n, 1920, 1080, seed=0, clustered=clustered)
g = ts.GaussianSet(**params)
c = ts.Camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], 1920, 1080, cam["R"], cam["t"])
b = ts.project(g, c)
idx = ts.bin_sequential(b)
torch.cuda.synchronize()
print("P", idx.n_pairs)
