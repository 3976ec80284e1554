"""Per-tile pair-count distribution of the canonical scenes (sizing K2's
per-tile sort): python tools/tile_probe.py [c2|c3]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2601_19489_b200 as ts  # noqa: E402
from paper_2601_19489_b200.synthetic import make_scene  # noqa: E402

for name in sys.argv[1:] or ["c2", "c3"]:
    n, clustered = {"c2": (1_000_000, False), "c3": (3_000_000, True)}[name]
    params, cam, _ = make_scene(n, 1920, 1080, seed=0, clustered=clustered)
    g = ts.GaussianSet(**params)
    c = ts.Camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], 1920, 1080, cam["R"], cam["t"])
    b = ts.project(g, c)
    idx = ts.bin_sequential(b)
    cnt = np.diff(idx.offsets.cpu().numpy())
    q = np.percentile(cnt, [50, 90, 99, 99.9, 100])
    print(name, "M", len(b), "P", int(idx.n_pairs), "tiles", len(cnt), "pct50/90/99/99.9/max", q)
    for cap in (2048, 4096, 8192, 16384):
        heavy = cnt[cnt > cap]
        print(f"  > {cap}: {len(heavy)} tiles, {heavy.sum()} pairs, chunks {np.ceil(heavy / cap).sum():.0f}")
    d = b.depth_bits.cpu().numpy().view(np.uint32) if hasattr(b, "depth_bits") else None
    torch.cuda.synchronize()
