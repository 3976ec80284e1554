#!/bin/bash
mkdir -p gpurun_out
for f in tiles units; do
  TSR_K4=$f timeout 600 python bench.py --config c3lo --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3lo_$f.log 2>&1
done
TSR_K4=tiles timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_tiles.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3lo.csv python bench.py --config c3lo --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python - <<'P' > gpurun_out/c3lo_stats.txt 2>&1
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2601_19489_b200 as ts
from paper_2601_19489_b200.synthetic import make_scene
params, cam, gt = make_scene(3_000_000, 1920, 1080, seed=0, clustered=True, cluster_opacity=(0.005, 0.03))
g = ts.GaussianSet(**params)
c = ts.Camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], 1920, 1080, cam["R"], cam["t"])
vr = ts.render_view(g, c, ts.TrainConfig())
nc = vr.buffers.n_considered.cpu().numpy(); nb = vr.buffers.n_contrib.cpu().numpy()
cnt = np.diff(vr.tiles.offsets.cpu().numpy())
print("P", vr.tiles.n_pairs, "max tile", cnt.max(), "sum ncons", nc.sum(), "sum ncontrib", nb.sum())
print("ncons max", nc.max(), "p99", np.percentile(nc, 99), "mean", nc.mean())
pad = np.zeros((1088, 1920), np.int64); pad[:1080] = nc
t = pad.reshape(68, 16, 120, 16).transpose(0, 2, 1, 3).reshape(-1, 256).max(1)
print("per-tile max ncons: top10", np.sort(t)[-10:], "tiles>2000:", (t > 2000).sum())
P
