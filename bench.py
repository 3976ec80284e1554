#!/usr/bin/env python
"""Benchmark: train steps/s (fwd + bwd + Adam) at 1M Gaussians, 1080p.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c1]
    python bench.py --impl reference ...        # CPU reference arm
    python bench.py --config c5 [--budget S]    # the 1-minute training loop

A step is one training step over one camera view per GPU: K1 preprocess ->
K2 keys/sort/ranges -> K3 render -> photometric loss -> K4 per-Gaussian
backward -> K4b+K5 (fused projection VJP + Adam at N=1; VJP, NCCL allreduce,
Adam at N>1).  Inputs: the canonical synthetic scene of SURVEY.md §8(d),
resident in HBM.  `value` is whole-job view-steps/s (= steps/s at N=1).
Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "c1": dict(n=10_000, width=256, height=256, clustered=False),
    "c2": dict(n=1_000_000, width=1920, height=1080, clustered=False),
    "c3": dict(n=3_000_000, width=1920, height=1080, clustered=True),
    # C3 with a low-opacity cluster (U(0.005, 0.03)): the
    # cluster tiles need thousands of blends per pixel before terminating,
    # the heavy-tile stress case for K3/K4 load balance
    "c3lo": dict(n=3_000_000, width=1920, height=1080, clustered=True,
                 cluster_opacity=(0.005, 0.03)),
    # BASELINE configs[3]: a batch of 8 ring views per optimizer step, split
    # across the GPUs (strong scaling), one gradient allreduce per step
    "c4": dict(n=1_000_000, width=1920, height=1080, clustered=False, views=8),
}
METRIC = "train steps/sec (fwd+bwd+Adam) at 1M Gaussians 1080p"
# one training step over one camera view; at N GPUs the job runs N views per
# step (weak scaling), so the whole-job unit is view-steps/s in BOTH arms
UNIT = "view-steps/s"
# FP32 lane-op counts per unit of work
RENDER_OPS = (12, 7)       # per evaluation, per blend
BACKWARD_OPS = (12, 45)
NOMINAL_FP32_LANES = 148 * 128


def fp32_peak(sm_mhz):
    """FP32 lane-op peak (T/s): the measured FFMA/FFMA2 throughput of this
    part (profiles/r2_fp32_peak.json, tools/ubench/fma_pipe.cu), scaled to the
    SM clock sampled during the timed region; nominal 148 x 128 x clock if the
    measurement is missing."""
    f = ROOT / "profiles" / "r2_fp32_peak.json"
    if f.exists():
        d = json.loads(f.read_text())
        meas = d["peak_lane_ops_tops"] * sm_mhz / d["sm_clock_mhz_sampled"]
        return meas, (f"measured FP32 peak {d['peak_lane_ops_tops']:.2f} T lane-ops/s at "
                      f"{d['sm_clock_mhz_sampled']} MHz (profiles/r2_fp32_peak.json, "
                      f"tools/ubench/fma_pipe.cu), scaled to the sampled {sm_mhz:.0f} MHz")
    return (NOMINAL_FP32_LANES * sm_mhz * 1e6 / 1e12,
            "nominal FP32 lane-ops/s = 148 SMs x 128 lanes x sampled SM clock")


def k4_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum of ONE K4 launch from the
    committed ncu --set full capture of the current kernel."""
    f = ROOT / "profiles" / "k4_traffic.json"
    if not f.exists():
        return None, None
    d = json.loads(f.read_text())
    return d["bytes_per_launch"], d["source"]


def _env_int(name, default):
    return int(os.environ.get(name, default))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS) + ["c5"])
    ap.add_argument("--budget", type=float, default=60.0, help="c5 wall-clock budget (s)")
    ap.add_argument("--c5-views", type=int, default=200)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--peer", action="store_true",
                    help="N>1 / c4: ZeRO-1 fused into one kernel over peer memory (CUDA IPC)")
    ap.add_argument("--zero1", action="store_true",
                    help="N>1 / c4: ZeRO-1 update (reduce-scatter, K5 on the row shard, all-gather)")
    ap.add_argument("--deterministic", action="store_true",
                    help="K4 deterministic merge (bitwise reproducible)")
    ap.add_argument("--vp", action="store_true",
                    help="N=1: run the view-parallel (N>1) step, with its NCCL collectives "
                         "on a world-size-1 communicator")
    return ap.parse_args()


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md)."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-i", str(self.gpu), "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        os.unlink(self.path)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# -------------------------------------------------------------- CPU oracle --
def _cpu_sample_step(scene, tile_frac, cores=1, gauss_frac=1.0, seed=0):
    """One bounded-sample training step of the CPU oracle; returns the
    extrapolated full-step seconds and a per-stage dict.

    Vectorised stages (project, bin, loss, VJP, Adam) run on a `gauss_frac`
    subset of Gaussians / image rows and are scaled by 1/gauss_frac; render and
    backward run on a random `tile_frac` of the non-empty tiles and are scaled
    by the pair-count fraction (per-tile work is proportional to list length
    up to termination)."""
    from oracle import raster as O
    params, cam, gt = scene
    rng = np.random.default_rng(seed)
    n = len(params["positions"])
    k = max(1, int(n * gauss_frac))
    sub = {key: v[:k] for key, v in params.items()}
    st = {}
    t0 = time.perf_counter()
    batch, colors = O.project(sub, cam)
    st["project"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    idx = O.bin_sequential(batch)
    st["bin"] = time.perf_counter() - t0
    counts = np.diff(idx["offsets"])
    busy = np.flatnonzero(counts > 0)
    m = max(1, int(round(len(busy) * tile_frac)))
    pick = np.sort(rng.choice(busy, m, replace=False))
    frac_pairs = counts[pick].sum() / max(counts.sum(), 1)
    t0 = time.perf_counter()
    if cores <= 1:
        bufs = O.render(batch, idx, colors, np.zeros(3), tiles=pick)
    else:
        bufs = _pool_render(cores, batch, idx, colors, pick)
    st["render"] = time.perf_counter() - t0
    rows = max(16, int(cam["height"] * gauss_frac))
    t0 = time.perf_counter()
    _, _, _, gcol = O.photometric(bufs["color"][:rows], gt[:rows])
    st["loss"] = time.perf_counter() - t0
    gfull = np.zeros_like(bufs["color"])
    gfull[:rows] = gcol
    gfull[rows:] = rng.normal(0, 1e-7, gfull[rows:].shape)
    t0 = time.perf_counter()
    if cores <= 1:
        g2 = O.backward_per_gaussian(bufs, batch, idx, colors, gfull, tiles=pick)
    else:
        g2 = _pool_backward(cores, bufs, batch, idx, colors, gfull, pick)
    st["backward"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    g3 = O.project_vjp(sub, cam, batch, g2)
    st["vjp"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    for name in ("positions", "log_scales", "rotations", "opacity_logits", "colors"):
        p = sub[name].copy()
        O.adam_step(p, g3[name], np.zeros_like(p), np.zeros_like(p), 1, 1e-3,
                    renormalize=(name == "rotations"))
    st["adam"] = time.perf_counter() - t0
    scale = {"project": 1 / gauss_frac, "bin": 1 / gauss_frac, "loss": cam["height"] / rows,
             "vjp": 1 / gauss_frac, "adam": 1 / gauss_frac,
             "render": 1 / frac_pairs, "backward": 1 / frac_pairs}
    est = {key: st[key] * scale[key] for key in st}
    return sum(est.values()), est, dict(tiles=int(m), busy_tiles=int(len(busy)),
                                        pair_frac=float(frac_pairs), gauss_frac=gauss_frac)


_SHARED = {}


def _render_tiles(tiles):
    from oracle import raster as O
    s = _SHARED
    return tiles, O.render(s["batch"], s["idx"], s["colors"], np.zeros(3), tiles=tiles)


def _backward_tiles(tiles):
    from oracle import raster as O
    s = _SHARED
    return O.backward_per_gaussian(s["bufs"], s["batch"], s["idx"], s["colors"], s["g"],
                                   tiles=tiles)


def _forked_map(fn, chunks, cores, **shared):
    """Map over tile chunks in `cores` forked workers that inherit `shared`
    copy-on-write (no pickling of the scene)."""
    import multiprocessing as mp
    _SHARED.clear()
    _SHARED.update(shared)
    with mp.get_context("fork").Pool(cores) as pool:
        return pool.map(fn, chunks)


def _pool_render(cores, batch, idx, colors, pick):
    chunks = [c for c in np.array_split(pick, cores) if len(c)]
    results = _forked_map(_render_tiles, chunks, cores, batch=batch, idx=idx, colors=colors)
    W, H = batch["width"], batch["height"]
    bufs = dict(color=np.zeros((H, W, 3)), depth=np.zeros((H, W)), final_T=np.ones((H, W)),
                n_contrib=np.zeros((H, W), np.int32), n_considered=np.zeros((H, W), np.int32),
                checkpoints={})
    for tiles, out in results:
        for t in tiles:
            ty, tx = divmod(int(t), idx["tiles_x"])
            sl = (slice(ty * 16, ty * 16 + 16), slice(tx * 16, tx * 16 + 16))
            for key in ("color", "depth", "final_T", "n_contrib", "n_considered"):
                bufs[key][sl] = out[key][sl]
        bufs["checkpoints"].update(out["checkpoints"])
    return bufs


def _pool_backward(cores, bufs, batch, idx, colors, g, pick):
    chunks = [c for c in np.array_split(pick, cores) if len(c)]
    results = _forked_map(_backward_tiles, chunks, cores, bufs=bufs, batch=batch, idx=idx,
                          colors=colors, g=g)
    out = results[0]
    for r in results[1:]:
        for key in ("d_means2d", "d_conics", "d_opacities", "d_colors", "d_depths"):
            out[key] += r[key]
        out["merges"] += r["merges"]
    return out


def cpu_baseline(cfg_name, target_s=20.0):
    """Single-core oracle, bounded sample (~10-30 s of CPU work)."""
    from paper_2601_19489_b200.synthetic import make_scene
    c = CONFIGS[cfg_name]
    scene = make_scene(c["n"], c["width"], c["height"], seed=0, clustered=c["clustered"],
                       cluster_opacity=c.get("cluster_opacity"))
    frac = 0.01 if c["n"] >= 1_000_000 else 0.25
    t0 = time.perf_counter()
    est, stages, sample = _cpu_sample_step(scene, frac)
    wall = time.perf_counter() - t0
    return {"value": 1.0 / est, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": (f"oracle/raster.py (float64 NumPy restatement, pinned to the reference's "
                       f"golden vectors), 1 thread; one step of {cfg_name} with project/bin/"
                       f"loss/VJP/Adam at full size and render+backward on "
                       f"{sample['tiles']}/{sample['busy_tiles']} random non-empty tiles "
                       f"({sample['pair_frac']:.3%} of pairs), extrapolated by pair count; "
                       f"{wall:.1f} s of CPU work"),
            "est_step_s": est, "stages_s": {k: round(v, 3) for k, v in stages.items()}}


def reference_arm(args):
    """`--impl reference`: the CPU restatement of the reference path on all host
    cores, bounded sample per step, rank 0 only."""
    rank = _env_int("RANK", 0)
    if rank != 0:
        return
    from paper_2601_19489_b200.synthetic import make_scene
    c = CONFIGS[args.config]
    scene = make_scene(c["n"], c["width"], c["height"], seed=0, clustered=c["clustered"],
                       cluster_opacity=c.get("cluster_opacity"))
    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    gauss_frac = 1.0 / 16 if c["n"] >= 1_000_000 else 1.0
    tile_frac = min(1.0, 0.002 * cores) if c["n"] >= 1_000_000 else 1.0
    ests, walls = [], []
    info = None
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        est, stages, info = _cpu_sample_step(scene, tile_frac, cores, gauss_frac, seed=i)
        if i >= args.warmup:
            ests.append(est)
            walls.append(time.perf_counter() - t0)
    est = float(np.mean(ests))
    sample_s = float(np.mean(walls))
    value = 1.0 / est
    # the same metric, unit and config as the GPU arm (one view per step at
    # N=1), so the driver's ratio is defined; each timed step is a bounded
    # sample of the full step (measured wall time below) whose per-stage
    # times are scaled up to the full workload
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": est * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: " + _workload(args.config, 1),
                       "views_per_step": 1},
            "ms_per_step_note": ("ms_per_step is the extrapolated full-step time; the timed "
                                 "region measured sample_s_per_step x steps of wall clock"),
            "sample_s_per_step": sample_s, "timed_region_s": float(np.sum(walls)),
            "extrapolation_factor": est / sample_s,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": (f"oracle/raster.py float64 NumPy port on {cores} "
                                        f"processes; per step: project/bin/VJP/Adam on "
                                        f"{gauss_frac:.4g} of the Gaussians and loss on the "
                                        f"same fraction of rows (x{1/gauss_frac:.0f}), render+"
                                        f"backward on {info['tiles']} random non-empty tiles "
                                        f"({info['pair_frac']:.3%} of pairs); measured "
                                        f"{sample_s:.2f} s per sampled step, extrapolated "
                                        f"x{est / sample_s:.0f} to the full step")},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _workload(name, n_gpus):
    c = CONFIGS[name]
    views = (f"a batch of {c['views']} ring views per step split over the GPUs, one "
             f"gradient allreduce" if c.get("views") else "one view per GPU per step")
    lo = " low-opacity" if c.get("cluster_opacity") else ""
    return (f"{c['n']:,} Gaussians{f' ({lo} clustered depth)'.replace('( ', '(') if c['clustered'] else ''}, "
            f"{c['width']}x{c['height']}, SH0, {views}, "
            f"fwd+loss+bwd+Adam, {n_gpus} GPU(s)")


# ---------------------------------------------------------------- GPU arm --
def gpu_arm(args):
    import torch
    import torch.distributed as dist

    import paper_2601_19489_b200 as ts
    from paper_2601_19489_b200.parallel import ViewParallelStep
    from paper_2601_19489_b200.synthetic import make_scene, ring_poses
    from paper_2601_19489_b200.trainer import phase_times

    rank, world = _env_int("RANK", 0), _env_int("WORLD_SIZE", 1)
    local = _env_int("LOCAL_RANK", 0)
    # TSR_BENCH_BACKEND=gloo + more ranks than GPUs: a functional check of the
    # N>1 path on a one-GPU box (ranks share devices); timings are not valid
    backend = os.environ.get("TSR_BENCH_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1) if backend != "nccl" else local
    torch.cuda.set_device(local)
    if world > 1 or args.vp:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29611")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    c = CONFIGS[args.config]
    params, cam, gt = make_scene(c["n"], c["width"], c["height"], seed=0,
                                 clustered=c["clustered"],
                                 cluster_opacity=c.get("cluster_opacity"))
    gset = ts.GaussianSet(**params)
    batch_views = c.get("views", 0)
    ring = ring_poses(batch_views or max(world, 1), 4.0, cam["fx"], c["width"], c["height"])
    rc = ring[rank % len(ring)]
    camera = ts.Camera(rc["fx"], rc["fy"], rc["cx"], rc["cy"], c["width"], c["height"],
                       rc["R"], rc["t"])
    gt_host = torch.from_numpy(np.asarray(gt, np.float32)).pin_memory()
    gt_dev = gt_host.to("cuda")
    cfg = ts.TrainConfig(max_iters=30_000)
    if batch_views:
        from paper_2601_19489_b200.parallel import shard_views
        mine = shard_views(batch_views, world, rank)
        cams = [ts.Camera(ring[v]["fx"], ring[v]["fy"], ring[v]["cx"], ring[v]["cy"],
                          c["width"], c["height"], ring[v]["R"], ring[v]["t"]) for v in mine]
        plain = not (args.zero1 or args.peer)
        stepper = ViewParallelStep(gset, cfg, extent=4.0, sharded=args.zero1, peer=args.peer,
                                   chunks=4 if plain else None,
                                   graphs=plain and os.environ.get("TSR_VP_GRAPHS", "1") == "1")
        run = lambda timer=None: stepper.step_views(cams, [gt_dev] * len(cams), timer)  # noqa
        args.no_e2e = True
    elif world == 1 and not args.vp:
        # the step replays as one CUDA graph (captured during warm-up)
        stepper = ts.TrainStep(gset, cfg, extent=4.0, graphs=True,
                               deterministic=args.deterministic)
        run = lambda timer=None: stepper.step(camera, gt_dev, timer)  # noqa: E731
    else:
        stepper = ViewParallelStep(gset, cfg, extent=4.0, sharded=args.zero1, peer=args.peer,
                                   force_collectives=args.vp,
                                   chunks=4 if args.vp else None,
                                   graphs=os.environ.get("TSR_VP_GRAPHS", "1") == "1")
        run = lambda timer=None: stepper.step_views([camera], [gt_dev], timer)  # noqa: E731

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    for _ in range(args.warmup):
        run()
    barrier()
    # The scene trains during the run (splats shrink while fitting the noise
    # GT, so per-step work grows with the step count: tools/drift_probe.py).
    # Snapshot the optimisation state after warm-up so the e2e loop below
    # replays the SAME training segment as the device-timed loop.
    snap = {k: v.clone() for k, v in gset.params().items()}
    snap_m = {k: v.clone() for k, v in stepper.opt._m.items()}
    snap_v = {k: v.clone() for k, v in stepper.opt._v.items()}
    snap_steps = dict(stepper.opt._steps)
    snap_it = stepper.iteration

    def restore():
        torch.cuda.synchronize()
        for k, v in gset.params().items():
            v.copy_(snap[k])
        for k in snap_m:
            stepper.opt._m[k].copy_(snap_m[k])
            stepper.opt._v[k].copy_(snap_v[k])
        stepper.opt._steps.update(snap_steps)
        stepper.iteration = snap_it
        torch.cuda.synchronize()

    graphs = (world == 1 and not batch_views and not args.vp) or getattr(stepper, "graphs", False)
    clocks = ClockSampler(local)
    clocks.start()
    timer = {}
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    h0 = time.perf_counter()
    for _ in range(args.steps):
        run(None if graphs else timer)
    host_ms = (time.perf_counter() - h0) * 1e3 / args.steps
    e1.record()
    barrier()
    ms = e0.elapsed_time(e1) / args.steps
    clock = clocks.stop()
    if graphs:
        # per-phase device times: the same segment again, eagerly with events
        # between the phases (outside the timed region)
        restore()
        prev_graphs = stepper.graphs
        stepper.graphs = False
        for _ in range(args.steps):
            run(timer)
        stepper.graphs = prev_graphs
        barrier()
    phases = {k: v / args.steps for k, v in phase_times(timer).items()}
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = (batch_views or world) * 1e3 / ms

    # work counters of the last timed step (for the roofline), outside the timed region
    batch, tiles, bufs = stepper.last_view()
    evals = int(bufs.n_considered.sum().item())
    blends = int(bufs.n_contrib.sum().item())
    pairs = tiles.n_pairs

    # e2e: the public API fed from HOST memory.  Every step copies its GT image
    # H2D from pinned memory (double-buffered on a copy stream, so the copy of
    # step k+1 overlaps step k) and reads its loss back D2H into pinned memory;
    # all of it inside the timed region.
    e2e = None
    if not args.no_e2e:
        copy_stream = torch.cuda.Stream()
        bufs = [torch.empty_like(gt_dev) for _ in range(2)]
        if graphs:  # capture the graphs of both GT buffers before timing
            for b in bufs:
                b.copy_(gt_host)
                if world == 1 and not args.vp:
                    stepper.step(camera, b)
                else:
                    stepper.step_views([camera], [b])
        restore()  # same training segment as the timed loop (outside both timed regions)
        copied = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]
        loss_host = torch.zeros(args.steps, dtype=torch.float32).pin_memory()
        # the step's GT buffer is free once its loss kernels have read it
        # (TrainStep.gt_consumed): the copy for step k + 2 then runs under step
        # k's backward (FP32-bound, little HBM traffic) instead of under the
        # next step's binning / render
        gt_done = getattr(stepper, "gt_consumed", None) if world == 1 and not args.vp else None
        barrier()
        t0 = time.perf_counter()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        with torch.cuda.stream(copy_stream):
            bufs[0].copy_(gt_host, non_blocking=True)
            copied[0].record(copy_stream)
            if gt_done is not None and args.steps > 1:
                bufs[1].copy_(gt_host, non_blocking=True)
                copied[1].record(copy_stream)
        for k in range(args.steps):
            cur, nxt = k % 2, (k + 1) % 2
            torch.cuda.current_stream().wait_event(copied[cur])
            if gt_done is None and k + 1 < args.steps:
                if k >= 1:
                    copy_stream.wait_event(consumed[nxt])
                with torch.cuda.stream(copy_stream):
                    bufs[nxt].copy_(gt_host, non_blocking=True)
                    copied[nxt].record(copy_stream)
            if world == 1 and not args.vp:
                loss = stepper.step(camera, bufs[cur])
            else:
                loss = stepper.step_views([camera], [bufs[cur]])
            consumed[cur].record()
            if gt_done is not None and k + 2 < args.steps:
                copy_stream.wait_event(gt_done)  # step k has read bufs[cur]
                with torch.cuda.stream(copy_stream):
                    bufs[cur].copy_(gt_host, non_blocking=True)
                    copied[cur].record(copy_stream)
            loss_host[k:k + 1].copy_(loss.reshape(1), non_blocking=True)
        e2e_host_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        ev1.record()
        barrier()
        e2e_s = (time.perf_counter() - t0) / args.steps
        e2e_dev_ms = ev0.elapsed_time(ev1) / args.steps
        losses_seen = loss_host.numpy()
        if not np.all(np.isfinite(losses_seen)):
            raise RuntimeError("non-finite loss in the e2e loop")
        if world > 1:
            t = torch.tensor([e2e_s], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": world / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(gt_host.numel() * 4),
               "d2h_bytes_per_step": 4, "ms_per_step": e2e_s * 1e3,
               "last_loss": float(losses_seen[-1]),
               "host_launch_ms_per_step": e2e_host_ms, "device_ms_per_step": e2e_dev_ms,
               "note": "wall clock over the same training segment as the timed loop (state "
                       "restored from the post-warm-up snapshot); GT H2D double-buffered on a "
                       "copy stream (refilled once the step's loss kernels have read it), loss D2H "
                       "async into pinned memory every step"}

    if rank != 0:
        if dist.is_available() and dist.is_initialized():
            dist.destroy_process_group()
        return

    sm_mhz = clock.get("sm_mhz") or 1965.0
    peak_ops, peak_note = fp32_peak(sm_mhz)
    # the backward phase covers every view this rank rasterised in the step;
    # the work counters are the last view's, so time one view's launch
    views_here = len(mine) if batch_views else 1
    bwd_ms = phases.get("backward", 0.0) / views_here
    bwd_ops = BACKWARD_OPS[0] * evals + BACKWARD_OPS[1] * blends
    achieved = bwd_ops / (bwd_ms * 1e-3) / 1e12 if bwd_ms > 0 else None
    # HBM roofline of the fused projection-VJP + Adam kernel (N=1)
    hbm_line = None
    peaks = ROOT / "MEASURED_PEAKS.json"
    hbm_peak = json.loads(peaks.read_text()).get("hbm_gbs") if peaks.exists() else None
    hbm_src = "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    if hbm_peak is None:
        hbm_peak, hbm_src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
    if world == 1 and phases.get("vjp_adam"):
        n = len(gset)
        algo = n * (14 * 4 * 6 + 4) + len(batch) * (10 * 4 * 2 + 32)
        ach = algo / (phases["vjp_adam"] * 1e-3) / 1e9
        hbm_line = {"kernel": "vjp_adam_sh0_kernel (K4b+K5)", "bound": "hbm", "achieved": ach,
                    "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                    "algorithmic_bytes": algo, "peak_source": hbm_src,
                    "bytes_model": "per Gaussian p,m,v read+write (14 x 4 B x 6) + row index 4 B; per row "
                                   "Grad2D read+zero (80 B) + rec 32 B"}
    traffic, traffic_src = k4_traffic()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong" if batch_views else "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (canonical generator, SURVEY.md §8(d), seed 0)",
        "config": {"workload": f"{args.config}: " + _workload(args.config, world),
                   "views_per_step": batch_views or world,
                   "parallelism": f"view-parallel dp{world}"
                                  + (" zero1 fused over peer memory (one kernel: peer gradient "
                                     "reads, sharded Adam, peer parameter stores)" if args.peer
                                     else " zero1 (reduce-scatter + sharded Adam + all-gather)"
                                     if args.zero1 else ""),
                   "launch": ("one CUDA graph replay per step" if graphs and
                              getattr(stepper, "graphs", True) else "eager launches"
                              + (f" (graph capture failed: {stepper.graph_error})"
                                 if getattr(stepper, "graph_error", None) else "")),
                   "merge": "deterministic (slots + emission-order row sums)"
                            if args.deterministic else "float atomics (FP32-tolerance)",
                   "l2": "inputs larger than L2 (Gaussian state + Adam moments 168 MB, "
                         "per-step buffers ~1 GB)",
                   "window": f"training steps {args.warmup + 1}-{args.warmup + args.steps} from "
                             "the seeded init (the scene trains during the run; the e2e loop "
                             "replays the same segment from a post-warm-up snapshot)"},
        "roofline": {"kernel": ("render_bwd_regions_kernel (K4r, region-culled: evaluates only "
                                "the splats of each 8x8 region's K3 list; work counted as the "
                                "reference's full per-pixel evaluation)"
                                if getattr(stepper, "regions", None) is not None
                                else "render_bwd_kernel (K4)"), "bound": "fp32",
                     "achieved": achieved, "peak": peak_ops, "unit": "Tops/s",
                     "frac": (achieved / peak_ops) if achieved else None,
                     "traffic": traffic, "traffic_source": traffic_src,
                     "peak_note": peak_note,
                     "per_view_launch_ms": bwd_ms,
                     "ops_per_unit": {"per_eval": BACKWARD_OPS[0], "per_blend": BACKWARD_OPS[1]},
                     "units": {"evals": evals, "blends": blends, "pairs": pairs}},
        "roofline_hbm": hbm_line,
        "collective": ({"backend": dist.get_backend(), "world": dist.get_world_size(),
                        "chunks": getattr(stepper, "chunks", 1),
                        "exchange": "per-row-chunk allreduce + Adam on a communication stream, "
                                    "overlapping K4b of the next chunk"
                        if getattr(stepper, "chunks", 1) > 1 else "one flat-buffer allreduce"}
                       if dist.is_available() and dist.is_initialized() else None),
        "phases_ms": {k: round(v, 4) for k, v in phases.items()},
        "host_launch_ms_per_step": host_ms,
        "gpu_launches": stepper.kernels_per_step() * args.steps,
        "clocks": clock,
    }
    if e2e is not None:
        line["e2e"] = e2e
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config)
    print(json.dumps(line), flush=True)
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()


# ------------------------------------------------------------------- C5 ---
def c5_arm(args):
    """BASELINE.json configs[4]: the 1-minute loop on a synthetic 200-view
    1080p scene with multi-view-consistency splitting/pruning (SURVEY.md
    §8(d) C5).  GT = the canonical 1M-splat scene rendered by the B200
    renderer into a camera ring (with exact depth priors, round2); the init
    keeps a random half of the GT splats, perturbed as in the reference's
    ablation setup (test_acceptance.py:427-440); densify on; the loop runs
    `train()` until the wall-clock budget.  Reports training iterations/s
    (densify rounds, PSNR evals and the budget checks included) and the
    held-out PSNR before and after."""
    import torch
    import paper_2601_19489_b200 as ts
    from paper_2601_19489_b200.synthetic import make_scene, synthetic_scene
    torch.cuda.set_device(_env_int("LOCAL_RANK", 0))
    t0 = time.perf_counter()
    params, cam, _ = make_scene(1_000_000, 1920, 1080, seed=0)
    gt_set = ts.GaussianSet(**params)
    scene, _ = synthetic_scene(n_views=args.c5_views, width=1920, height=1080, fx=cam["fx"],
                               gt_set=gt_set)
    rng = np.random.default_rng(22)
    n = len(gt_set)
    keep = np.sort(rng.choice(n, size=n // 2, replace=False))
    init = {k: v[keep].copy() for k, v in params.items()}
    m = len(keep)
    init["positions"] = init["positions"] * (1.0 + rng.normal(0, 0.02, (m, 1))) + \
        rng.normal(0, 0.005, (m, 3))
    init["log_scales"] += rng.normal(0, 0.15, (m, 3)) + 0.15
    init["colors"] += rng.normal(0, 0.05, init["colors"].shape)
    init = ts.GaussianSet(**init)
    holdout = tuple(range(0, args.c5_views, max(args.c5_views // 4, 1)))
    cfg = ts.TrainConfig(round_profile="round2", max_iters=200_000,
                         budget_seconds=args.budget, eval_interval=10**9, seed=0,
                         densify_start=500, densify_interval=300, densify_end=10**9,
                         holdout_views=holdout, deterministic=args.deterministic)
    eval_cams = [scene.cameras[i] for i in holdout]
    psnr0 = ts.evaluate(init, eval_cams, cfg)
    setup_s = time.perf_counter() - t0
    res = ts.train(scene, cfg, initial=init)
    psnr1 = ts.evaluate(res.gset, eval_cams, cfg)
    line = {"metric": "C5 training iterations/s (1-minute loop, densify on)",
            "value": res.iterations / res.elapsed, "unit": "iterations/s", "n_gpus": 1,
            "higher_is_better": True, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"c5: 1M-splat GT rendered into {args.c5_views} 1920x1080 "
                                   f"ring views (+depth priors); init = 500k perturbed; round2; "
                                   f"densify every 300 its (K=10); budget {args.budget:g} s",
                       "holdout_views": list(holdout),
                       "merge": "deterministic (slots + emission-order row sums)"
                                if args.deterministic else "float atomics (FP32-tolerance)"},
            "iterations": res.iterations, "elapsed_s": res.elapsed,
            "stop_reason": res.stop_reason, "splats_final": len(res.gset),
            "psnr_holdout_before": psnr0, "psnr_holdout_after": psnr1,
            "setup_s": setup_s}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.config == "c5":
        c5_arm(args)
    elif args.impl == "reference":
        reference_arm(args)
    else:
        gpu_arm(args)


if __name__ == "__main__":
    main()
