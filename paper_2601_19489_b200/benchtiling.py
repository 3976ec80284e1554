"""The reference's own benchmark harness, `tilesplat bench-tiling`
(cli.py:170-202): one random batch binned by the three
strategies (AABB baseline, SnugBox sequential, SnugBox load-balanced), each
timed, with pair counts and TileIndex checksums.  The two SnugBox checksums
must agree (the reference's exit-code-2 check); here they are also
bit-identical to the reference's for the same (n, anisotropy, seed) because
the batch is drawn the same way and K1/K2 are bit-exact.  Times are device
times of the index build (CUDA events on the launching stream), median of
`repeats` after one warm-up."""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import binning
from .synthetic import random_splat_batch


@dataclass
class BenchResult:
    strategy: str  # aabb | snug_seq | snug_lb
    splats: int
    pairs: int
    millis: float
    checksum: str


STRATEGIES = (("aabb", 2), ("snug_seq", 0), ("snug_lb", 1))


def run_bench_tiling(n_splats: int, anisotropy: float, seed: int, width: int = 640,
                     height: int = 480, repeats: int = 5) -> list[BenchResult]:
    batch = random_splat_batch(n_splats, anisotropy, seed, width=width, height=height)
    results = []
    for name, strategy in STRATEGIES:
        idx = binning.build_index(batch, strategy)  # warm-up (and sizes P once)
        times = []
        for _ in range(repeats):
            batch.counts = None  # time the strategy's count pass too
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            idx = binning.build_index(batch, strategy)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        times.sort()
        results.append(BenchResult(name, n_splats, idx.n_pairs, times[len(times) // 2],
                                   idx.checksum()))
    return results


def bench_tiling_csv(results: list[BenchResult]) -> str:
    """The reference's CSV (cli.py:191-197); raises on a SnugBox checksum
    mismatch (the reference exits with code 2)."""
    by_name = {r.strategy: r for r in results}
    if by_name["snug_seq"].checksum != by_name["snug_lb"].checksum:
        raise RuntimeError("checksum mismatch between snug_seq and snug_lb")
    lines = ["strategy,splats,pairs,millis"]
    lines += [f"{r.strategy},{r.splats},{r.pairs},{r.millis:.3f}" for r in results]
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser(description="bench-tiling on the B200 (cli.py:170-202)")
    ap.add_argument("--n-splats", type=int, default=100_000)
    ap.add_argument("--anisotropy", type=float, default=8.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--width", type=int, default=640)
    ap.add_argument("--height", type=int, default=480)
    a = ap.parse_args()
    res = run_bench_tiling(a.n_splats, a.anisotropy, a.seed, a.width, a.height)
    print(bench_tiling_csv(res), end="")
    print(f"# snug checksums: {res[1].checksum} (seq == lb)")
