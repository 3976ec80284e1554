#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
for r in 8 4 8 4; do
TSR_K4R_REGION=$r timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e >> gpurun_out/bench_r4ab_$r.log 2>&1
done
