#!/bin/bash
mkdir -p gpurun_out
make -j16 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
for rep in 1 2; do
  timeout 300 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c1_tiles_$rep.log 2>&1
  TSR_K4_REGIONS_MIN_PAIRS=0 timeout 300 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c1_reg_$rep.log 2>&1
done
