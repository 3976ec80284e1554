#!/bin/bash
mkdir -p gpurun_out
make -j16 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
for rep in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_shp_base_$rep.log 2>&1
  TSR_K4R_REGION=4 TSR_K4R_PX=8 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_shp_r4p8_$rep.log 2>&1
  TSR_K4R_REGION=8 TSR_K4R_PX=4 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_shp_r8p4_$rep.log 2>&1
done
