#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
for c in c3 c3lo; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_now_$c.log 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"render_bwd_regions|render_fwd" -s 2 -c 2 -o gpurun_out/k4r_now python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_now.log 2>&1
