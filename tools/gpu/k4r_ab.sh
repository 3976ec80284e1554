#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
for r in 8 4; do
TSR_K4R_REGION=$r timeout 600 ncu --set full --import-source on --clock-control none -k regex:"render_bwd_regions" -s 1 -c 1 -o gpurun_out/k4r_r$r python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k4r_$r.log 2>&1
done
