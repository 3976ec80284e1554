#!/bin/bash
mkdir -p gpurun_out
TSR_K4=units timeout 600 ncu --set full --import-source on -k regex:"render_bwd" -s 2 -c 1 -o gpurun_out/k4_units python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_units.log 2>&1
TSR_K4=tiles timeout 600 ncu --set full --import-source on -k regex:"render_bwd" -s 2 -c 1 -o gpurun_out/k4_tiles python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_tiles.log 2>&1
