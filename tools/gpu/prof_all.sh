#!/bin/bash
# ubench + one ncu --set full capture of every hot kernel of one C2 step
mkdir -p gpurun_out
./tools/ubench/fma_pipe > gpurun_out/ubench_fma.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"render_bwd|render_fwd|ssim|preprocess_kernel|vjp_adam|emit_pairs|radix_scatter_kernel<8" \
  -s 9 -c 9 -o gpurun_out/prof_all python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
  > gpurun_out/ncu_all.log 2>&1; echo ncu=$? >> gpurun_out/status.txt
