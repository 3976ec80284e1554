#!/bin/bash
# ncu evidence for every hot kernel of one C2 step (kernel replay), plus the
# cooperative K2 kernel (application replay: ncu cannot kernel-replay it)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"render_bwd|render_fwd|ssim|preprocess_kernel|cull_compact|vjp_adam" \
  -s 8 -c 7 -o gpurun_out/prof_final python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
  > gpurun_out/ncu_final.log 2>&1; echo ncu=$? >> gpurun_out/status.txt
timeout 1500 ncu --replay-mode application --section SpeedOfLight --section MemoryWorkloadAnalysis \
  --section WarpStateStats --section LaunchStats --clock-control none -k regex:"build_index" -s 2 -c 1 \
  -o gpurun_out/prof_k2 python tools/k2_trace.py c2 > gpurun_out/ncu_k2.log 2>&1; echo ncuk2=$? >> gpurun_out/status.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$? >> gpurun_out/status.txt
