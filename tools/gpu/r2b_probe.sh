#!/bin/bash
# round-2 (session 2) probe: K2 phase timeline, K4 + SSIM source-level captures, C2 bench
mkdir -p gpurun_out
make -j8 all > gpurun_out/make.log 2>&1 && make trace >> gpurun_out/make.log 2>&1
for c in c2 c3; do
  TSR_LIB=build/libtilesplat_b200_trace.so timeout 300 python tools/k2_trace.py $c > gpurun_out/k2trace_$c.txt 2>&1
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_probe.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"render_bwd|ssim|build_index" -s 3 -c 4 -o gpurun_out/probe_full python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_probe.log 2>&1
echo done > gpurun_out/probe_status.txt
