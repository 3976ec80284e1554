#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_regions.py -q -x --timeout=600 > gpurun_out/pytest_regions.log 2>&1; echo pytest=$? > gpurun_out/status_regions.txt
for r in 8; do
TSR_K4R_REGION=$r timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_r$r.log 2>&1
TSR_K4R_REGION=$r timeout 600 ncu --set full --import-source on --clock-control none -k regex:"render_bwd_regions" -s 1 -c 1 -o gpurun_out/k4r_r$r python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k4r_$r.log 2>&1
done
