#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
for px in 4 8; do
TSR_K4R_PX=$px timeout 900 python -m pytest tests/test_gpu_regions.py -q -x --timeout=600 > gpurun_out/pytest_px$px.log 2>&1; echo px$px pytest=$? >> gpurun_out/status_px.txt
TSR_K4R_PX=$px timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_px$px.log 2>&1
done
TSR_K4R_PX=8 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"render_bwd_regions" -s 1 -c 1 -o gpurun_out/k4r_px8 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_px8.log 2>&1
