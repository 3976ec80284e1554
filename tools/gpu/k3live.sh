#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_regions.py tests/test_gpu_raster.py tests/test_gpu_scene.py tests/test_gpu_parity_scale.py tests/test_gpu_density.py -q -x --timeout=600 > gpurun_out/pytest_k3l.log 2>&1; echo pytest=$? > gpurun_out/status_k3l.txt
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_k3l.log 2>&1
timeout 300 python bench.py --config c3lo --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_k3l_c3lo.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_k3l.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
