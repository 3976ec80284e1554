#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_regions.py tests/test_gpu_parity_scale.py -q -x --timeout=600 > gpurun_out/pytest_ex.log 2>&1; echo pytest=$? > gpurun_out/status_ex.txt
for r in 8 4; do
TSR_K4R_REGION=$r timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_ex$r.log 2>&1
TSR_K4R_REGION=$r timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_ex$r.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
