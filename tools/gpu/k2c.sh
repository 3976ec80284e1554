#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
make trace >> gpurun_out/make.log 2>&1
timeout 900 python -m pytest tests/test_gpu_binning.py tests/test_gpu_scene.py -q -x --timeout=600 > gpurun_out/pytest_k2.log 2>&1; echo pytest=$? > gpurun_out/status_k2.txt
for c in c2 c3; do TSR_LIB=build/libtilesplat_b200_trace.so timeout 300 python tools/k2_trace.py $c > gpurun_out/k2trace_$c.txt 2>&1; done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_k2_c2.log 2>&1
timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_k2_c3.log 2>&1
