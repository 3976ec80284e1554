#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
make trace >> gpurun_out/make.log 2>&1
timeout 900 python -m pytest tests/test_gpu_binning.py -q -x --timeout=600 > gpurun_out/pytest_k2.log 2>&1; echo pytest=$? > gpurun_out/status_k2.txt
for c in c2; do TSR_LIB=build/libtilesplat_b200_trace.so timeout 300 python tools/k2_trace.py $c > gpurun_out/k2trace_$c.txt 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"build_index" -s 2 -c 1 -o gpurun_out/k2_full python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_k2.log 2>&1
