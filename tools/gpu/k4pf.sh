#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/k4pf_status.txt
make -j16 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_regions.py tests/test_gpu_parity_scale.py -q -x > gpurun_out/k4pf_pytest.log 2>&1; echo "pytest=$?" >> gpurun_out/k4pf_status.txt
for v in "$@"; do
  if [ "$v" = "base" ]; then lib=paper_2601_19489_b200/libtilesplat_b200.so; else lib=build/libtilesplat_b200_$v.so; fi
  for rep in 1 2 3; do
    TSR_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${v}_$rep.log 2>&1
  done
done
