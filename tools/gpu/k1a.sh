#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/k1a_status.txt
make -j16 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_scene.py tests/test_gpu_projection_adam.py tests/test_gpu_binning.py tests/test_gpu_projection_contract.py -q -x > gpurun_out/k1a_pytest.log 2>&1; echo "pytest=$?" >> gpurun_out/k1a_status.txt
for v in "$@"; do
  if [ "$v" = "base" ]; then lib=paper_2601_19489_b200/libtilesplat_b200.so; else lib=build/libtilesplat_b200_$v.so; fi
  for rep in 1 2; do
    TSR_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${v}_$rep.log 2>&1
  done
  TSR_LIB=$lib timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${v}_c3.log 2>&1
done
TSR_LIB=paper_2601_19489_b200/libtilesplat_b200.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cull_compact --csv --log-file gpurun_out/k1a_new.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
TSR_LIB=build/libtilesplat_b200_k1aold.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cull_compact --csv --log-file gpurun_out/k1a_old.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
