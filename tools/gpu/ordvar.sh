#!/bin/bash
mkdir -p gpurun_out
make -j16 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
for v in "$@"; do
  if [ "$v" = "base" ]; then lib=paper_2601_19489_b200/libtilesplat_b200.so; else lib=build/libtilesplat_b200_$v.so; fi
  for rep in 1 2; do
    TSR_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${v}_$rep.log 2>&1
  done
  TSR_LIB=$lib timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${v}_c3.log 2>&1
  TSR_LIB=$lib timeout 300 python bench.py --config c3lo --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${v}_c3lo.log 2>&1
done
