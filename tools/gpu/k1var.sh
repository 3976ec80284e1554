#!/bin/bash
mkdir -p gpurun_out
for mb in 4 3; do
  TSR_LIB=build/var/lib_k1_$mb.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_k1_$mb.log 2>&1
done
