#!/bin/bash
mkdir -p gpurun_out
for mb in 6 7 8; do
  TSR_LIB=build/var/lib_vjp$mb.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_vjp$mb.log 2>&1
done
