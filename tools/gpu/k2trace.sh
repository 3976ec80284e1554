#!/bin/bash
mkdir -p gpurun_out
for c in c2 c3; do
  TSR_LIB=build/libtilesplat_b200_trace.so timeout 300 python tools/k2_trace.py $c > gpurun_out/k2trace_$c.txt 2>&1
done
