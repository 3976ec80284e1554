#!/bin/bash
# K2 per-phase traces for instrumented variants: bash tools/gpu/k2tracevar.sh trace trace_x ...
mkdir -p gpurun_out
for v in "$@"; do
  TSR_LIB=build/libtilesplat_b200_$v.so timeout 300 python tools/k2_trace.py c2 > gpurun_out/k2trace_$v.txt 2>&1
done
