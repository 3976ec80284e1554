#!/bin/bash
# FP32 pipe peak (FFMA / FFMA2 / FMUL / FADD) + a short C2 bench on the same box
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm --format=csv > gpurun_out/peak_nvsmi.csv 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fma_pipe tools/ubench/fma_pipe.cu && \
  (nvidia-smi --query-gpu=clocks.sm --format=csv,noheader -lms 200 > gpurun_out/peak_clk.txt & P=$!; /tmp/fma_pipe > gpurun_out/fma_pipe.txt 2>&1; /tmp/fma_pipe >> gpurun_out/fma_pipe.txt 2>&1; kill $P)
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_peak.log 2>&1; echo bench=$? >> gpurun_out/status_peak.txt
