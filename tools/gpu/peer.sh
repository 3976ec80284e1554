#!/bin/bash
# peer ZeRO-1 kernel: parity tests + launch times under ncu
mkdir -p gpurun_out
make -j16 > gpurun_out/make.log 2>&1 || { tail -20 gpurun_out/make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parallel.py -x -q 2>&1 | tail -15 | tee gpurun_out/peer_tests.log
