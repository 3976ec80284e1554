#!/bin/bash
mkdir -p gpurun_out
make -j16 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
timeout 600 python tools/k4_order_probe.py > gpurun_out/k4_order_probe.txt 2>&1
