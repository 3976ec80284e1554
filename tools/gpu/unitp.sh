#!/bin/bash
mkdir -p gpurun_out
make -j16 all > gpurun_out/make.log 2>&1 || { echo make failed; exit 1; }
timeout 600 python tools/unit_probe.py > gpurun_out/unit_probe.txt 2>&1
TSR_K4R_REGION=8 timeout 600 python tools/unit_probe.py >> gpurun_out/unit_probe.txt 2>&1
