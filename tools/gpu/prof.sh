#!/bin/bash
# usage: tools_gpu_prof.sh <kernel regex> <skip> <count> <name>
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$1" -s $2 -c $3 -o gpurun_out/$4 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$4.log 2>&1; echo ncu=$? >> gpurun_out/status.txt
