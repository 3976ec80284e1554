#!/bin/bash
# quick GPU check: parity tests + bench + launch list
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -rf --timeout=300 -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/status.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$? >> gpurun_out/status.txt
