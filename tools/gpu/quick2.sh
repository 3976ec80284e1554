#!/bin/bash
# parity subset + C2 bench
mkdir -p gpurun_out
export TSR_PARITY_LOG=gpurun_out/parity_stats.jsonl; rm -f $TSR_PARITY_LOG
timeout 900 python -m pytest tests/test_gpu_parity_scale.py tests/test_gpu_raster.py tests/test_gpu_scene.py tests/test_gpu_acceptance.py tests/test_gpu_density.py -q -x --timeout=600 > gpurun_out/pytest_q2.log 2>&1; echo pytest=$? > gpurun_out/status_q2.txt
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_q2.log 2>&1
