#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_scene.py tests/test_gpu_capacity.py tests/test_gpu_trainer.py tests/test_gpu_acceptance.py tests/test_gpu_projection_adam.py tests/test_gpu_density.py -q -x --timeout=900 > gpurun_out/pytest_fused.log 2>&1; echo pytest=$? > gpurun_out/status_fused.txt
for f in 1 0 1; do TSR_FUSED_ADAM=$f timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_fused$f.log 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fused.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
