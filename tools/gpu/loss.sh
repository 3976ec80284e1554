#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_loss.py tests/test_gpu_loss_contract.py tests/test_gpu_acceptance.py tests/test_gpu_scene.py -q -x --timeout=600 > gpurun_out/pytest_loss.log 2>&1; echo pytest=$? > gpurun_out/status_loss.txt
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_loss.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv -k regex:ssim --log-file gpurun_out/launches_loss.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
